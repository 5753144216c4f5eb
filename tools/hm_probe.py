"""Quick GPU probe: build / assemble / Cholesky / loglik timings and stats at several sizes."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1709_04419_b200 as hm
from synthetic import uniform_iid, perturbed_mesh, standard_normal

cases = [(16384, 32, 1e-8, (1.0, 0.0334, 0.5), "uniform"), (16384, 32, 1e-5, (1.0, 0.0334, 0.5), "uniform"),
         (65536, 64, 1e-7, (1.0, 0.1, 0.5), "mesh"), (65536, 64, 1e-7, (1.0, 0.1, 1.0), "mesh"),
         (16384, 32, 1e-8, (1.0, 0.2, 1.5), "uniform")]
if len(sys.argv) > 1:
    cases = cases[: int(sys.argv[1])]
for n, leaf, eps, theta, kind in cases:
    pts = uniform_iid(n, 1) if kind == "uniform" else perturbed_mesh(int(round(n ** 0.5)), 0.4, 2)
    try:
        t0 = time.time()
        H = hm.HMatrix(pts, theta, eps=eps, leaf=leaf, eta=2.0, kmax=160)
        t1 = time.time()
        H.cholesky()
        t2 = time.time()
        Z = standard_normal(n, 1, 3)
        out = H.loglik(Z)
        t3 = time.time()
        print(f"n={n} leaf={leaf} eps={eps} theta={theta}: build {t1-t0:.2f}s chol {t2-t1:.3f}s loglik {t3-t2:.3f}s",
              H.timings(), {k: round(v, 3) for k, v in H.stats().items()}, out.tolist(), flush=True)
        H.profile(True)
        for rep in range(2):
            t0 = time.time(); H.assemble(theta); H.cholesky(); out = H.loglik(Z); t1 = time.time()
            print("  repeat eval %.3fs" % (t1 - t0), H.timings(), flush=True)
        ks = H.kernel_stats()
        for k, v in ks.items():
            print("   ", k, {a: (round(b, 3) if a == "ms" else b) for a, b in v.items()},
                  "GF/s=%.1f GB/s=%.1f" % (v["flops"] / max(v["ms"], 1e-9) / 1e6, v["bytes"] / max(v["ms"], 1e-9) / 1e6))
        H.close()
    except Exception as e:
        print(f"n={n} eps={eps} theta={theta}: FAILED {e}", flush=True)
