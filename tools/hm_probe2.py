"""Per-kernel-family profile of one evaluation (diagnostics): both executors."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1709_04419_b200 as hm
from synthetic import uniform_iid, perturbed_mesh, standard_normal
cases = [(8192, 32, "uniform", (1.0, 0.0334, 0.5), 1e-8, (0, 1)), (65536, 64, "mesh", (1.0, 0.1, 0.5), 1e-7, (1,))]
for n, leaf, kind, theta, eps, modes in cases:
    pts = uniform_iid(n, 1) if kind == "uniform" else perturbed_mesh(256, 0.4, 2)
    Z = standard_normal(n, 1, 3)
    H = hm.HMatrix(pts, theta, eps=eps, leaf=leaf, eta=2.0, kmax=160)
    for mode in modes:
        H.set_exec_mode(mode)
        for rep in range(2):
            H.assemble(theta)
            H.profile(True)
            t0 = time.time(); H.cholesky(); t1 = time.time()
            out = H.loglik(Z)
            print(f"n={n} mode={mode} rep={rep}: chol {t1-t0:.3f}s", H.timings(), out.tolist(), flush=True)
        print({k: round(v, 3) for k, v in H.stats().items()})
        for k, v in H.kernel_stats().items():
            if v["launches"]:
                print("   ", k, {a: (round(b, 3) if a == "ms" else b) for a, b in v.items()},
                      "GF/s=%.1f GB/s=%.1f" % (v["flops"] / max(v["ms"], 1e-9) / 1e6, v["bytes"] / max(v["ms"], 1e-9) / 1e6), flush=True)
    H.close()
