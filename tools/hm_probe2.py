"""Per-kernel-family profile of one evaluation at moderate n (diagnostics)."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1709_04419_b200 as hm
from synthetic import uniform_iid, perturbed_mesh, standard_normal
for n, leaf in [(2048, 32), (4096, 32), (8192, 32)]:
    pts = uniform_iid(n, 1)
    theta = (1.0, 0.0334, 0.5)
    H = hm.HMatrix(pts, theta, eps=1e-8, leaf=leaf, eta=2.0, kmax=160)
    H.profile(True)
    t0 = time.time(); H.cholesky(); t1 = time.time()
    Z = standard_normal(n, 1, 3); out = H.loglik(Z)
    print(f"n={n}: chol {t1-t0:.3f}s", H.timings(), {k: round(v, 3) for k, v in H.stats().items()}, flush=True)
    for k, v in H.kernel_stats().items():
        print("   ", k, {a: (round(b, 3) if a == "ms" else b) for a, b in v.items()},
              "GF/s=%.1f GB/s=%.1f" % (v["flops"] / max(v["ms"], 1e-9) / 1e6, v["bytes"] / max(v["ms"], 1e-9) / 1e6), flush=True)
    H.close()
