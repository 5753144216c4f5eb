"""Scaling probe toward configs[4]: one evaluation at n = 2^18 (and 2^20 if asked)."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1709_04419_b200 as hm
from synthetic import perturbed_mesh, standard_normal
for side in [int(a) for a in sys.argv[1:]] or [512]:
    pts = perturbed_mesh(side, 0.4, 2)
    n = len(pts)
    t0 = time.perf_counter()
    H = hm.HMatrix(pts, (1.0, 0.1, 0.5), eps=1e-7, leaf=64, eta=2.0, kmax=64)
    t1 = time.perf_counter()
    H.cholesky()
    Z = H.sample(standard_normal(n, 1, 3))
    for th in [(1.0, 0.1, 0.5), (1.0, 0.102, 0.5)]:
        H.assemble(th)
        H.cholesky()
        ll = H.loglik(Z)[0]
        print(f"n={n} build(host plan + upload + assemble)={t1 - t0:.1f}s theta={th} loglik={ll.tolist()} "
              f"timings={H.timings()} stats={ {k: v for k, v in H.stats().items() if k in ('max_rank_L', 'bytes_L', 'pool_bytes')} }",
              flush=True)
    H.close()
