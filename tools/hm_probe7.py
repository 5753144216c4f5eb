"""config1 grid points: H (eps 1e-5 / 1e-8) vs GPU dense, relative vs absolute eps; timings."""
import os, sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1709_04419_b200 as hm
from synthetic import uniform_iid, standard_normal
n = 16384
pts = uniform_iid(n, 1)
Ht = hm.HMatrix(pts, (1.0, 0.2, 1.5), eps=1e-10, leaf=32)
Ht.cholesky()
Z = Ht.sample(standard_normal(n, 1, 3))[:, 0]
Ht.close()
for th in [(1.0, 0.2880493075077518, 0.7473684210526316), (1.0, 0.1, 0.8), (1.0, 0.3, 0.5), (1.0, 0.05, 1.5)]:
    d = hm.dense_loglik(pts, th, Z)[0, 0]
    row = [tuple(round(x, 3) for x in th)]
    for eps in (1e-5, 1e-8):
        try:
            H = hm.HMatrix(pts, th, eps=eps, leaf=32)
            t0 = time.time(); H.cholesky(); t1 = time.time()
            g = H.loglik(Z)[0, 0]
            row.append((eps, "%.1e" % ((g - d) / abs(d)), "chol %.0f ms" % (H.timings()["cholesky_ms"]), "rkL %d" % H.stats()["max_rank_L"]))
            H.close()
        except Exception as e:
            row.append((eps, str(e)[:28]))
    print(row, flush=True)
