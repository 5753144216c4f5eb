"""config1 sensitive point: H vs GPU dense at several eps."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1709_04419_b200 as hm
from synthetic import uniform_iid, standard_normal
n = 16384
pts = uniform_iid(n, 1)
Ht = hm.HMatrix(pts, (1.0, 0.2, 1.5), eps=1e-10, leaf=32)
Ht.cholesky()
Z = Ht.sample(standard_normal(n, 1, 3))[:, 0]
for th in [(1.0, 0.20743100888923838, 1.2842105263157895), (1.0, 0.1, 0.8), (1.0, 0.05, 1.5), (1.0, 0.3, 0.5)]:
    d = hm.dense_loglik(pts, th, Z)[0]
    row = [th, d[0]]
    for eps in (1e-5, 1e-8, 1e-9, 1e-10):
        try:
            H = hm.HMatrix(pts, th, eps=eps, leaf=32)
            H.cholesky()
            g = H.loglik(Z)[0]
            row.append((eps, float((g[0] - d[0]) / abs(d[0]))))
            H.close()
        except Exception as e:
            row.append((eps, str(e)[:30]))
    print(row, flush=True)
