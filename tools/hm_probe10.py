"""configs[1] sensitive point: dense rounding floor (permuted points) vs H error per eps."""
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
Ht.close()
th = (1.0, 0.20743100888923838, 1.2842105263157895)
d = hm.dense_loglik(pts, th, Z)[0, 0]
for seed in (5, 6, 7):
    perm = np.random.default_rng(seed).permutation(n)
    dp = hm.dense_loglik(pts[perm], th, Z[perm])[0, 0]
    print("perm floor", abs(d - dp) / abs(d), flush=True)
for eps in (1e-8, 1e-9, 1e-10, 1e-11):
    H = hm.HMatrix(pts, th, eps=eps, leaf=32)
    H.cholesky()
    v = H.loglik(Z)[0, 0]
    print(eps, abs(v - d) / abs(d), v, d, flush=True)
    H.close()
