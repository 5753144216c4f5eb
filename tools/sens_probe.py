"""Relative error of the H likelihood at the configs[1] 'sensitive point' vs eps
(tests/test_gpu_fullsize.py::test_config1_sensitive_point_converges), printed per eps."""
import sys
sys.path.insert(0, "/root/repo")
import paper_1709_04419_b200 as hm
from synthetic import uniform_iid, standard_normal
n = 16384
pts = uniform_iid(n, seed=1)
Ht = hm.HMatrix(pts, (1.0, 0.2, 1.5), eps=1e-10, leaf=32, eta=2.0)
Ht.cholesky()
Z = Ht.sample(standard_normal(n, 1, seed=3))[:, 0]
Ht.close()
th = (1.0, 0.20743100888923838, 1.2842105263157895)
dense = hm.dense_loglik(pts, th, Z)[0, 0]
for eps in (1e-8, 1e-9, 1e-10, 1e-11, 1e-12):
    H = hm.HMatrix(pts, th, eps=eps, leaf=32, eta=2.0)
    H.cholesky()
    print(f"eps {eps:.0e}  rel err {abs(H.loglik(Z)[0, 0] - dense) / abs(dense):.3e}", flush=True)
    H.close()
