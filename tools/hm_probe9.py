"""Rounding floor of the configs[1] likelihood in the smooth corner: the GPU
dense fp64 path on the same points in two orders (a permutation changes only the
rounding order), next to the H error at eps = 1e-8 / 1e-10."""
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
perm = np.random.default_rng(5).permutation(n)
for th in [(1.0, 0.4, 1.0158), (1.0, 0.2, 1.5), (1.0, 0.1667, 1.9105), (1.0, 0.0964, 1.8210), (1.0, 0.2880, 0.7474), (1.0, 0.05, 0.3)]:
    d = hm.dense_loglik(pts, th, Z)[0, 0]
    dp = hm.dense_loglik(pts[perm], th, Z[perm])[0, 0]
    row = [f"theta={th} dense={d:.10e} perm_floor={abs(d - dp) / abs(d):.2e}"]
    for eps in (1e-5, 1e-8, 1e-10):
        try:
            H = hm.HMatrix(pts, th, eps=eps, leaf=32)
            H.cholesky()
            row.append(f"H{eps:g}={abs(H.loglik(Z)[0, 0] - d) / abs(d):.2e}")
            H.close()
        except hm.HMError as ex:
            row.append(f"H{eps:g}=NOT_SPD")
    print(" ".join(row), flush=True)
