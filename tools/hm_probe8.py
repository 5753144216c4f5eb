"""configs[1] grid (n = 16384): H (absolute eps, default) vs GPU dense path on a
random sample + the four corners; prints max relative errors per eps."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1709_04419_b200 as hm
from synthetic import uniform_iid, standard_normal, theta_grid_ell_nu
n = 16384
pts = uniform_iid(n, 1)
Ht = hm.HMatrix(pts, (1.0, 0.2, 1.5), eps=1e-10, leaf=32)
Ht.cholesky()
Z = Ht.sample(standard_normal(n, 1, 3))[:, 0]
Ht.close()
grid = theta_grid_ell_nu()
rng = np.random.default_rng(11)
idx = sorted(set(rng.choice(len(grid), 36, replace=False).tolist()) | {0, 19, 380, 399})
H5 = hm.HMatrix(pts, tuple(grid[0]), eps=1e-5, leaf=32)
H8 = hm.HMatrix(pts, tuple(grid[0]), eps=1e-8, leaf=32)
worst = {1e-5: (0, None), 1e-8: (0, None)}
fails = {1e-5: 0, 1e-8: 0}
t0 = time.time()
for i in idx:
    th = tuple(grid[i])
    d = hm.dense_loglik(pts, th, Z)[0, 0]
    for eps, H in ((1e-5, H5), (1e-8, H8)):
        H.assemble(th)
        try:
            H.cholesky()
            e = abs(H.loglik(Z)[0, 0] - d) / abs(d)
            if e > worst[eps][0]:
                worst[eps] = (e, th)
        except hm.HMError as ex:
            fails[eps] += 1
            print("fail", eps, th, ex, flush=True)
print("points", len(idx), "worst", worst, "fails", fails, "%.0fs" % (time.time() - t0), flush=True)
