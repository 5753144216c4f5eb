"""configs[1] accuracy table on the B200 (diagnostic; writes gpurun_out/config1_table.json).

n = 16,384 uniform iid points (synthetic.uniform_iid(16384, 1)), Z from
tests/golden/config1_Z.npy (oracle-drawn at theta* = (1, 0.2, 1.5)).  For every
point of the 20 x 20 (ell, nu) grid (synthetic.theta_grid_ell_nu):
  * the GPU dense fp64 path (hm_dense_loglik; pinned to the oracle in
    tests/test_gpu_dense.py) and its own rounding floor (points permuted),
  * the H likelihood at eps in {1e-8, 1e-5} with eps_chol = eps (one accuracy for
    C~ and L~, Table 3 l.483) and with eps_chol = eps / 1000 (separate
    factor accuracy, PAPER.md l.474-476 / Fig. 7), |dL| / |L| or NOT_SPD;
  * on every 40th point and theta*: lambda_min(C) (torch eigvalsh on the device);
  * at theta*: rho(C~^-1 C - I) (Theorem 2's hypothesis, l.291-300) for every
    factor that exists, C~ = L~ L~^T with L~ expanded by the sampler.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1709_04419_b200 as hm  # noqa: E402
from synthetic import theta_grid_ell_nu, uniform_iid  # noqa: E402

n = 16384
pts = uniform_iid(n, 1)
Z = np.load(os.path.join(ROOT, "tests", "golden", "config1_Z.npy"))
grid = [tuple(map(float, g)) for g in theta_grid_ell_nu()]
STAR = (1.0, 0.2, 1.5)
perm = np.random.default_rng(0).permutation(n)
VARIANTS = [(1e-8, 1e-8), (1e-5, 1e-5), (1e-8, 1e-11), (1e-5, 1e-8)]
only = os.environ.get("CFG1_POINTS")          # e.g. "0:40" for a quick look
sel = list(range(len(grid)))
if only:
    a, b = map(int, only.split(":"))
    sel = sel[a:b]


def lam_min(theta):
    import torch
    C = hm.matern_block(pts, pts, theta)
    C[np.arange(n), np.arange(n)] = theta[0]
    return float(torch.linalg.eigvalsh(torch.from_numpy(C).cuda())[0])


def rho(theta, eps, eps_chol):
    """rho(C~^-1 C - I), C~ = L~ L~^T: eigenvalues of L~^-1 C L~^-T - I."""
    import torch
    H = hm.HMatrix(pts, theta, eps=eps, leaf=32, eta=2.0, eps_chol=eps_chol)
    H.cholesky()
    t = hm.Tree(pts, 32, 2.0)
    p = t.perm()
    S = H.sample(np.eye(n))                       # S = P^T L~ P (original order)
    H.close()
    L = torch.from_numpy(S[np.ix_(p, p)]).cuda()  # L~ in tree order (lower triangular)
    C = hm.matern_block(pts[p], pts[p], theta)
    C[np.arange(n), np.arange(n)] = theta[0]
    C = torch.from_numpy(C).cuda()
    X = torch.linalg.solve_triangular(L, C, upper=False)
    M = torch.linalg.solve_triangular(L, X.T.contiguous(), upper=False)
    M = 0.5 * (M + M.T)
    ev = torch.linalg.eigvalsh(M)
    return float(torch.max(torch.abs(ev - 1.0)))


rows = []
H = {}
t0 = time.time()
for i in sel:
    th = grid[i]
    rec = {"i": i, "theta": th}
    try:
        d = hm.dense_loglik(pts, th, Z)[0, 0]
        d2 = hm.dense_loglik(pts[perm], th, Z[perm])[0, 0]
        rec["dense"] = d
        rec["floor"] = abs(d2 - d) / abs(d)
    except hm.HMError as e:
        rec["dense"] = None
        rec["dense_error"] = str(e)
    for eps, epsl in VARIANTS:
        key = f"{eps:g}/{epsl:g}"
        if key not in H:
            H[key] = hm.HMatrix(pts, th, eps=eps, leaf=32, eta=2.0, eps_chol=epsl)
        h = H[key]
        try:
            h.assemble(th)
            h.cholesky()
            ll = h.loglik(Z)[0, 0]
            rec[key] = abs(ll - d) / abs(d) if rec["dense"] is not None else None
        except hm.HMError as e:
            rec[key] = "NOT_SPD" if e.code == -3 else str(e)
    if i % 40 == 0:
        rec["lambda_min"] = lam_min(th)
    rows.append(rec)
    print(json.dumps(rec), flush=True)
out = {"n": n, "variants": [f"{a:g}/{b:g}" for a, b in VARIANTS], "rows": rows, "seconds": time.time() - t0}
# theta*: conditioning and Theorem 2's rho for each factor that exists
star = {"theta": STAR, "lambda_min": lam_min(STAR)}
for eps, epsl in VARIANTS:
    key = f"{eps:g}/{epsl:g}"
    try:
        star["rho " + key] = rho(STAR, eps, epsl)
    except hm.HMError as e:
        star["rho " + key] = str(e)
out["star"] = star
print(json.dumps(star), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "config1_table.json"), "w") as f:
    json.dump(out, f, indent=1)
