"""Where does the H-likelihood error of configs[1] come from? (diagnostic, B200)

For theta* = (1, 0.2, 1.5) and a few smooth grid points, n = 16,384 uniform points,
Z = tests/golden/config1_Z.npy:
  * C (dense, device Matern), its spectrum: lambda_min and how many eigenvalues fall
    below eps * sigma^2 for eps in {1e-5, 1e-8};
  * C~ = hm_to_dense after assembly at eps: max over admissible blocks of
    ||C - C~||_F (>= the spectral norm Remark 2 asks to be <= eps sigma^2), lambda_min(C~), and the EXACT
    likelihood of C~ (dense Cholesky of C~ on the device) -- the assembly error;
  * L~ from the H-Cholesky: the H likelihood -- assembly + factorisation error;
  * rho(C~^-1 C - I) (Theorem 2, l.291-300) whenever C~ is positive definite.
Writes gpurun_out/assembly_error.json.
"""
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1709_04419_b200 as hm  # noqa: E402
from synthetic import uniform_iid  # noqa: E402

n = 16384
pts = uniform_iid(n, 1)
Z = np.load(os.path.join(ROOT, "tests", "golden", "config1_Z.npy"))
tree = hm.Tree(pts, 32, 2.0)
perm = tree.perm()
blocks = tree.blocks()
adm = blocks[blocks[:, 5] == 1]
dev = "cuda"
Zt = torch.from_numpy(Z).to(dev)


def ll_of(Cd):
    L, info = torch.linalg.cholesky_ex(Cd)
    if int(info) != 0:
        return None
    v = torch.linalg.solve_triangular(L, Zt[:, None], upper=False)
    ld = 2.0 * torch.log(torch.diagonal(L)).sum()
    q = (v * v).sum()
    return float(-0.5 * n * math.log(2 * math.pi) - 0.5 * ld - 0.5 * q)


out = []
thetas = [(1.0, 0.2, 1.5), (1.0, 0.20743100888923838, 1.5526315789473684),
          (1.0, 0.35853283845514233, 1.5526315789473684), (1.0, 0.1338904101224472, 2.0),
          (1.0, 0.0964175997942495, 1.2842105263157895)]
for th in thetas:
    C = hm.matern_block(pts, pts, th)
    C[np.arange(n), np.arange(n)] = th[0]
    Cd = torch.from_numpy(C).to(dev)
    ev = torch.linalg.eigvalsh(Cd)
    rec = {"theta": th, "lambda_min": float(ev[0]),
           "n_eig_below_1e-5": int((ev < 1e-5).sum()), "n_eig_below_1e-8": int((ev < 1e-8).sum()),
           "loglik_exact": ll_of(Cd)}
    Ct = Cd[perm][:, perm]            # tree order
    for eps in (1e-8, 1e-5):
        H = hm.HMatrix(pts, th, eps=eps, leaf=32, eta=2.0)
        Ch = torch.from_numpy(H.to_dense()).to(dev)
        Cht = Ch[perm][:, perm]
        worst = 0.0
        for (a, b, c, d, lvl, _) in adm:
            D = Ct[a:b, c:d] - Cht[a:b, c:d]
            worst = max(worst, float(torch.linalg.matrix_norm(D)))
        r = {"max_block_err_F": worst, "lambda_min_Ctilde": float(torch.linalg.eigvalsh(Ch)[0]),
             "loglik_Ctilde_exact": ll_of(Ch)}
        try:
            H.cholesky()
            r["loglik_H"] = float(H.loglik(Z)[0, 0])
        except hm.HMError as e:
            r["loglik_H"] = str(e)
        if r["loglik_Ctilde_exact"] is not None:
            Lc = torch.linalg.cholesky(Ch)
            X = torch.linalg.solve_triangular(Lc, Cd, upper=False)
            M = torch.linalg.solve_triangular(Lc, X.T.contiguous(), upper=False)
            r["rho_Ctilde"] = float(torch.max(torch.abs(torch.linalg.eigvalsh(0.5 * (M + M.T)) - 1.0)))
        H.close()
        rec[f"{eps:g}"] = r
        del Ch, Cht
    print(json.dumps(rec), flush=True)
    out.append(rec)
    del Cd, Ct
    torch.cuda.empty_cache()
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "assembly_error.json"), "w"), indent=1)
