"""Writes the configs[1] golden values -- calls ONLY oracle/ and synthetic/.

BASELINE.json configs[1]: n = 16,384 locations iid uniform in [0,1]^2, Matern
(sigma^2, ell, nu) = (1.0, 0.2, 1.5), likelihood on a 20 x 20 (ell, nu) grid at
fixed sigma^2 compared with the dense oracle.  Data recipe (configs[0]'s, the
only one BASELINE states): Z = L xi from the dense Cholesky of the true C
(sec. 4, l.308 "Z = L xi", here with the exact L).

Outputs (tests/golden/):
  config1_Z.npy         Z (16,384 doubles, original point order)
  config1_oracle.json   {"theta": [...], "loglik", "logdet", "quad"} per point for theta*
                        and a 5 x 5 sub-grid of synthetic.theta_grid_ell_nu()
                        (ell index and nu index in {0, 5, 10, 15, 19}), each the
                        oracle's Eq. (1) (oracle.dense.loglik, quadrature K_nu);
                        for theta* also lambda_min(C) (scipy eigh) and the oracle's
                        own rounding floor (|L(perm) - L| / |L| for a permuted
                        point order).

Run:  python tests/golden/gen_config1.py [--workers 3]     (~1 h on 8 cores)
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import dense as od  # noqa: E402
from synthetic import standard_normal, theta_grid_ell_nu, uniform_iid  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
N = 16384
THETA_STAR = (1.0, 0.2, 1.5)
SUB = (0, 5, 10, 15, 19)


def points():
    return uniform_iid(N, seed=1)


def grid_points():
    g = theta_grid_ell_nu()
    return [tuple(map(float, g[i * 20 + j])) for i in SUB for j in SUB]


def one(theta):
    pts = points()
    Z = np.load(os.path.join(HERE, "config1_Z.npy"))
    t0 = time.time()
    try:
        ll, ld, q = od.loglik(pts, Z, theta)
        rec = {"theta": list(theta), "loglik": ll, "logdet": ld, "quad": q}
    except np.linalg.LinAlgError as e:          # C numerically indefinite in fp64
        rec = {"theta": list(theta), "loglik": None, "logdet": None, "quad": None, "error": str(e)}
    rec["seconds"] = round(time.time() - t0, 1)
    print(json.dumps(rec), flush=True)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=3)
    args = ap.parse_args()
    pts = points()
    zpath = os.path.join(HERE, "config1_Z.npy")
    star = {}
    if not os.path.exists(zpath):
        C = od.covariance(pts, THETA_STAR)
        L = np.linalg.cholesky(C)
        Z = L @ standard_normal(N, 1, seed=3)[:, 0]
        np.save(zpath, Z)
        import scipy.linalg
        lam = scipy.linalg.eigh(C, eigvals_only=True, subset_by_index=[0, 0])[0]
        ll, ld, q = od.loglik_from_cov(C, Z)
        p = np.random.default_rng(0).permutation(N)
        ll2, _, _ = od.loglik_from_cov(C[np.ix_(p, p)], Z[p])
        star = {"lambda_min": float(lam), "oracle_perm_floor": abs(ll2 - ll) / abs(ll)}
        del C, L
    thetas = [THETA_STAR] + grid_points()
    with mp.Pool(args.workers) as pool:
        recs = pool.map(one, thetas, chunksize=1)
    recs[0].update(star)
    out = {"config": "BASELINE configs[1]", "n": N, "points": "synthetic.uniform_iid(16384, seed=1)",
           "Z": "config1_Z.npy = L* xi, L* = chol(oracle.dense.covariance(points, theta*)), "
                "xi = synthetic.standard_normal(16384, 1, seed=3)",
           "theta_star": list(THETA_STAR), "records": recs}
    with open(os.path.join(HERE, "config1_oracle.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
