"""Exec-mode determinism / correctness probe."""
import os, sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1709_04419_b200 as hm
from synthetic import uniform_iid, standard_normal
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-10
pts = uniform_iid(n, 11)
theta = (1.0, 0.0864, 0.5)
Z = standard_normal(n, 1, 5)
H = hm.HMatrix(pts, theta, eps=eps, leaf=32, eta=2.0)
for mode in (0, 1, 0, 1, 1, 1):
    H.set_exec_mode(mode)
    H.assemble(theta)
    try:
        H.cholesky()
        out = H.loglik(Z)[0]
        print("mode", mode, repr(out.tolist()), H.stats()["max_rank_L"], flush=True)
    except Exception as e:
        print("mode", mode, "FAILED", e, flush=True)
