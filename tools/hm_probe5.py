"""Determinism bisection: checksums after assemble / after Cholesky, repeated."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1709_04419_b200 as hm
from synthetic import perturbed_mesh, uniform_iid, standard_normal
for kind, n, leaf, eps, theta in [("mesh", 16384, 64, 1e-7, (1.0, 0.1, 0.5)), ("mesh", 65536, 64, 1e-7, (1.0, 0.1, 0.5)),
                                  ("uniform", 16384, 32, 1e-8, (1.0, 0.0334, 0.5))]:
    pts = perturbed_mesh(int(n ** 0.5), 0.4, 2) if kind == "mesh" else uniform_iid(n, 1)
    Z = standard_normal(n, 1, 3)
    H = hm.HMatrix(pts, theta, eps=eps, leaf=leaf, eta=2.0)
    H.set_exec_mode(0)
    for rep in range(3):
        H.assemble(theta)
        ca = H.checksum()
        H.cholesky()
        cl = H.checksum()
        out = H.loglik(Z)[0]
        print(kind, n, leaf, rep, "asm", ca.tolist(), "chol", cl.tolist(), "ll", out.tolist(), flush=True)
    H.close()
