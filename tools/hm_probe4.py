"""64k determinism probe: wave vs exec executor, repeated."""
import os, sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1709_04419_b200 as hm
from synthetic import perturbed_mesh, standard_normal
pts = perturbed_mesh(256, 0.4, 2)
theta = (1.0, 0.1, 0.5)
Z = standard_normal(65536, 1, 3)
H = hm.HMatrix(pts, theta, eps=1e-7, leaf=64, eta=2.0)
for mode in [int(c) for c in (sys.argv[1] if len(sys.argv) > 1 else "0011")]:
    H.set_exec_mode(mode)
    H.assemble(theta)
    H.cholesky()
    out = H.loglik(Z)[0]
    print("mode", mode, repr(out.tolist()), H.timings(), flush=True)
