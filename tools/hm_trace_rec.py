"""Trace the assembly's recompression phase and the solve at n = 64k (bench config)."""
import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import numpy as np
import paper_1709_04419_b200 as hm
from synthetic import perturbed_mesh, standard_normal
from trace_analyze import analyse
pts, leaf, theta, eps = perturbed_mesh(256, 0.4, 2), 64, (1.0, 0.1, 0.5), 1e-7
H = hm.HMatrix(pts, theta, eps=eps, leaf=leaf, eta=2.0, kmax=64)
H.cholesky()
T = hm.Tree(pts, leaf, 2.0)
T.plan_dump("/tmp/plan_64k.bin", 64)
H.trace(True)
H.assemble(theta)
H.trace(False, "/tmp/trace_rec.bin")
print(H.timings())
print(analyse("/tmp/plan_64k.bin", "/tmp/trace_rec.bin", "recompress", grid=148, top=8))
H.cholesky()
Z = standard_normal(len(pts), 1, 3)
H.trace(True)
H.loglik(Z)
H.trace(False, "/tmp/trace_sol.bin")
print(H.timings())
print(analyse("/tmp/plan_64k.bin", "/tmp/trace_sol.bin", "solve", grid=148, top=8))
