"""Trace one H-Cholesky (persistent executor) and analyse it against its plan."""
import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import paper_1709_04419_b200 as hm
from synthetic import uniform_iid, perturbed_mesh, standard_normal
from trace_analyze import analyse
which = sys.argv[1] if len(sys.argv) > 1 else "8k"
KMAX = int(sys.argv[2]) if len(sys.argv) > 2 else 64
if which == "8k":
    pts, leaf, theta, eps = uniform_iid(8192, 1), 32, (1.0, 0.0334, 0.5), 1e-8
else:
    pts, leaf, theta, eps = perturbed_mesh(256, 0.4, 2), 64, (1.0, 0.1, 0.5), 1e-7
H = hm.HMatrix(pts, theta, eps=eps, leaf=leaf, eta=2.0, kmax=KMAX)
H.cholesky()
H.assemble(theta)
H.trace(True)
H.cholesky()
H.trace(False, f"/tmp/trace_{which}.bin")
T = hm.Tree(pts, leaf, 2.0)
T.plan_dump(f"/tmp/plan_{which}.bin", KMAX)
print(H.timings())
print(analyse(f"/tmp/plan_{which}.bin", f"/tmp/trace_{which}.bin", "chol", grid=148))
import subprocess
print(subprocess.run([sys.executable, "/root/repo/tools/stall_probe.py", f"/tmp/plan_{which}.bin", f"/tmp/trace_{which}.bin"],
                     capture_output=True, text=True).stdout)
