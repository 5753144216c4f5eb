"""Small wave-mode evaluation (for compute-sanitizer)."""
import sys
sys.path.insert(0, "/root/repo")
import paper_1709_04419_b200 as hm
from synthetic import uniform_iid, standard_normal
n = int(sys.argv[1]) if len(sys.argv) > 1 else 600
pts = uniform_iid(n, 11)
theta = (1.0, 0.0864, 0.5)
H = hm.HMatrix(pts, theta, eps=1e-8, leaf=16, eta=2.0)
H.set_exec_mode(0)
H.assemble(theta)
try:
    H.cholesky()
    print("ok", H.loglik(standard_normal(n, 1, 5))[0].tolist())
except Exception as e:
    print("FAILED", e)
