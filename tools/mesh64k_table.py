"""configs[2] full-size accuracy (diagnostic): n = 65,536 jittered mesh (Eq. 3,
synthetic.perturbed_mesh(256, 0.4, 2)), leaf 64, nu in {0.5, 1.0}; H likelihood at
eps in {1e-8, 1e-7, 1e-5} against the GPU dense fp64 path at n = 65,536 (34 GB),
Z = L~ xi drawn by the H sampler at eps = 1e-10 (an input, the same for both)."""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1709_04419_b200 as hm
from synthetic import perturbed_mesh, standard_normal
pts = perturbed_mesh(256, 0.4, 2)
n = len(pts)
out = []
for nu in (0.5, 1.0):
    th = (1.0, 0.1, nu)
    t0 = time.time()
    Hs = hm.HMatrix(pts, th, eps=1e-10, leaf=64, eta=2.0)
    Hs.cholesky()
    Z = Hs.sample(standard_normal(n, 1, seed=42))[:, 0]
    Hs.close()
    t1 = time.time()
    d = hm.dense_loglik(pts, th, Z)[0]
    t2 = time.time()
    rec = {"theta": th, "dense": d.tolist(), "dense_s": t2 - t1, "sample_s": t1 - t0}
    for eps in (1e-8, 1e-7, 1e-5):
        try:
            H = hm.HMatrix(pts, th, eps=eps, leaf=64, eta=2.0, kmax=64)
            H.cholesky()
            g = H.loglik(Z)[0]
            rec[f"{eps:g}"] = abs(g[0] - d[0]) / abs(d[0])
            H.close()
        except hm.HMError as e:
            rec[f"{eps:g}"] = str(e)
    print(json.dumps(rec), flush=True)
    out.append(rec)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "mesh64k_table.json"), "w"), indent=1)
