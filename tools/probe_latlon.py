"""configs[4] geometry probe (diagnostic): n points of synthetic.latlon_dropout, Matern
(1, 0.1 deg, 0.35); max ranks of C~ and L~, device pool and timings at eps in
{1e-6, 1e-8}, for choosing the rank capacity kmax at n = 2,000,000.
usage: python tools/probe_latlon.py N [kmax]"""
import json, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1709_04419_b200 as hm
from synthetic import latlon_dropout, standard_normal
n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 64
pts = latlon_dropout(n, 0)
th = (1.0, 0.1, 0.35)
for eps in (1e-6, 1e-8):
    t0 = time.perf_counter()
    try:
        H = hm.HMatrix(pts, th, eps=eps, leaf=64, eta=2.0, kmax=kmax)
    except hm.HMError as e:
        print(json.dumps({"n": n, "eps": eps, "kmax": kmax, "build": str(e)}), flush=True)
        continue
    t1 = time.perf_counter()
    rec = {"n": n, "eps": eps, "kmax": kmax, "build_s": t1 - t0}
    try:
        H.cholesky()
        Z = H.sample(standard_normal(n, 1, 3))
        out = H.loglik(Z)[0]
        rec.update(loglik=out.tolist(), quad_over_n=out[2] / n)
        t2 = time.perf_counter()
        H.assemble((1.0, 0.102, 0.35))
        H.cholesky()
        H.loglik(Z)
        rec["eval_s"] = time.perf_counter() - t2
        rec["timings_ms"] = H.timings()
    except hm.HMError as e:
        rec["error"] = str(e)
    rec["stats"] = H.stats()
    print(json.dumps(rec), flush=True)
    H.close()
