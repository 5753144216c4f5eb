"""S co-scheduled handles (SMs split, one stream and host thread each) vs one handle."""
import sys, time, threading
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_1709_04419_b200 as hm
from synthetic import perturbed_mesh, standard_normal
pts = perturbed_mesh(256, 0.4, 2)
n = len(pts)
ths = [(1.0, 0.1 * (1 + 0.02 * ((i % 5) - 2)), 0.5 if i % 2 == 0 else 1.0) for i in range(24)]
Z = standard_normal(n, 1, 11)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2


def run(H, seq, out):
    for th in seq:
        H.assemble(th)
        H.cholesky()
        out.append(H.loglik(Z)[0, 0])


s0 = torch.cuda.Stream()
H = hm.HMatrix(pts, ths[0], eps=1e-7, leaf=64, eta=2.0, kmax=160, stream=s0.cuda_stream)
H.cholesky()
run(H, ths[:2], [])
torch.cuda.synchronize()
t0 = time.perf_counter()
out = []
run(H, ths[:steps], out)
torch.cuda.synchronize()
t1 = time.perf_counter()
print(f"single: {steps / (t1 - t0):.3f} evals/s", flush=True)
H.close()
streams = [torch.cuda.Stream() for _ in range(S)]
Hs = [hm.HMatrix(pts, ths[0], eps=1e-7, leaf=64, eta=2.0, kmax=160, stream=st.cuda_stream, coop_max=8) for st in streams]
caps = [148 // S + (1 if i < 148 % S else 0) for i in range(S)]
for Hx, c in zip(Hs, caps):
    Hx.set_exec_grid(c)
    Hx.cholesky()


def go(seqs):
    outs = [[] for _ in range(S)]
    th = [threading.Thread(target=run, args=(Hs[i], seqs[i], outs[i])) for i in range(S)]
    for t in th: t.start()
    for t in th: t.join()
    torch.cuda.synchronize()
    return outs


go([ths[:1]] * S)
t0 = time.perf_counter()
outs = go([ths[i:steps:S] for i in range(S)])
t1 = time.perf_counter()
flat = [v for o in outs for v in o]
print(f"{S} streams ({caps} CTAs): {len(flat) / (t1 - t0):.3f} evals/s", flush=True)
print("match", np.allclose(sorted(flat), sorted(out), rtol=1e-9), flush=True)
