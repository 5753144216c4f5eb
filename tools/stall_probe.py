"""Find long stalls inside executor tasks (consecutive stage stamps > 500 us apart)
in an hm_trace of one phase and check whether the rest of the GPU kept working
during them.  usage: python tools/stall_probe.py plan.bin trace.bin [phase]"""
import sys

import numpy as np

sys.path.insert(0, "/root/repo/tests")
from plan_interp import Plan  # noqa: E402

P = Plan(sys.argv[1])
ph = getattr(P, sys.argv[3] if len(sys.argv) > 3 else "chol")
raw = np.fromfile(sys.argv[2], dtype=np.uint64)
n = len(ph.xt)
tr = raw[:4 * n].reshape(n, 4)
stg = raw[4 * n:].reshape(n, 64).astype(np.int64)
t0 = int(tr[:, 0].min())
end = (tr[:, 2].astype(np.int64) - t0) * 1e-3
cta = (tr[:, 3] >> 32).astype(np.int64)
smid = (tr[:, 3] & 0xffff).astype(np.int64)
kind = ph.xt["kind"]
stalls = []
for i in range(n):
    s = stg[i]
    s = s[(s > 0)]
    if s.size < 2:
        continue
    s = (s - t0) * 1e-3
    s = np.sort(s)
    d = np.diff(s)
    j = int(np.argmax(d))
    if d[j] > 500:
        stalls.append((i, int(kind[i]), int(cta[i]), int(smid[i]), s[j], s[j + 1], d[j]))
print(f"tasks with a stage gap > 500 us: {len(stalls)} of {n}")
gaps = np.array([x[6] for x in stalls]) if stalls else np.zeros(0)
if stalls:
    print(f"  gap us: min {gaps.min():.0f} median {np.median(gaps):.0f} max {gaps.max():.0f}")
for (i, k, c, sm, a, b, d) in stalls[:40]:
    inside = (end > a) & (end < b)
    others = inside & (cta != c)
    print(f"  task {i:7d} kind {k} cta {c:3d} sm {sm:3d} gap [{a:9.1f}, {b:9.1f}] {d:7.1f} us; "
          f"tasks finishing inside: {int(others.sum())} on {len(set(cta[others].tolist()))} other CTAs")
# clusters in time
if stalls:
    st = sorted(stalls, key=lambda x: x[4])
    print("  stall starts (us):", " ".join(f"{x[4]:.0f}" for x in st[:60]))
