"""Analyse a persistent-executor trace (hm_trace) of one phase against its plan.

usage (on the GPU box, see tools/hm_trace_probe.py): writes a text summary:
makespan, per-kind busy time, utilisation, dependency-wait time, the critical
path through the dependency DAG with measured task durations, and the longest
tasks.
"""
from __future__ import annotations

import sys

import numpy as np

sys.path.insert(0, "/root/repo/tests")
from plan_interp import Plan  # noqa: E402


def analyse(plan_path: str, trace_path: str, phase: str = "chol", grid: int = 296, top: int = 15) -> str:
    P = Plan(plan_path)
    ph = getattr(P, phase)
    raw = np.fromfile(trace_path, dtype=np.uint64)
    n = len(ph.xt)
    assert raw.size == 68 * n, (raw.size, n)
    tr = raw[:4 * n].reshape(n, 4)
    stg = raw[4 * n:].reshape(n, 64)
    t0 = tr[:, 0].min()
    claim = (tr[:, 0] - t0).astype(np.float64) * 1e-3   # us
    ready = (tr[:, 1] - t0).astype(np.float64) * 1e-3
    end = (tr[:, 2] - t0).astype(np.float64) * 1e-3
    kind = ph.xt["kind"]
    dur = end - ready
    wait = ready - claim
    mk = end.max()
    lines = [f"phase={phase} tasks={n} makespan={mk / 1e3:.3f} ms grid={grid}"]
    for k, nm in ((0, "vm"), (1, "trunc")):
        sel = kind == k
        lines.append(f"  {nm:6s} n={sel.sum():8d} busy={dur[sel].sum() / 1e3:10.3f} ms  mean={dur[sel].mean() if sel.any() else 0:8.2f} us"
                     f"  max={dur[sel].max() if sel.any() else 0:9.1f} us  dep-wait={wait[sel].sum() / 1e3:9.3f} ms")
    lines.append(f"  utilisation (busy / (makespan * grid)) = {dur.sum() / (mk * grid):.3f}")
    # truncation busy time by class (m, q, nsub) and by actual stacked width
    tsel = np.nonzero(kind == 1)[0]
    if tsel.size:
        cls = {}
        for i in tsel:
            t = ph.tt[ph.xt[i]["idx"]]
            key = (int(t["m"]), int(t["q"]), int(ph.xt[i]["nsub"]), "exact" if int(t["kmax_tot"]) <= 160 and int(t["m"]) <= 512 and int(t["q"]) <= 512 else "rand")
            c = cls.setdefault(key, [0, 0.0]); c[0] += 1; c[1] += dur[i]
        lines.append("  truncation busy by (m, q, nsub, path): CTA-tasks, CTA-ms")
        for k, (c, d) in sorted(cls.items(), key=lambda kv: -kv[1][1])[:12]:
            lines.append(f"    {str(k):32s} {c:7d} {d / 1e3:10.1f}")
    # critical path with measured durations
    cp = np.zeros(n)
    arg = np.full(n, -1)
    for i in range(n):
        x = ph.xt[i]
        d = ph.xdeps[x["dep_begin"]: x["dep_begin"] + x["dep_count"]]
        if d.size:
            j = d[np.argmax(cp[d])]
            cp[i] = cp[j] + dur[i]
            arg[i] = j
        else:
            cp[i] = dur[i]
    i = int(np.argmax(cp))
    path = []
    while i >= 0:
        path.append(i)
        i = int(arg[i])
    path.reverse()
    pk = kind[path]
    lines.append(f"  critical path: {cp.max() / 1e3:.3f} ms over {len(path)} tasks "
                 f"(vm {int((pk == 0).sum())}: {dur[path][pk == 0].sum() / 1e3:.3f} ms, "
                 f"trunc {int((pk == 1).sum())}: {dur[path][pk == 1].sum() / 1e3:.3f} ms)")
    # composition of the critical path
    comp = {}
    for i in path:
        x = ph.xt[i]
        if x["kind"] == 1:
            t = ph.tt[x["idx"]]
            key = f"trunc m={t['m']} q={t['q']} nsub={x['nsub']}"
        else:
            v = ph.vt[x["idx"]]
            ops = ph.ins["op"][v["ins_begin"]: v["ins_begin"] + v["ins_count"]]
            names = {1: "LD", 2: "ST", 3: "GEMM", 4: "POTRF", 5: "TRSM", 6: "TRSMLN", 7: "TRMM", 8: "ZERO", 9: "MG",
                     10: "TRTRI", 11: "ADD"}
            sig = []
            for o in ops:
                nm = names.get(int(o), str(int(o)))
                if not sig or sig[-1][0] != nm:
                    sig.append([nm, 1])
                else:
                    sig[-1][1] += 1
            key = "vm " + " ".join(f"{a}{'x' + str(b) if b > 1 else ''}" for a, b in sig)
        c = comp.setdefault(key, [0, 0.0])
        c[0] += 1
        c[1] += dur[i]
    # single-instruction MGEMM_ST tasks on the critical path by number of terms
    hist = {}
    for i in path:
        x = ph.xt[i]
        if x["kind"] != 0:
            continue
        v = ph.vt[x["idx"]]
        insv = ph.ins[v["ins_begin"]: v["ins_begin"] + v["ins_count"]]
        if len(insv) == 1 and int(insv["op"][0]) == 12:
            nt = int(insv["t1"][0])
            b = 1 if nt <= 1 else 2 if nt <= 2 else 4 if nt <= 4 else 8 if nt <= 8 else 16 if nt <= 16 else 64 if nt <= 64 else 999
            h = hist.setdefault(b, [0, 0.0, 0])
            h[0] += 1
            h[1] += dur[i]
            h[2] += nt
    # stage stamps of single-instruction MGEMM_ST tasks on the critical path (ns since claim)
    sel = []
    for i in path:
        x = ph.xt[i]
        if x["kind"] == 0:
            v = ph.vt[x["idx"]]
            if v["ins_count"] == 1 and int(ph.ins["op"][v["ins_begin"]]) == 12 and stg[i, 5] > 0:
                sel.append(i)
    if sel:
        sel = np.array(sel)
        c0 = tr[sel, 0].astype(np.float64)
        st = [(stg[sel, k].astype(np.float64) - c0).mean() * 1e-3 for k in range(6)]
        lines.append("  CP MGEMM_ST stage stamps (us after claim): start %.2f ins %.2f terms %.2f compute %.2f store %.2f"
                     " completion %.2f end %.2f (n=%d)" % (*st, (tr[sel, 2].astype(np.float64) - c0).mean() * 1e-3, len(sel)))
        one = sel[[int(ph.ins["t1"][ph.vt[ph.xt[i]["idx"]]["ins_begin"]]) == 1 for i in sel]]
        if one.size:
            c0 = tr[one, 0].astype(np.float64)
            st = [(stg[one, k].astype(np.float64) - c0).mean() * 1e-3 for k in range(6)]
            lines.append("    1-term only:                                start %.2f ins %.2f terms %.2f compute %.2f store %.2f"
                         " completion %.2f (n=%d)" % (*st, len(one)))
        # the gap between a CP task's end and its CP successor's claim (queue latency)
        pos = {int(j): k for k, j in enumerate(path)}
        gaps = [claim[path[k + 1]] - end[path[k]] for k in range(len(path) - 1)]
        lines.append("  CP hand-over gap (claim of next - end of previous), us: mean %.2f median %.2f total %.1f ms"
                     % (np.mean(gaps), np.median(gaps), np.sum(np.maximum(gaps, 0)) / 1e3))
        cta = (tr[:, 3] >> 32).astype(np.int64)
        same = np.array([cta[path[k + 1]] == cta[path[k]] for k in range(len(path) - 1)])
        g = np.array(gaps)
        lines.append("    same CTA (continuation): %d of %d, gap total %.1f ms; other CTA: gap mean %.2f us, total %.1f ms,"
                     " >20us: %d (total %.1f ms)" % (same.sum(), len(same), np.sum(np.maximum(g[same], 0)) / 1e3,
                                                     g[~same].mean() if (~same).any() else 0,
                                                     np.sum(np.maximum(g[~same], 0)) / 1e3, (g[~same] > 20).sum(),
                                                     np.sum(g[~same][g[~same] > 20]) / 1e3))
        big = [k for k in range(len(path) - 1) if gaps[k] > 20]
        kinds = {}
        for k in big:
            key = ("trunc" if kind[path[k]] == 1 else "vm") + "->" + ("trunc" if kind[path[k + 1]] == 1 else "vm")
            a = kinds.setdefault(key, [0, 0.0]); a[0] += 1; a[1] += gaps[k]
        lines.append("    gaps > 20 us by (prev -> next) kind: " + ", ".join(f"{k}: {v[0]} / {v[1] / 1e3:.1f} ms" for k, v in kinds.items()))
        # how busy was the machine when those CP tasks waited: tasks running at the ready instant
        st_ = np.sort(claim); en_ = np.sort(end)
        busy = [int(np.searchsorted(st_, end[path[k]]) - np.searchsorted(en_, end[path[k]])) for k in big[:2000]]
        if busy:
            lines.append("    running tasks when a >20 us-gap CP task became ready: mean %.0f, min %d, max %d (grid %d)"
                         % (np.mean(busy), np.min(busy), np.max(busy), grid))
    lines.append("  critical-path MGEMM_ST tasks by terms (<=b: count, ms, mean us, mean terms):")
    for b in sorted(hist):
        c, d, nt = hist[b]
        lines.append(f"    <= {b:4d}: {c:6d} {d / 1e3:9.3f} {d / c:8.1f} {nt / c:7.1f}")
    lines.append("  critical-path composition (count, ms):")
    for k, (cnt, d) in sorted(comp.items(), key=lambda kv: -kv[1][1])[:14]:
        lines.append(f"    {k:40s} {cnt:6d} {d / 1e3:9.3f}")
    # stage breakdown of the randomized truncations (leader stamps)
    tsel = np.nonzero((kind == 1) & (stg[:, 0] > 0))[0]
    if tsel.size:
        lines.append("  randomized truncation stages (leader), us: [start->sync1, sync1->sync2, ...]")
        mid = np.array([i for i in tsel if ph.tt[ph.xt[i]["idx"]]["m"] <= 512], dtype=np.int64)
        pick = list(tsel[np.argsort(-dur[tsel])][:3]) + (list(mid[np.argsort(-dur[mid])][:6]) if mid.size else [])
        for i in pick:
            st = stg[i].copy()
            Kc, ellc = int(st[62]), int(st[63])
            st[62] = st[63] = 0
            k = int(np.max(np.nonzero(st)[0]))
            d = np.diff(st[:k + 1].astype(np.float64)) * 1e-3
            x = ph.xt[i]; t = ph.tt[x["idx"]]
            lines.append(f"    m={t['m']} q={t['q']} nsub={x['nsub']} K={Kc} ell={ellc} total={dur[i]:.0f}: " + " ".join(f"{v:.0f}" for v in d))
    order = np.argsort(-dur)[:top]
    lines.append("  longest tasks:")
    for i in order:
        x = ph.xt[i]
        if x["kind"] == 1:
            t = ph.tt[x["idx"]]
            desc = f"trunc m={t['m']} q={t['q']} cap={t['cap']} Kstat={t['kmax_tot']} pieces={t['piece_count']}"
        else:
            v = ph.vt[x["idx"]]
            desc = f"vm ins={v['ins_count']}"
        lines.append(f"    #{i:7d} {dur[i]:10.1f} us  on_cp={i in set(path)}  {desc}")
    return "\n".join(lines)


if __name__ == "__main__":
    print(analyse(*sys.argv[1:3], phase=sys.argv[3] if len(sys.argv) > 3 else "chol"))
