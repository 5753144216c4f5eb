#!/usr/bin/env python
"""bench.py -- H-matrix Gaussian log-likelihood evaluations per second on B200.

Metric (BASELINE.json): "H-log-likelihood evals/sec at n=64k & 2M".  One STEP
is one full likelihood evaluation of PAPER.md Eq. (4) for a new theta on a
fixed location set -- the unit of work of the paper's MLE loop (sec. 3.1):

    hm_assemble(theta)   Matern blocks (device K_nu) + ACA + QR/SVD recompression
    hm_cholesky()        H-Cholesky with truncated low-rank updates
    hm_loglik(Z)         forward solve L~ v = Z, log det = 2 sum log L~_ii, Eq. (4)

Default workload = BASELINE configs[2]: n = 65,536 = 256 x 256 jittered grid
(Eq. 3, delta = 0.4), Matern sigma^2 = 1, ell = 0.1, nu alternating
0.5 / 1.0 (closed-form and general-nu Bessel paths), leaf 64, eta = 2,
eps = 1e-7, fp64.  Z is drawn once by the library's own H-sampler (Z = L~ xi,
PAPER.md l.308) at the first theta.  The H-matrix storage of C~/L~ (hundreds
of MB) exceeds the 126 MB L2, so no explicit flush is needed between steps.

Multi-GPU (torchrun, one rank per GPU): the evaluations are independent
(different theta points of the MLE search), so each rank evaluates its own
theta sequence on its own GPU -- weak scaling, no data-path collective; the
per-rank log-likelihoods are gathered once after the timed region.

--impl reference times the CPU fp64 oracle (dense Eq. 1; oracle/) on a
bounded sample of the same workload (a smaller n, scaled to evals/sec at the
workload's n by the O(n^3) dense cost) -- there is no upstream code to run.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (n, builder, thetas, leaf, eta, eps)
    "n64k": dict(n=65536, kind="mesh", sqrt_n=256, delta=0.4, thetas=[(1.0, 0.1, 0.5), (1.0, 0.1, 1.0)],
                 leaf=64, eta=2.0, eps=1e-7, cfg="configs[2]"),
    "n16k": dict(n=16384, kind="uniform", thetas=[(1.0, 0.2, 1.5)], leaf=32, eta=2.0, eps=1e-8, cfg="configs[1]"),
    "n2k": dict(n=2000, kind="uniform", thetas=[(1.0, 0.0864, 0.5)], leaf=32, eta=2.0, eps=1e-8, cfg="configs[0]"),
    # configs[3]: Monte-Carlo MLE, replicates of n = 16,384 uniform points, theta* = (1, 0.0334, 0.5),
    # 60 Nelder-Mead evaluations each; a "step" = one replicate per rank (bench.py --workload mc)
    "mc": dict(n=16384, kind="uniform", thetas=[(1.0, 0.0334, 0.5)], leaf=32, eta=2.0, eps=1e-6, cfg="configs[3]",
               evals=60, start=(0.8, 0.05, 0.7)),
}


def make_points(w, seed=2):
    from synthetic import perturbed_mesh, uniform_iid
    if w["kind"] == "mesh":
        return perturbed_mesh(w["sqrt_n"], w["delta"], seed)
    return uniform_iid(w["n"], seed)


def workload_str(w, args):
    """The configuration both arms name in their JSON line (config.workload)."""
    if w["cfg"] == "configs[3]":
        return f"{w['cfg']}: MC-MLE, n={w['n']}, {w['evals']} Nelder-Mead evals per replicate, eps={w['eps']}"
    return (f"{w['cfg']}: n={w['n']} {w['kind']}, theta={w['thetas']} (ell swept +-2%), leaf={w['leaf']}, "
            f"eta={w['eta']}, eps={w['eps']}, kmax={args.kmax}")


def theta_schedule(w, steps):
    """Per-step theta: alternate the workload's nu values, sweep ell by +-2 %
    (a Nelder-Mead-like walk around the truth; every step is a new theta)."""
    out = []
    base = w["thetas"]
    for s in range(steps):
        s2, ell, nu = base[s % len(base)]
        f = 1.0 + 0.02 * math.sin(0.7 * (s + 1))
        out.append((s2, ell * f, nu))
    return out


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for nm, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = {"hbm_gbs": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)"}
    if os.path.exists(p):
        d = json.load(open(p))
        peaks["hbm_gbs"] = float(d.get("hbm_gbs", 6650.0))
        peaks["hbm_src"] = "measured (MEASURED_PEAKS.json)"
    # FP64 peak: own DMMA/DFMA microbenchmark on this pool (tools/fp64_peak.cu,
    # profiles/r01_fp64_peak.txt); MEASURED_PEAKS.json carries no fp64 figure.
    peaks["fp64_tflops"] = 37.2
    peaks["fp64_src"] = "measured (tools/fp64_peak.cu, profiles/r01_fp64_peak.txt)"
    return peaks


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rk = int(os.environ.get("RANK", "0"))
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rk, lr


# ---------------------------------------------------------------------------- reference (oracle) arm
def run_reference(args, w):
    ws, rk, lr = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        if rk != 0:
            dist.barrier()
            dist.destroy_process_group()
            return
    from oracle import dense as od
    from synthetic import standard_normal, uniform_iid
    # bounded sample: dense Eq. (1) at n_s points of the workload's distribution,
    # scaled to the workload's n by the dense O(n^3) cost (the oracle is dense).
    n_s = min(int(os.environ.get("HM_REF_SAMPLE_N", "3000")), w["n"])
    pts = make_points(w)
    rng = np.random.default_rng(5)
    sub = pts[np.sort(rng.choice(w["n"], size=n_s, replace=False))]
    Z = standard_normal(n_s, 1, 7)[:, 0]
    ths = theta_schedule(w, args.warmup + args.steps)
    for s in range(args.warmup):
        od.loglik(sub, Z, ths[s], bessel="scipy")
    t0 = time.perf_counter()
    for s in range(args.steps):
        od.loglik(sub, Z, ths[args.warmup + s], bessel="scipy")
    dt = (time.perf_counter() - t0) / args.steps
    scale = (n_s / w["n"]) ** 3
    value = scale / dt
    cores = len(os.sched_getaffinity(0))
    line = {"metric": f"H-log-likelihood evals/sec at n={w['n']}", "value": value, "unit": "evals/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": workload_str(w, args), "oracle_sample_n": n_s},
            "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": "oracle",
                             "sample": f"dense Eq.(1) oracle at n={n_s} ({dt:.2f} s/eval), scaled by (n_s/n)^3"},
            "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def cpu_baseline(w, budget_s=20.0):
    """Oracle (dense Eq. 1, CPU fp64) timed on a bounded sample; evals/s scaled to n."""
    from oracle import dense as od
    from synthetic import standard_normal
    pts = make_points(w)
    n_s = min(int(os.environ.get("HM_REF_SAMPLE_N", "3000")), w["n"])
    rng = np.random.default_rng(5)
    sub = pts[np.sort(rng.choice(w["n"], size=n_s, replace=False))]
    Z = standard_normal(n_s, 1, 7)[:, 0]
    th = w["thetas"][0]
    t0 = time.perf_counter()
    reps = 0
    while True:
        od.loglik(sub, Z, th, bessel="scipy")
        reps += 1
        if time.perf_counter() - t0 > budget_s / 2 or reps >= 5:
            break
    dt = (time.perf_counter() - t0) / reps
    return {"value": (n_s / w["n"]) ** 3 / dt, "unit": "evals/s", "cores": len(os.sched_getaffinity(0)),
            "kind": "oracle",
            "sample": f"{reps} dense Eq.(1) oracle evals at n={n_s} sub-sampled from the workload "
                      f"({dt:.2f} s each), scaled to n={w['n']} by (n_s/n)^3"}


# ---------------------------------------------------------------------------- GPU arm
def run_mc(args, w):
    """configs[3]: each rank fits its own replicates (60 Nelder-Mead evaluations each,
    paper_1709_04419_b200.mle); value = likelihood evaluations per second, whole job."""
    import torch
    ws, rk, lr = dist_env()
    torch.cuda.set_device(lr)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    from paper_1709_04419_b200.mle import mc_mle
    S = max(1, args.theta_streams)
    sms = torch.cuda.get_device_properties(lr).multi_processor_count
    strs = [torch.cuda.Stream(device=lr) for _ in range(S)] if S > 1 else None
    handles = [x.cuda_stream for x in strs] if strs else None
    # warm-up replicates (untimed), then args.steps * S replicates per rank, timed (S co-scheduled)
    mc_mle(w["n"], ws * S, w["thetas"][0], w["start"], eps=w["eps"], evals=w["evals"], leaf=w["leaf"],
           rank=rk, world=ws, device=lr, seed=10_000, gather=False, streams=handles, sms=sms, kmax=args.kmax)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(lr) as clk:
        e0.record(stream)
        res = mc_mle(w["n"], ws * args.steps * S, w["thetas"][0], w["start"], eps=w["eps"], evals=w["evals"],
                     leaf=w["leaf"], rank=rk, world=ws, device=lr, seed=0, gather=False, streams=handles, sms=sms,
                     kmax=args.kmax)
        torch.cuda.synchronize()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device=f"cuda:{lr}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rk == 0:
        n_evals = ws * args.steps * S * w["evals"]
        line = {"metric": f"H-log-likelihood evals/sec (MC-MLE, n={w['n']})", "value": n_evals / (ms / 1e3),
                "unit": "evals/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_str(w, args),
                           "step": f"{S} replicate(s) per rank (incl. their H-build and sampler)",
                           "parallelism": f"replicas x{ws}; {S} co-scheduled replicates per GPU"},
                "estimates_rank0": res.tolist(), "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_gpu(args, w):
    """configs[2]-style throughput: each rank evaluates its own theta sequence.  On one
    GPU, S handles (same locations, own factor storage) run side by side, each on its
    own CUDA stream and host thread with 1/S of the SMs for its persistent executor
    (hm_set_exec_grid): a step is S complete, independent likelihood evaluations
    (assemble + H-Cholesky + solve each).  --theta-streams 1 is the single-evaluation
    latency configuration."""
    import threading
    import torch
    ws, rk, lr = dist_env()
    torch.cuda.set_device(lr)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    import paper_1709_04419_b200 as hm
    from synthetic import standard_normal

    S = max(1, args.theta_streams)
    sms = torch.cuda.get_device_properties(lr).multi_processor_count
    caps = [sms // S + (1 if i < sms % S else 0) for i in range(S)] if S > 1 else [0]
    # cooperative groups <= 8 CTAs when co-scheduled, and within the deadlock bound
    # 4 * (coop - 1) < executor CTAs (hm_set_exec_grid)
    coop = 16 if S == 1 else max(1, min(8, (min(caps) - 1) // 4 + 1))
    pts = make_points(w)
    n = pts.shape[0]
    steps, warm = args.steps, args.warmup
    # each (rank, stream) walks its own theta sequence (independent evaluations)
    ths_all = theta_schedule(w, (warm + steps) * ws * S)
    seqs = [ths_all[rk * S + i::ws * S] for i in range(S)]
    streams = [torch.cuda.Stream(device=lr) for _ in range(S)]
    Hs = []
    for i in range(S):
        H = hm.HMatrix(pts, seqs[i][0], eps=w["eps"], leaf=w["leaf"], eta=w["eta"], kmax=args.kmax, device=lr,
                       stream=streams[i].cuda_stream, coop_max=coop)
        H.set_exec_grid(caps[i])
        Hs.append(H)
    Hs[0].cholesky()
    xi = standard_normal(n, 1, 11)
    Zh = np.asfortranarray(Hs[0].sample(xi))
    Zd = torch.from_numpy(np.ascontiguousarray(Zh[:, 0])).to(f"cuda:{lr}")
    torch.cuda.synchronize()

    def step(H, th, Z):
        H.assemble(th)
        H.cholesky()
        return H.loglik(Z)

    def run_all(first, count, Z, outs):
        def worker(i):
            for s_ in range(first, first + count):
                outs[i].append(step(Hs[i], seqs[i][s_], Z)[0].copy())
        th = [threading.Thread(target=worker, args=(i,)) for i in range(S)]
        for t in th:
            t.start()
        for t in th:
            t.join()

    run_all(0, warm, Zd, [[] for _ in range(S)])
    if not args.no_profile:
        for H in Hs:
            H.profile(True)

    def timed(Z):
        outs = [[] for _ in range(S)]
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(streams[0])
        run_all(warm, steps, Z, outs)
        e1 = []
        for st in streams:
            e = torch.cuda.Event(enable_timing=True)
            e.record(st)
            e1.append(e)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        return max(e0.elapsed_time(e) for e in e1), outs

    with ClockSampler(lr) as clk:
        ms, outs = timed(Zd)
    kst = [H.kernel_stats() for H in Hs]
    for H in Hs:
        H.profile(False)
    kstats = {}
    for k in kst[0]:
        kstats[k] = {f: sum(x[k][f] for x in kst) for f in kst[0][k]}
    launches = int(sum(v["launches"] for v in kstats.values()))
    # end-to-end through the C-ABI with HOST buffers: per evaluation the host Z goes
    # h2d and the (loglik, logdet, quad) triple comes back d2h
    Zp = torch.from_numpy(np.ascontiguousarray(Zh[:, 0])).pin_memory()   # pinned host input
    ms_e2e, _ = timed(Zp)
    if dist:
        t = torch.tensor([ms, ms_e2e], device=f"cuda:{lr}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_e2e = t.tolist()
    st = Hs[0].stats()
    if rk == 0:
        ev = ws * steps * S
        value = ev / (ms / 1e3)
        peaks = load_peaks()
        roof = roofline(kstats, peaks)
        if roof is not None:
            roof["concurrent_launches"] = S
            roof["aggregate_achieved"] = (kstats["k_exec"]["flops"] / 1e12) / (ms / 1e3) if "k_exec" in kstats else None
        line = {"metric": f"H-log-likelihood evals/sec at n={n}", "value": value, "unit": "evals/s",
                "n_gpus": ws, "steps": steps, "warmup": warm, "ms_per_step": ms / steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_str(w, args),
                           "l2": "no flush: H-matrix storage > 126 MB L2",
                           "parallelism": f"replicas x{ws}; {S} co-scheduled theta streams per GPU "
                                          f"(executor CTAs {caps if S > 1 else sms}, coop_max {coop}); "
                                          f"a step = {S} independent evaluations per GPU",
                           "evals_per_step": ev,
                           "max_rank_C": st["max_rank_C"], "max_rank_L": st["max_rank_L"],
                           "bytes_L_MB": round(st["bytes_L"] / 2**20, 1)},
                "e2e": {"value": ev / (ms_e2e / 1e3), "unit": "evals/s", "h2d_bytes_per_step": 8 * n * S,
                        "d2h_bytes_per_step": 24 * S},
                "gpu_launches": launches,
                "roofline": roof,
                "kernels": {k: {"launches_per_step": v["launches"] / steps, "ms_per_step": v["ms"] / steps,
                                "share": v["ms"] / max(1e-9, sum(x["ms"] for x in kstats.values()))}
                            for k, v in kstats.items()},
                "loglik_first": outs[0][0].tolist(),
                "clocks": clk.summary()}
        if not args.no_cpu_baseline and ws == 1:
            line["cpu_baseline"] = cpu_baseline(w)
        print(json.dumps(line), flush=True)
    for H in Hs:
        H.close()
    if dist:
        dist.destroy_process_group()


def roofline(kstats, peaks):
    """Dominant kernel (largest device time in the timed region) against its bound."""
    if not kstats:
        return None
    name, v = max(kstats.items(), key=lambda kv: kv[1]["ms"])
    if v["ms"] <= 0.0:
        return None
    if name == "k_exec":   # the family's kernel in the default execution mode (ready queues)
        name = "k_exec_rq (persistent executor: recompression, H-Cholesky, solve launches averaged)"
    per_launch_s = v["ms"] / 1e3 / max(1, v["launches"])
    flops = v["flops"] / max(1, v["launches"])
    byts = v["bytes"] / max(1, v["launches"])
    t_f = flops / (peaks["fp64_tflops"] * 1e12)
    t_b = byts / (peaks["hbm_gbs"] * 1e9)
    if t_f >= t_b:
        ach = flops / per_launch_s / 1e12
        return {"kernel": name, "bound": "fp64", "achieved": ach, "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                "frac": ach / peaks["fp64_tflops"], "traffic": None, "algorithmic_flops_per_launch": flops,
                "algorithmic_bytes_per_launch": byts, "peak_src": peaks["fp64_src"]}
    ach = byts / per_launch_s / 1e9
    return {"kernel": name, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": ach / peaks["hbm_gbs"], "traffic": None, "algorithmic_flops_per_launch": flops,
            "algorithmic_bytes_per_launch": byts, "peak_src": peaks["hbm_src"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hm", choices=["hm", "reference"])
    ap.add_argument("--workload", default="n64k", choices=sorted(WORKLOADS))
    ap.add_argument("--kmax", type=int, default=64,
                    help="rank capacity per low-rank block (ranks at the workloads' eps stay <= 30; HM_ERR_RANK_CAP if exceeded)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true", help="no per-launch CUDA events (kernel table empty)")
    ap.add_argument("--theta-streams", type=int, default=4,
                    help="independent theta evaluations co-scheduled per GPU (1 = single-evaluation latency)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, w)
    elif args.workload == "mc":
        run_mc(args, w)
    else:
        run_gpu(args, w)


if __name__ == "__main__":
    main()
