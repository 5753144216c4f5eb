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
    # configs[4]: 2,000,000 lat/lon locations (jittered 0.0067 deg grid, 30 % dropout), ell in degrees;
    # Z drawn by the H sampler at eps 1e-8, likelihood at eps 1e-6; one evaluation at a time (S = 1).
    # Rank capacities: the n = 262,144 probe had max ranks 18 (1e-6) and 28 (1e-8); at 2M the
    # 1e-8 assembly needs more than 48 (measured HM_ERR_RANK_CAP at kmax 32 and 48): with an
    # absolute eps the blocks' singular values grow with their point counts (sqrt(m q)).
    "n2m": dict(n=2_000_000, kind="latlon", thetas=[(1.0, 0.1, 0.35)], leaf=64, eta=2.0, eps=1e-6, cfg="configs[4]",
                eps_sample=1e-8, kmax=48, kmax_sample=64, adaptive=True),
}


def make_points(w, seed=2):
    from synthetic import latlon_dropout, perturbed_mesh, uniform_iid
    if w["kind"] == "mesh":
        return perturbed_mesh(w["sqrt_n"], w["delta"], seed)
    if w["kind"] == "latlon":
        return latlon_dropout(w["n"], seed)
    return uniform_iid(w["n"], seed)


def workload_str(w, args):
    """The configuration both arms name in their JSON line (config.workload)."""
    if w["cfg"] == "configs[3]":
        return f"{w['cfg']}: MC-MLE, n={w['n']}, {w['evals']} Nelder-Mead evals per replicate, eps={w['eps']}"
    extra = f", Z by the H sampler at eps={w['eps_sample']}" if "eps_sample" in w else ""
    return (f"{w['cfg']}: n={w['n']} {w['kind']}, theta={w['thetas']} (ell swept +-2%), leaf={w['leaf']}, "
            f"eta={w['eta']}, eps={w['eps']}, kmax={w.get('kmax', args.kmax)}{extra}")


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


def rank_thetas(w, steps, S, rank, world):
    """The thetas rank `rank` evaluates: every rank walks its own slice of one global
    schedule (round-robin, steps * S each; independent evaluations, no collective)."""
    return theta_schedule(w, steps * world * S)[rank::world]


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
def oracle_sample(w, th):
    """One oracle evaluation (dense Eq. 1, CPU fp64, oracle/ as it stands) on a bounded
    sub-sample of n_s workload points, timed in its two parts: the dense covariance
    (O(n^2) K_nu evaluations) and the Cholesky + solve (O(n^3)).  Returns
    (seconds assembly, seconds factorisation, n_s)."""
    from oracle import dense as od
    from synthetic import standard_normal
    n_s = min(int(os.environ.get("HM_REF_SAMPLE_N", "3000")), w["n"])
    pts = make_points(w)
    rng = np.random.default_rng(5)
    sub = pts[np.sort(rng.choice(w["n"], size=n_s, replace=False))]
    Z = standard_normal(n_s, 1, 7)[:, 0]
    t0 = time.perf_counter()
    C = od.covariance(sub, th, bessel="scipy")
    t1 = time.perf_counter()
    od.loglik_from_cov(C, Z)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1, n_s


def extrapolate(ta, tc, n_s, n):
    """Seconds of one oracle evaluation at the workload's n: assembly scaled by (n/n_s)^2,
    factorisation + solve by (n/n_s)^3 (the dense algorithm's own complexities)."""
    return ta * (n / n_s) ** 2 + tc * (n / n_s) ** 3


def run_reference(args, w):
    ws, rk, lr = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        if rk != 0:
            dist.barrier()
            dist.destroy_process_group()
            return
    ths = theta_schedule(w, args.warmup + args.steps)
    for s in range(args.warmup):
        oracle_sample(w, ths[s])
    ta = tc = 0.0
    t0 = time.perf_counter()
    for s in range(args.steps):
        a, c, n_s = oracle_sample(w, ths[args.warmup + s])
        ta += a
        tc += c
    wall = (time.perf_counter() - t0) / args.steps
    ta, tc = ta / args.steps, tc / args.steps
    t_n = extrapolate(ta, tc, n_s, w["n"])
    value = 1.0 / t_n
    cores = len(os.sched_getaffinity(0))
    line = {"metric": f"H-log-likelihood evals/sec at n={w['n']}", "value": value, "unit": "evals/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": workload_str(w, args), "oracle_sample_n": n_s,
                       "step": f"one dense oracle evaluation at n_s={n_s} points of the workload "
                               f"(measured {1e3 * wall:.0f} ms = ms_per_step)",
                       "extrapolation": f"value = 1 / (t_asm (n/n_s)^2 + t_chol (n/n_s)^3) with t_asm = {ta:.3f} s, "
                                        f"t_chol = {tc:.3f} s measured at n_s: {t_n:.0f} s per evaluation at "
                                        f"n = {w['n']} (not run: {8 * w['n'] ** 2 / 1e9:.0f} GB dense matrix)"},
            "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": "oracle",
                             "sample": f"dense Eq.(1) oracle at n_s={n_s}, assembly scaled by (n/n_s)^2, "
                                       f"Cholesky + solve by (n/n_s)^3"},
            "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "paper_cpu_context": paper_context(w)}
    print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def cpu_baseline(w, budget_s=20.0):
    """The oracle (dense Eq. 1, CPU fp64) on a bounded sample, extrapolated to the
    workload's n with the dense algorithm's own complexities (see extrapolate)."""
    th = w["thetas"][0]
    oracle_sample(w, th)                     # warm (imports, scipy)
    t0 = time.perf_counter()
    ta = tc = 0.0
    reps = 0
    while True:
        a, c, n_s = oracle_sample(w, th)
        ta += a
        tc += c
        reps += 1
        if time.perf_counter() - t0 > budget_s / 2 or reps >= 5:
            break
    ta, tc = ta / reps, tc / reps
    return {"value": 1.0 / extrapolate(ta, tc, n_s, w["n"]), "unit": "evals/s", "cores": len(os.sched_getaffinity(0)),
            "kind": "oracle",
            "sample": f"{reps} dense Eq.(1) oracle evals at n_s={n_s} sub-sampled from the workload "
                      f"(assembly {ta:.2f} s, Cholesky + solve {tc:.2f} s each), extrapolated to n={w['n']} "
                      f"by (n/n_s)^2 and (n/n_s)^3"}


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
    reps = args.replicates or ws * args.steps * S
    # warm-up replicates (untimed), then `reps` replicates over all ranks, timed; each rank
    # fits its replicates S at a time (lockstep Nelder-Mead, one hm_loglik_multi per round)
    mc_mle(w["n"], ws * S, w["thetas"][0], w["start"], eps=w["eps"], evals=w["evals"], leaf=w["leaf"],
           rank=rk, world=ws, device=lr, seed=10_000, gather=False, streams=S, sms=sms, kmax=args.kmax)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(lr) as clk:
        e0.record(stream)
        res = mc_mle(w["n"], reps, w["thetas"][0], w["start"], eps=w["eps"], evals=w["evals"],
                     leaf=w["leaf"], rank=rk, world=ws, device=lr, seed=0, gather=False, streams=S, sms=sms,
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
        n_evals = reps * w["evals"]
        line = {"metric": f"H-log-likelihood evals/sec (MC-MLE, n={w['n']})", "value": n_evals / (ms / 1e3),
                "unit": "evals/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_str(w, args),
                           "replicates": reps,
                           "step": f"{S} replicate(s) per rank (incl. their H-build and sampler)",
                           "parallelism": f"replicas x{ws}; {S} co-scheduled replicates per GPU"},
                "estimates_rank0": res.tolist(), "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def paper_context(w):
    """PAPER.md Table 3 (l.483-500): HLIBpro on 40 cores (Dell workstation, 20
    processors, 128 GB, l.210), eps = 1e-5 for C~ and L~, theta = (0.98, 0.64, 0.325)
    on soil-moisture locations -- context, not a target (other machine, other data)."""
    rows = {64000: (5.3, 5.1), 2000000: (227.0, 471.0), 128000: (13.2, 13.7), 32000: (3.2, 2.3)}
    n = min(rows, key=lambda r: abs(r - w["n"]))
    c, l = rows[n]
    return {"source": "PAPER.md Table 3 (l.494-500)", "n": n, "C_build_s": c, "cholesky_s": l,
            "evals_per_s_equiv": 1.0 / (c + l), "cores": 40,
            "hardware": "Dell workstation, 20 processors (40 cores), 128 GB RAM (PAPER.md l.210)",
            "eps": 1e-5, "theta": [0.98, 0.64, 0.325]}


def traffic_of(kernel_key, workload):
    """DRAM bytes per launch of the dominant kernel from the committed ncu --set full
    summary (profiles/traffic.json, written from the capture), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None, None
    d = json.load(open(p))
    e = d.get(workload, {}).get(kernel_key)
    if not e:
        return None, None
    return e["dram_bytes_per_launch"], e["source"]


def run_gpu(args, w):
    """configs[2]-style throughput through the C-ABI's batched entry point: each rank
    evaluates its own theta sequence with hm_loglik_batch, S thetas per call; inside
    the library S executors (the handle + S - 1 siblings on the same tree and plan)
    run the evaluations co-scheduled on the GPU, each persistent executor capped at
    1/S of the SMs (include/hmlik.h).  A step = one hm_loglik_batch call = S complete,
    independent likelihood evaluations (assemble + H-Cholesky + solve each).  The
    single-evaluation latency (S = 1) is measured in the same run."""
    import torch
    ws, rk, lr = dist_env()
    torch.cuda.set_device(lr)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    import paper_1709_04419_b200 as hm
    from paper_1709_04419_b200.dist import gather_results
    from synthetic import standard_normal

    S = max(1, args.theta_streams) if "eps_sample" not in w else 1   # 2M: one handle fills the GPU
    sms = torch.cuda.get_device_properties(lr).multi_processor_count
    # cooperative groups <= 8 CTAs when co-scheduled, and within the deadlock bound
    # 4 * (coop - 1) < executor CTAs = sms / S
    coop = 16 if S == 1 else max(1, min(8, (sms // S - 1) // 4 + 1))
    if args.coop_max > 0:
        coop = min(args.coop_max, (sms // S - 1) // 4 + 1)
    kmax = w.get("kmax", args.kmax)
    pts = make_points(w)
    n = pts.shape[0]
    steps, warm = args.steps, args.warmup
    mine = rank_thetas(w, warm + steps, S, rk, ws)   # this rank's thetas, S per step
    xi = standard_normal(n, 1, 11)
    t_build = time.perf_counter()
    if "eps_sample" in w:
        # configs[4]: Z = L~ xi by the H sampler at its own accuracy, on its own
        # handle, freed before the likelihood handle is built (device memory)
        Hs = hm.HMatrix(pts, w["thetas"][0], eps=w["eps_sample"], leaf=w["leaf"], eta=w["eta"],
                        kmax=w["kmax_sample"], device=lr, coop_max=coop, adaptive_cap=w.get("adaptive", False))
        Hs.cholesky()
        Zh = np.ascontiguousarray(Hs.sample(xi)[:, 0])
        sampler_stats = Hs.stats()
        Hs.close()
        H = hm.HMatrix(pts, mine[0], eps=w["eps"], leaf=w["leaf"], eta=w["eta"], kmax=kmax, device=lr,
                       coop_max=coop, adaptive_cap=w.get("adaptive", False))
    else:
        sampler_stats = None
        H = hm.HMatrix(pts, mine[0], eps=w["eps"], leaf=w["leaf"], eta=w["eta"], kmax=kmax, device=lr,
                       coop_max=coop)
        H.cholesky()
        Zh = np.ascontiguousarray(H.sample(xi)[:, 0])
    t_build = time.perf_counter() - t_build
    Zd = torch.from_numpy(Zh).to(f"cuda:{lr}")
    H.set_batch_streams(S)
    torch.cuda.synchronize()

    def batch(s, Z):
        out, rc = H.loglik_batch(mine[s * S:(s + 1) * S], Z)
        hm._binding.check(rc)
        return out

    for s in range(warm):
        batch(s, Zd)
    if not args.no_profile:
        H.profile(True)

    def timed(Z, first, count):
        outs = []
        cur = torch.cuda.current_stream()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for s in range(first, first + count):
            outs.append(batch(s, Z))      # synchronous: returns when its S evaluations are done
        e1.record(cur)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        return e0.elapsed_time(e1), outs

    with ClockSampler(lr) as clk:
        ms, outs = timed(Zd, warm, steps)
    kstats = H.kernel_stats()
    H.profile(False)
    launches = int(sum(v["launches"] for v in kstats.values()))
    # end-to-end through the C-ABI with HOST data: every evaluation copies Z h2d and
    # its (loglik, logdet, quad) triple d2h
    ms_e2e, _ = timed(Zh, warm, steps)
    # single-evaluation latency (one executor on the whole GPU, same plan)
    H.set_batch_streams(1)
    lat_n = (min(steps, 2) if "eps_sample" in w else min(steps, 6)) * S
    lat_ms, _ = timed(Zd, warm, lat_n // S)
    H.set_batch_streams(S)
    res = np.concatenate([o.reshape(-1, 3) for o in outs])       # this rank's (loglik, logdet, quad)
    allres = gather_results(res, len(res) * ws, rk, ws, device=f"cuda:{lr}") if dist else res
    if dist:
        t = torch.tensor([ms, ms_e2e, lat_ms], device=f"cuda:{lr}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_e2e, lat_ms = t.tolist()
    st = H.stats()
    if rk == 0:
        ev = ws * steps * S
        value = ev / (ms / 1e3)
        peaks = load_peaks()
        roof = roofline(kstats, peaks, w)
        if roof is not None:
            roof["concurrent_launches"] = S
            roof["aggregate_achieved"] = (kstats["k_exec"]["flops"] / 1e12) / (ms / 1e3) if "k_exec" in kstats else None
        line = {"metric": f"H-log-likelihood evals/sec at n={n}", "value": value, "unit": "evals/s",
                "n_gpus": ws, "steps": steps, "warmup": warm, "ms_per_step": ms / steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_str(w, args),
                           "l2": "no flush: H-matrix storage > 126 MB L2",
                           "parallelism": f"replicas x{ws}; hm_loglik_batch with {S} co-scheduled executors per GPU "
                                          f"(persistent executor CTAs {sms // S} each, coop_max {coop})",
                           "evals_per_step_per_gpu": S, "evals_timed_total": ev,
                           "max_rank_C": st["max_rank_C"], "max_rank_L": st["max_rank_L"],
                           "bytes_L_MB": round(st["bytes_L"] / 2**20, 1), "kmax": kmax,
                           "adaptive_cap": bool(w.get("adaptive", False)),
                           "setup_s": round(t_build, 1),
                           "sampler": None if sampler_stats is None else
                           {"eps": w["eps_sample"], "kmax": w["kmax_sample"], "max_rank_L": sampler_stats["max_rank_L"]}},
                "latency": {"ms_per_eval": lat_ms / lat_n, "evals_per_s": lat_n / (lat_ms / 1e3),
                            "how": f"{lat_n} evaluations one at a time (hm_set_batch_streams 1), whole GPU"},
                "e2e": {"value": ev / (ms_e2e / 1e3), "unit": "evals/s", "h2d_bytes_per_step": 8 * n * S,
                        "d2h_bytes_per_step": 24 * S},
                "gpu_launches": launches,
                "roofline": roof,
                "kernels": {k: {"launches_per_step": v["launches"] / steps, "ms_per_step": v["ms"] / steps,
                                "share": v["ms"] / max(1e-9, sum(x["ms"] for x in kstats.values()))}
                            for k, v in kstats.items()},
                "results": {"gathered": int(allres.shape[0]), "loglik_first": allres[0].tolist(),
                            "finite": bool(np.isfinite(allres).all())},
                "paper_cpu_context": paper_context(w),
                "clocks": clk.summary()}
        if not args.no_cpu_baseline and ws == 1:
            line["cpu_baseline"] = cpu_baseline(w)
        print(json.dumps(line), flush=True)
    H.close()
    if dist:
        dist.destroy_process_group()


def roofline(kstats, peaks, w):
    """Dominant kernel (largest device time in the timed region) against its bound."""
    if not kstats:
        return None
    name, v = max(kstats.items(), key=lambda kv: kv[1]["ms"])
    if v["ms"] <= 0.0:
        return None
    key = name
    if name == "k_exec":   # the family's kernel in the default execution mode (ready queues)
        name = "k_exec_rq (persistent executor: recompression, H-Cholesky, solve launches averaged)"
    traffic, tsrc = traffic_of(key, w["cfg"])
    per_launch_s = v["ms"] / 1e3 / max(1, v["launches"])
    flops = v["flops"] / max(1, v["launches"])
    byts = v["bytes"] / max(1, v["launches"])
    t_f = flops / (peaks["fp64_tflops"] * 1e12)
    t_b = byts / (peaks["hbm_gbs"] * 1e9)
    if t_f >= t_b:
        ach = flops / per_launch_s / 1e12
        return {"kernel": name, "bound": "fp64", "achieved": ach, "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                "frac": ach / peaks["fp64_tflops"], "traffic": traffic, "traffic_src": tsrc,
                "algorithmic_flops_per_launch": flops,
                "algorithmic_bytes_per_launch": byts, "peak_src": peaks["fp64_src"]}
    ach = byts / per_launch_s / 1e9
    return {"kernel": name, "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": ach / peaks["hbm_gbs"], "traffic": traffic, "traffic_src": tsrc,
            "algorithmic_flops_per_launch": flops,
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
    ap.add_argument("--replicates", type=int, default=0,
                    help="--workload mc: replicates in the timed region (0 = gpus * steps * theta-streams; "
                         "configs[3] is 128)")
    ap.add_argument("--coop-max", type=int, default=0,
                    help="cap of cooperative truncation groups (0 = 16 at S = 1, else min(8, deadlock bound))")
    ap.add_argument("--theta-streams", type=int, default=4,
                    help="independent theta evaluations co-scheduled per GPU (1 = single-evaluation latency)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    w = WORKLOADS[args.workload]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch this command under torchrun (the driver launches
        # it that way itself; this makes `bench.py --gpus N` do the same)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", os.environ.get("MASTER_PORT", "29517"),
               os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={os.environ['WORLD_SIZE']} but --gpus {args.gpus}")
    if args.impl == "reference":
        run_reference(args, w)
    elif args.workload == "mc":
        run_mc(args, w)
    else:
        run_gpu(args, w)


if __name__ == "__main__":
    main()
