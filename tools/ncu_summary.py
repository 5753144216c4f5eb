"""Summarise tools/ncu_profile.sh output (gpurun_out/) into profiles/ (committed evidence).

usage: python tools/ncu_summary.py TAG WORKLOAD_CFG
  TAG           file-name tag, e.g. r02_v1
  WORKLOAD_CFG  BASELINE config the bench line names (bench.py WORKLOADS[..]["cfg"]),
                e.g. configs[2] -- key of profiles/traffic.json, which bench.py reads
writes profiles/TAG_ncu_launches.txt, profiles/TAG_ncu_full_kexecrq.txt and updates
profiles/traffic.json with the DRAM bytes per k_exec_rq launch of the full capture.
"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches(tag):
    path = os.path.join(OUT, "ncu_launches.csv")
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0].split("<")[0].strip()
        v = float(r[iv].replace(",", ""))
        unit = r[iu]
        ms = v / 1e6 if unit == "ns" else v / 1e3 if unit in ("us", "usecond") else v if unit in ("ms", "msecond") else v
        tot[name][0] += 1
        tot[name][1] += ms
    allms = sum(v[1] for v in tot.values())
    lines = ["ncu --metrics gpu__time_duration.sum --clock-control none -c 600: python bench.py --steps 2 --warmup 3 "
             "--no-cpu-baseline (n64k, kmax 64, hm_loglik_batch with 4 co-scheduled executors)",
             "(ncu serialises the co-scheduled launches and replays cold: shares, not step times; k_exec_rq runs "
             "3 phases per evaluation: recompression, H-Cholesky, solve)"]
    for k, (n, ms) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:30s} launches={n:6d} total_ms={ms:11.3f} share={ms / allms:.4f}")
    open(os.path.join(PROF, f"{tag}_ncu_launches.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__registers_per_thread",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]


def to_bytes(v, unit):
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit)
    return v * f if f else v


def full(tag, cfg):
    path = os.path.join(OUT, "kexec_full_raw.csv")
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    lines = [f"ncu --set full --clock-control none --import-source on -k regex:k_exec_rq -s 3 -c 12: python bench.py "
             f"--steps 2 --warmup 3 --no-cpu-baseline ({cfg}: the first warm-up hm_loglik_batch call = 4 co-scheduled "
             f"evaluations x (recompression, H-Cholesky, solve), each executor capped at 37 CTAs; per launch)"]
    phases = {"recompression": [], "cholesky": [], "solve": []}
    for r in data:
        d = {}
        for m in WANT:
            if m in hdr:
                i = hdr.index(m)
                try:
                    d[m] = (float(r[i].replace(",", "")), units[i])
                except ValueError:
                    pass
        ms = d["gpu__time_duration.sum"][0]
        # the three phases of one evaluation differ by an order of magnitude in duration
        ph = "cholesky" if ms > 300 else "recompression" if ms > 50 else "solve"
        rb = to_bytes(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else float("nan")
        wb = to_bytes(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else float("nan")
        if rb == rb and wb == wb:
            phases[ph].append(rb + wb)
        lines.append(f"launch {r[hdr.index('ID')]} ({ph}): " +
                     ", ".join(f"{m}={v:g} {u}" for m, (v, u) in d.items()))
    per = {k: sum(v) / len(v) for k, v in phases.items() if v}
    # one evaluation = one launch of each phase: per-launch average as bench.py's roofline counts it
    avg = sum(per.values()) / len(per)
    lines.append("DRAM bytes (read + write) per launch by phase (launches with the metric): " +
                 ", ".join(f"{k} {v:.4g} ({len(phases[k])})" for k, v in per.items()))
    lines.append(f"per k_exec_rq launch, averaged over the three phases of an evaluation: {avg:.4g}")
    out = os.path.join(PROF, f"{tag}_ncu_full_kexecrq.txt")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    tj = os.path.join(PROF, "traffic.json")
    t = json.load(open(tj)) if os.path.exists(tj) else {}
    t.setdefault(cfg, {})["k_exec"] = {"dram_bytes_per_launch": avg, "by_phase": per,
                                       "source": os.path.relpath(out, ROOT)}
    json.dump(t, open(tj, "w"), indent=1)


if __name__ == "__main__":
    tag, cfg = sys.argv[1], sys.argv[2]
    launches(tag)
    full(tag, cfg)
