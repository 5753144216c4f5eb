#!/bin/bash
# ncu evidence for the bench line (run under gpurun, one GPU, after bench.py exited 0 without ncu):
#  1. launch list of the bench command (cold, serialised: shares, not step times)
#  2. --set full capture of 12 k_exec_rq launches = one warm-up batch of 4 co-scheduled
#     evaluations x (recompression, H-Cholesky, solve), exported as raw CSV
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/ncu_launches.csv $B > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
timeout 3000 ncu --set full --clock-control none --import-source on -k regex:k_exec_rq -s 3 -c 12 \
  -o gpurun_out/kexec_full $B > gpurun_out/ncu_full.log 2>&1
echo "full capture rc=$?"
ncu -i gpurun_out/kexec_full.ncu-rep --page raw --csv > gpurun_out/kexec_full_raw.csv 2>/dev/null
ls -la gpurun_out/kexec_full.ncu-rep
rm -f gpurun_out/kexec_full.ncu-rep   # ~190 MB: over the 64 MiB gpurun_out merge limit
