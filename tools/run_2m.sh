#!/bin/bash
# configs[4] bench line (n = 2,000,000 lat/lon, Z by the H sampler at 1e-8, likelihood at 1e-6)
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
free -g | head -2 > gpurun_out/n2m_host.txt; nproc >> gpurun_out/n2m_host.txt
( while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/n2m_mem.txt; sleep 10; done ) &
MP=$!
HM_PLAN_VERBOSE=1 timeout 5400 python bench.py --workload n2m --steps 3 --warmup 3 > gpurun_out/bench_n2m.json 2> gpurun_out/bench_n2m.err
echo "rc=$?"
kill $MP
tail -c 3000 gpurun_out/bench_n2m.json; tail -5 gpurun_out/bench_n2m.err
