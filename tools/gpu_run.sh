#!/bin/bash
# One gpurun call: build in place, then run the steps named on the command line.
#   tools/gpu_run.sh tests | bench | mesh | cfg1 | ncu | "python ..."
# usage: /usr/local/graft/bin/gpurun --timeout 3600 -- 'bash tools/gpu_run.sh tests mesh cfg1'
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail gpurun_out/build.log; exit 1; }
for step in "$@"; do
  echo "=== $step $(date +%T)"
  case "$step" in
    tests) timeout 2400 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; tail -15 gpurun_out/pytest_gpu.log ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3 ;;
    bench) timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 1500 gpurun_out/bench.json ;;
    mesh) timeout 1500 python tools/mesh64k_table.py > gpurun_out/mesh.log 2>&1; tail -5 gpurun_out/mesh.log ;;
    cfg1) timeout 3000 python tools/config1_table.py > gpurun_out/cfg1.log 2>&1; tail -3 gpurun_out/cfg1.log | cut -c1-400 ;;
    *) timeout 3000 bash -c "$step" 2>&1 | tail -20 ;;
  esac
done
echo "=== done $(date +%T)"
