set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
./tools/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
cat gpurun_out/fp64_peak.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
