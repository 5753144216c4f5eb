set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python paper_1709_04419_b200/build.py > /dev/null
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 600 python tools/hm_probe.py > gpurun_out/probe.txt 2>&1
cat gpurun_out/probe.txt | tail -20
