set -x
python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python tools/hm_probe.py > gpurun_out/probe.txt 2>&1
cat gpurun_out/probe.txt | tail -40
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
cat gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.txt 2>&1
cat gpurun_out/bench.txt
