python paper_1709_04419_b200/build.py > /dev/null
timeout 120 python tools/hm_probe3.py 2000 1e-10
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt; tail -8 gpurun_out/pytest_gpu.txt
timeout 600 python tools/hm_probe2.py > gpurun_out/probe2.txt 2>&1; cat gpurun_out/probe2.txt
