python paper_1709_04419_b200/build.py > /dev/null
timeout 120 python tools/hm_probe3.py 2000 1e-10
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt; tail -8 gpurun_out/pytest_gpu.txt
timeout 600 python tools/hm_probe4.py 011 
timeout 600 python tools/hm_trace_probe.py 64k > gpurun_out/trace64k.txt 2>&1; cat gpurun_out/trace64k.txt
