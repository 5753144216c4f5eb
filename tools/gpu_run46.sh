python paper_1709_04419_b200/build.py > /dev/null
timeout 300 python -m pytest tests/test_gpu_hmatrix.py -q -x -k "exec_modes or config0 or repeat or general" 2>&1 | tail -3
timeout 300 python tools/hm_probe4.py 1122 2>&1 | tail -4
timeout 300 python tools/hm_trace_probe.py 64k > gpurun_out/trace64k_rq.txt 2>&1; grep -A20 "makespan" gpurun_out/trace64k_rq.txt | head -22
