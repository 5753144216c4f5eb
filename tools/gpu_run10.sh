python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python tools/hm_probe4.py 00111
HM_EXEC_GRID=148 timeout 300 python tools/hm_probe4.py 11
timeout 600 python tools/hm_trace_probe.py 8k > gpurun_out/trace8k.txt 2>&1; cat gpurun_out/trace8k.txt
timeout 600 python tools/hm_trace_probe.py 64k > gpurun_out/trace64k.txt 2>&1; cat gpurun_out/trace64k.txt
