python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python tools/hm_probe4.py 11
timeout 600 python tools/hm_trace_probe.py 64k > gpurun_out/trace64k.txt 2>&1; cat gpurun_out/trace64k.txt | head -40
