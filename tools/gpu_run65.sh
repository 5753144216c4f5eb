python paper_1709_04419_b200/build.py > /dev/null
timeout 300 python tools/hm_trace_probe.py 64k > gpurun_out/trace64k_rq.txt 2>&1; grep -A10 "makespan" gpurun_out/trace64k_rq.txt | head -11
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | cut -c1-200
