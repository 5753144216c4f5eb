python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python tools/hm_probe9.py 2>&1 | tail -8
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_n64k.txt 2>&1; cut -c1-1500 gpurun_out/bench_n64k.txt
timeout 600 python tools/hm_trace_probe.py 64k > gpurun_out/trace64k.txt 2>&1; grep -A24 "makespan" gpurun_out/trace64k.txt | head -30
