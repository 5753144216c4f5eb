python paper_1709_04419_b200/build.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_n64k.txt 2>&1; cut -c1-150 gpurun_out/bench_n64k.txt
timeout 300 python tools/hm_trace_probe.py 64k 64 > gpurun_out/trace64k_rq.txt 2>&1; grep -A30 "makespan" gpurun_out/trace64k_rq.txt | head -31
