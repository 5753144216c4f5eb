python paper_1709_04419_b200/build.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python tools/hm_trace_rec.py 2>&1 | grep -A5 "phase=solve"
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_n64k.txt 2>&1; cut -c1-250 gpurun_out/bench_n64k.txt
