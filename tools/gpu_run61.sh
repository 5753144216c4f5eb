rm -rf paper_1709_04419_b200/build; python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python -m pytest tests/test_gpu_hmatrix.py -q -x 2>&1 | tail -2
timeout 300 python tools/hm_trace_probe.py 64k > gpurun_out/trace64k_rq.txt 2>&1; grep -A12 "makespan" gpurun_out/trace64k_rq.txt | head -13
grep -A8 "randomized truncation stages" gpurun_out/trace64k_rq.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n64k.txt 2>&1; cut -c1-250 gpurun_out/bench_n64k.txt
