rm -rf paper_1709_04419_b200/build; HM_BUILD_DEFS="-DHM_EXEC_RQ_MINB=1" python paper_1709_04419_b200/build.py > /dev/null
timeout 300 python tools/hm_trace_probe.py 64k 2>&1 | grep -A8 "makespan" | head -9
timeout 300 python tools/hm_trace_rec.py 2>&1 | grep "makespan"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n64k.txt 2>&1; cut -c1-250 gpurun_out/bench_n64k.txt
timeout 300 python -m pytest tests/test_gpu_hmatrix.py -q -x 2>&1 | tail -2
