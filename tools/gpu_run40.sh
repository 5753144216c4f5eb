python paper_1709_04419_b200/build.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -6
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_n64k.txt 2>&1; head -c 700 gpurun_out/bench_n64k.txt
