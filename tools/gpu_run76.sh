python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --theta-streams 4 2>&1 | cut -c1-120
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_n64k.txt 2>&1; cut -c1-200 gpurun_out/bench_n64k.txt
