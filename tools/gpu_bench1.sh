python paper_1709_04419_b200/build.py > /dev/null
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_n64k.txt 2>&1; tail -3 gpurun_out/bench_n64k.txt
timeout 300 python bench.py --workload n2k --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2k.txt 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_n2k.csv python bench.py --workload n2k --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
tail -3 gpurun_out/ncu_launch.log
