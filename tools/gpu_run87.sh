python paper_1709_04419_b200/build.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_n64k.txt 2>&1; cut -c1-150 gpurun_out/bench_n64k.txt
timeout 900 python bench.py --steps 5 --warmup 3 --theta-streams 1 --no-cpu-baseline > gpurun_out/bench_n64k_s1.txt 2>&1; cut -c1-150 gpurun_out/bench_n64k_s1.txt
timeout 900 python bench.py --workload mc --steps 1 --warmup 3 > gpurun_out/bench_mc.txt 2>&1; tail -1 gpurun_out/bench_mc.txt | cut -c1-150
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.txt 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_n64k.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 python bench.py --steps 1 --warmup 3 --theta-streams 1 --no-cpu-baseline > gpurun_out/bench_s1b.txt 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_exec_rq -s 1 -c 1 -o gpurun_out/prof_exec_n64k_v9 python bench.py --steps 1 --warmup 3 --theta-streams 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -1 gpurun_out/ncu_full.log
timeout 300 python tools/hm_trace_probe.py 64k 64 > gpurun_out/trace64k_rq.txt 2>&1; grep -A5 "makespan" gpurun_out/trace64k_rq.txt | head -6
timeout 300 python tools/hm_trace_rec.py > gpurun_out/trace_rec.txt 2>&1; grep "makespan\|assemble_ms" gpurun_out/trace_rec.txt
