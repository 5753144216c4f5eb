rm -rf paper_1709_04419_b200/build; python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_n64k.txt 2>&1; cut -c1-150 gpurun_out/bench_n64k.txt
timeout 900 python bench.py --steps 5 --warmup 3 --theta-streams 1 --no-cpu-baseline > gpurun_out/bench_n64k_s1.txt 2>&1; cut -c1-150 gpurun_out/bench_n64k_s1.txt
