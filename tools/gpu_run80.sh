python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline 2>&1 | cut -c1-110
timeout 900 python bench.py --workload mc --steps 1 --warmup 3 --theta-streams 1 2>&1 | tail -1 | cut -c1-200
timeout 900 python bench.py --workload mc --steps 1 --warmup 3 2>&1 | tail -1 | cut -c1-200
timeout 600 python -m pytest tests/test_gpu_hmatrix.py -q -x -k "mc_mle or cosched" 2>&1 | tail -2
