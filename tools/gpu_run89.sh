python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python -m pytest tests/test_gpu_hmatrix.py -q -x 2>&1 | tail -1
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline 2>&1 | cut -c1-110
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --theta-streams 1 2>&1 | cut -c1-110
