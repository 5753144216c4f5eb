python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python tools/hm_probe_dual.py 12 2 2>&1 | tail -3
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --theta-streams 2 --no-profile 2>&1 | cut -c1-120
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --theta-streams 2 2>&1 | cut -c1-120
