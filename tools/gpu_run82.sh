python paper_1709_04419_b200/build.py > /dev/null
for k in 64 96; do
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --kmax $k 2>&1 | cut -c1-110
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --kmax $k --theta-streams 1 2>&1 | cut -c1-110
done
timeout 1200 python tools/hm_probe_large.py 512 2>&1 | tail -3
