python paper_1709_04419_b200/build.py > /dev/null
for S in 5 6; do timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --theta-streams $S 2>&1 | cut -c1-110; done
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --kmax 48 2>&1 | cut -c1-110
