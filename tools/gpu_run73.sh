python paper_1709_04419_b200/build.py > /dev/null
for S in 1 2 3 4; do timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --theta-streams $S 2>&1 | cut -c1-120; done
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
