python paper_1709_04419_b200/build.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 600 python bench.py --workload mc --steps 1 --warmup 1 2>&1 | tail -2 | cut -c1-600
