set -x
python paper_1709_04419_b200/build.py > /dev/null
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30
timeout 600 python tools/hm_probe.py 2>&1 | tail -20
