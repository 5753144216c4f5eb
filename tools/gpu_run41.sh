python paper_1709_04419_b200/build.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30
timeout 900 python tools/hm_probe8.py 2>&1 | tail -50
