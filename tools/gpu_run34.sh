python paper_1709_04419_b200/build.py > /dev/null
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x 2>&1 | tail -30
