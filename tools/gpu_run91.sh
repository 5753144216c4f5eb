python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python -m pytest tests/test_gpu_hmatrix.py -q -x -k "relative or parameters or validation" 2>&1 | tail -3
