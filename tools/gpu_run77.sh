python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python -m pytest tests/test_gpu_hmatrix.py -q -x -k "cosched or exec_modes" 2>&1 | tail -3
