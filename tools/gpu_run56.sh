python paper_1709_04419_b200/build.py > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "Error|error|assert|FAILED|^E " | head -30
