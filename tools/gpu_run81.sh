python paper_1709_04419_b200/build.py > /dev/null
timeout 1200 python tools/hm_probe_large.py 512 2>&1 | tail -5
