python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python tools/hm_probe10.py
