python paper_1709_04419_b200/build.py > /dev/null
timeout 900 python tools/hm_probe8.py
