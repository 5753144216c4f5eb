cd bisect_old && timeout 120 python tools/hm_probe3.py 2000 1e-8 2>&1 | head -3; cd ..
python paper_1709_04419_b200/build.py >/dev/null; timeout 120 python tools/hm_probe3.py 2000 1e-8 2>&1 | head -3
