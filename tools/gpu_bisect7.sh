rm -rf paper_1709_04419_b200/build paper_1709_04419_b200/lib
HM_BUILD_DEFS="-DHM_POISON_RING" python paper_1709_04419_b200/build.py > /dev/null
echo "poisoned"; timeout 120 python tools/hm_probe3.py 2000 1e-8 2>&1 | head -2; timeout 120 python tools/hm_probe3.py 2000 1e-7 2>&1 | head -2
rm -rf paper_1709_04419_b200/build paper_1709_04419_b200/lib
python paper_1709_04419_b200/build.py > /dev/null
echo "normal"; timeout 120 python tools/hm_probe3.py 2000 1e-8 2>&1 | head -2; timeout 120 python tools/hm_probe3.py 2000 1e-7 2>&1 | head -2
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
