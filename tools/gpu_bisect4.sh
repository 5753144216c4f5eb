rm -rf paper_1709_04419_b200/build paper_1709_04419_b200/lib
HM_BUILD_DEFS="-DHM_OLDLAYOUT=1" python paper_1709_04419_b200/build.py > /dev/null
timeout 120 python tools/hm_probe3.py 2000 1e-8 2>&1
