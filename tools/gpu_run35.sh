python paper_1709_04419_b200/build.py > /dev/null
echo STOP4; timeout 600 python tools/hm_probe6.py
rm -rf paper_1709_04419_b200/build paper_1709_04419_b200/lib
HM_BUILD_DEFS="-DHM_TR_STOP=0.5" python paper_1709_04419_b200/build.py > /dev/null
echo STOP0.5; timeout 600 python tools/hm_probe6.py
