set -x
for e in 1e-10 1e-8 1e-7; do timeout 120 python tools/hm_probe3.py 2000 $e 2>&1 | head -2; done
rm -rf paper_1709_04419_b200/build paper_1709_04419_b200/lib
HM_BUILD_DEFS="-DHM_COOP_WORK_LOG2=40" python paper_1709_04419_b200/build.py > /dev/null
for e in 1e-10 1e-8 1e-7; do timeout 120 python tools/hm_probe3.py 2000 $e 2>&1 | head -2; done
