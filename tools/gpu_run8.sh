python paper_1709_04419_b200/build.py > /dev/null
echo "== default grid"; timeout 120 python tools/hm_probe3.py 2000 1e-10
echo "== grid 1"; HM_EXEC_GRID=1 timeout 300 python tools/hm_probe3.py 2000 1e-10
echo "== grid 8"; HM_EXEC_GRID=8 timeout 300 python tools/hm_probe3.py 2000 1e-10
echo "== 8192 1e-8"; timeout 300 python tools/hm_probe3.py 8192 1e-8
