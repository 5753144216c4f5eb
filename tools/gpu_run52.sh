python paper_1709_04419_b200/build.py > /dev/null
for g in 148 222; do echo "GRID $g"; HM_EXEC_GRID=$g timeout 300 python tools/hm_trace_probe.py 64k 2>&1 | grep -A8 "makespan" | head -9; done
