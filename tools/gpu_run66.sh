python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python tools/hm_trace_rec.py 2>&1 | grep -B1 -A6 "makespan"
