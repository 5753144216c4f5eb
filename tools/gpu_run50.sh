python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python tools/hm_trace_rec.py 2>&1 | tail -60
