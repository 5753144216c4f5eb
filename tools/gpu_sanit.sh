python paper_1709_04419_b200/build.py > /dev/null
timeout 60 python tools/hm_probe_small.py 600
timeout 600 compute-sanitizer --tool initcheck --print-limit 20 python tools/hm_probe_small.py 600 > gpurun_out/initcheck.txt 2>&1
head -60 gpurun_out/initcheck.txt
