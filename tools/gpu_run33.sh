python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python tools/hm_trace_probe.py 64k > gpurun_out/trace64k.txt 2>&1; grep -B2 -A22 "makespan" gpurun_out/trace64k.txt | head -30
rm -rf paper_1709_04419_b200/build paper_1709_04419_b200/lib
HM_BUILD_DEFS="-DHM_COOP_ROWFAC=4" python paper_1709_04419_b200/build.py > /dev/null
echo "ROWFAC=4"; timeout 600 python tools/hm_trace_probe.py 64k 2>&1 | grep -A14 "makespan"
