for defs in "-DHM_COOP_ROWFAC=2" "-DHM_COOP_ROWFAC=3"; do
rm -rf paper_1709_04419_b200/build; HM_BUILD_DEFS="$defs" python paper_1709_04419_b200/build.py > /dev/null
echo "DEFS=$defs"; timeout 300 python tools/hm_trace_probe.py 64k 2>&1 | grep -A4 "makespan" | head -5
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | cut -c1-150
done
