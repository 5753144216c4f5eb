for defs in "-DHM_TR_COOP_MAX=16" "-DHM_TR_COOP_MAX=16 -DHM_COOP_ROWFAC=2" "-DHM_TR_COOP_MAX=8"; do
rm -rf paper_1709_04419_b200/build; HM_BUILD_DEFS="$defs" python paper_1709_04419_b200/build.py > /dev/null
echo "DEFS=$defs"; timeout 600 python tools/hm_probe_dual.py 12 2 2>&1 | tail -3
done
echo "3 streams, COOP_MAX 8"; timeout 600 python tools/hm_probe_dual.py 12 3 2>&1 | tail -2
