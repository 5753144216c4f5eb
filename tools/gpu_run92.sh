for defs in "-DHM_COOP_ROWFAC=2" "-DHM_COOP_ROWFAC=8"; do
rm -rf paper_1709_04419_b200/build; HM_BUILD_DEFS="$defs" python paper_1709_04419_b200/build.py > /dev/null
echo "DEFS=$defs"
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline 2>&1 | cut -c1-110
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --theta-streams 1 2>&1 | cut -c1-110
done
