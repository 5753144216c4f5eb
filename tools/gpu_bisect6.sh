for v in 0 15; do
rm -rf paper_1709_04419_b200/build paper_1709_04419_b200/lib
HM_BUILD_DEFS="-DHM_OLDLAYOUT=$v -DHM_POISON_RING" python paper_1709_04419_b200/build.py > /dev/null
echo "variant $v poisoned"; timeout 120 python tools/hm_probe3.py 2000 1e-8 2>&1 | head -2
done
