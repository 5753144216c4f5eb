rm -rf paper_1709_04419_b200/build; HM_BUILD_DEFS="-DHM_TR_COOP_MAX=16" python paper_1709_04419_b200/build.py > /dev/null
timeout 600 python tools/hm_probe_dual.py 8 74
