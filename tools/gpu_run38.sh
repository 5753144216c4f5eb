python paper_1709_04419_b200/build.py > /dev/null
echo REL; timeout 600 python tools/hm_probe7.py
echo ABS; HM_EPS_ABS=1 timeout 600 python tools/hm_probe7.py
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
