# exact-path truncations: Jacobi staged in shared memory (now) and the width limit TR_EXACT_K (diagnostic)
run() { timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline "$@" 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('value %.3f latency_ms %.1f e2e %.3f'%(d['value'], d['latency']['ms_per_eval'], d['e2e']['value']))
"; }
for ek in 160 64 96; do
  rm -rf paper_1709_04419_b200/build; HM_BUILD_DEFS="-DHM_TR_EXACT_K=$ek" python paper_1709_04419_b200/build.py > /dev/null
  echo "TR_EXACT_K=$ek S=4"; run
  echo "TR_EXACT_K=$ek S=1"; run --theta-streams 1
done
rm -rf paper_1709_04419_b200/build; python paper_1709_04419_b200/build.py > /dev/null
