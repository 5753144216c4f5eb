# split truncations on/off: throughput (S=4), single-evaluation latency (diagnostic)
run() { timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline "$@" 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('value %.3f latency_ms %.1f e2e %.3f rank_L %s'%(d['value'], d['latency']['ms_per_eval'], d['e2e']['value'], d['config']['max_rank_L']))
"; }
echo "split on"; run
echo "split off"; HM_TRUNC_SPLIT=0 run
echo "split on S=1"; run --theta-streams 1
echo "split off S=1"; HM_TRUNC_SPLIT=0 run --theta-streams 1
