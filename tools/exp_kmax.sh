# rank capacity kmax (static plan: widths, cooperative group sizes, memory) vs throughput (diagnostic)
run() { timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline "$@" 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('value %.3f latency_ms %.1f e2e %.3f rankL %s'%(d['value'], d['latency']['ms_per_eval'], d['e2e']['value'], d['config']['max_rank_L']))
"; }
for k in 32 48 64; do echo "kmax=$k"; run --kmax $k; done
