# throughput vs co-scheduled executors S x cooperative group cap (diagnostic):
#   bash tools/exp_streams2.sh "4 6" "4 4" "6 4" ...   (pairs "S coop_max")
run() { timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline "$@" 2>gpurun_out/sweep.err | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('value %.3f latency_ms %.1f e2e %.3f par %s'%(d['value'], d['latency']['ms_per_eval'], d['e2e']['value'], d['config']['parallelism'][-70:]))
"; tail -2 gpurun_out/sweep.err; }
for p in "$@"; do set -- $p; echo "S=$1 coop=$2"; run --theta-streams $1 --coop-max $2; done
