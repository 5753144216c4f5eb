# throughput vs co-scheduled executors S and cooperative group sizing (diagnostic)
run() { timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline "$@" 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('value %.3f latency_ms %.1f e2e %.3f par %s'%(d['value'], d['latency']['ms_per_eval'], d['e2e']['value'], d['config']['parallelism'][-60:]))
"; }
for S in 2 3 4 6; do echo "S=$S"; run --theta-streams $S; done
rm -rf paper_1709_04419_b200/build; HM_BUILD_DEFS="-DHM_COOP_WORK_LOG2=16" python paper_1709_04419_b200/build.py > /dev/null
echo "LOG2=16 S=4"; run --theta-streams 4
echo "LOG2=16 S=2"; run --theta-streams 2
rm -rf paper_1709_04419_b200/build; python paper_1709_04419_b200/build.py > /dev/null
