for defs in "-DHM_COOP_WORK_LOG2=17" "-DHM_COOP_WORK_LOG2=18" "-DHM_COOP_WORK_LOG2=19" "-DHM_COOP_WORK_LOG2=18 -DHM_TR_NB=3" "-DHM_COOP_WORK_LOG2=20"; do
rm -rf paper_1709_04419_b200/build; HM_BUILD_DEFS="$defs" python paper_1709_04419_b200/build.py > /dev/null
echo "DEFS=$defs"
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('value %.3f latency_ms %.1f e2e %.3f kexec_share %.3f'%(d['value'], d['latency']['ms_per_eval'], d['e2e']['value'], d['kernels']['k_exec']['share']))
"
done
