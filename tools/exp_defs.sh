#!/bin/bash
# Sweep compile-time tuning defines: for each argument (a quoted HM_BUILD_DEFS string,
# "" = defaults) rebuild in place and run a short bench (S = 4 throughput and S = 1 latency).
#   bash tools/exp_defs.sh "" "-DHM_COOP_ROWFAC=2" "-DHM_TR_EXACT_K=64"
cd "$(dirname "$0")/.." || exit 1
for defs in "$@"; do
  HM_BUILD_DEFS="$defs" python paper_1709_04419_b200/build.py > /dev/null || { echo "build failed: $defs"; continue; }
  timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print('%-40s value %.3f latency_ms %.1f e2e %.3f' % (sys.argv[1] or 'defaults', d['value'], d['latency']['ms_per_eval'], d['e2e']['value']))
" "$defs"
done
HM_BUILD_DEFS="" python paper_1709_04419_b200/build.py > /dev/null
