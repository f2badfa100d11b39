#!/bin/bash
# K2 on config 3 (device time over reps), twice
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for r in 1 2; do
  timeout 300 python tools/bench_paths.py --configs 3 --no-cpu --reps 5 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    r = d['record']; print(d['config'], 'device %.4f ms frac %.3f' % (r['device_ms'], r['frac_of_peak']), 'export %.4f' % d['export']['k3_ms'])
" >> gpurun_out/k2_c3.txt
done
