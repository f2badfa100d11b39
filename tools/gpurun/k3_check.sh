#!/bin/bash
# K3 export on configs 1-3 (device time), and the export / NDJSON GPU tests
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -k "export or ndjson or trajectory or manager or fullsize or golden or config" > gpurun_out/k3_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/k3_tests.log
for r in 1 2; do
  timeout 300 python tools/bench_paths.py --configs 1,2,3 --no-cpu --reps 5 2>/dev/null | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    x = d['export']; print(d['config'], 'k3 %.4f ms frac %.3f' % (x['k3_ms'], x['frac_of_peak']), 'record %.4f' % d['record']['device_ms'])
" >> gpurun_out/k3.txt
done
