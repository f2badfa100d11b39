# K2 ring-shape sweep on configs 2 and 3 (tuning build): device time of k_record + k_record_copy
for v in default; do
  echo "== $v"
  TM_LIB=paper_2508_11553_b200/libtmstore_tuning.so TM_RECORD_VARIANT=$v timeout 200 python tools/bench_paths.py --configs 2,3 --no-cpu 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    r=d['record']; print(d['config'], 'k2 %.4f copy %.4f frac %.3f' % (r['k1_k2_ms'], r['k2_copy_ms'], r['frac_of_peak']))
"
done
