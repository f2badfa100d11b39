python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for cfg in "--sessions 10000" "--sessions 40000 --mixed 1024,131072"; do
for mode in "100000000 0" "512 0" "512 1"; do set -- $mode
TM_PLAN_MIN=$1 TM_PLAN_ROOTS=$2 python bench.py $cfg --steps 100 --no-cpu --e2e-steps 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$cfg', 'plan_min=$1 roots=$2', round(d['value']/1e6,3), 'Mq/s', round(d['ms_per_step']*1e3,1), 'us/step walk', round(r['kernel_ms_avg']*1e3,1), 'us plan', round(r['planner_ms_avg']*1e3,1), round(r['achieved']), round(r['frac'],3))"
done; done
