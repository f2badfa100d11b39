# one GPU: routed walk at N=1 with the TMA-staged int32 compare vs the register path
set -x
timeout 300 python -m pytest tests/test_routing_gpu.py -q -x -k world1 > gpurun_out/l_tests.log 2>&1; tail -2 gpurun_out/l_tests.log
for mode in tma regs tma; do
  TM_ROUTED_LOCAL=$mode timeout 300 python bench.py --workload c5 --steps 20 > gpurun_out/l_c5_$mode.json 2> gpurun_out/l_c5_$mode.err
  tail -1 gpurun_out/l_c5_$mode.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$mode', round(d['value']/1e6,2),'Mq/s', round(d['ms_per_step'],4), 'walk', round(d['routed_walk_ms_avg_rank0'],4), d['phase_ms_avg_rank0'])"
done
echo done
