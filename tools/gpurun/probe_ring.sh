# 2-GPU box: routed walk remote-ring variants at N=2 (TM_ROUTED_RING; 0 = 4 x 1024 default)
set -x
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29516"
for r in 0 1 2 3; do
  TM_ROUTED_RING=$r $R --nproc-per-node 2 bench.py --gpus 2 --workload c5 --steps 20 > gpurun_out/y_ring$r.json 2> gpurun_out/y_ring$r.err
  tail -1 gpurun_out/y_ring$r.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ring=$r', round(d['value']/1e6,2),'Mq/s', round(d['ms_per_step'],4), 'walk', round(d['routed_walk_ms_avg_rank0'],4))"
done
echo done
