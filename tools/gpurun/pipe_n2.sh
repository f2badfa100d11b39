# 2-GPU box: routed c5 batches pipelined over two routing regions (default) vs back to back.
# (Also swept this round and dropped: a small pack grid / 64-thread or TMA-staged pack CTAs /
# a capped walk occupancy, to make the next batch's pack co-run with the walk - all slower.)
set -x
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29519"
for mode in --pipeline --no-pipeline; do
  timeout 300 $R --nproc-per-node 2 bench.py --gpus 2 --workload c5 --steps 20 $mode > gpurun_out/p$mode.json 2> gpurun_out/p$mode.err
  tail -1 gpurun_out/p$mode.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$mode', round(d['value']/1e6,2),'Mq/s', round(d['ms_per_step'],4), 'walk', round(d['routed_walk_ms_avg_rank0'],4), d['phase_ms_avg_rank0'])"
done
