# 2-GPU box: routed c5 batches - pipelined (side-stream pack) vs back to back
set -x
TM_PEER_TIMEOUT_MS=5000 timeout 400 python -m pytest tests/test_routing_gpu.py -q -x > gpurun_out/pt_tests.log 2>&1; tail -2 gpurun_out/pt_tests.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29519"
run() { tag=$1; shift; env "$@" timeout 300 $R --nproc-per-node 2 bench.py --gpus 2 --workload c5 --steps 20 $PIPE > gpurun_out/pt_$tag.json 2> gpurun_out/pt_$tag.err
  tail -1 gpurun_out/pt_$tag.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', round(d['value']/1e6,2),'Mq/s', round(d['ms_per_step'],4), 'walk', round(d['routed_walk_ms_avg_rank0'],4), d['phase_ms_avg_rank0'])"; }
PIPE=--pipeline run side TM_X=0
PIPE=--no-pipeline run none TM_X=0
echo done
