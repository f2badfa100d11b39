# 2-GPU box: pipelined routed batches (two regions; next batch's bucket + pack beside the walk)
set -x
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29519"
run() { tag=$1; shift; env "$@" timeout 300 $R --nproc-per-node 2 bench.py --gpus 2 --workload c5 --steps 20 $PIPE > gpurun_out/p_$tag.json 2> gpurun_out/p_$tag.err
  tail -1 gpurun_out/p_$tag.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$tag', round(d['value']/1e6,2),'Mq/s', round(d['ms_per_step'],4), 'walk', round(d['routed_walk_ms_avg_rank0'],4), d['phase_ms_avg_rank0'])"; }
PIPE=--pipeline run pipe_default TM_X=0
PIPE=--pipeline run pipe_nt64_148 TM_ROUTE_PACK_NT=64 TM_ROUTE_PACK_CTAS=148
PIPE=--pipeline run pipe_nt64_296 TM_ROUTE_PACK_NT=64 TM_ROUTE_PACK_CTAS=296
PIPE=--pipeline run pipe_nt64_1184 TM_ROUTE_PACK_NT=64 TM_ROUTE_PACK_CTAS=1184
PIPE=--pipeline run pipe_nt64_4736 TM_ROUTE_PACK_NT=64 TM_ROUTE_PACK_CTAS=4736
PIPE=--pipeline run pipe_ctas2368 TM_ROUTE_PACK_CTAS=2368
PIPE=--pipeline run pipe_ctas592 TM_ROUTE_PACK_CTAS=592
echo done
