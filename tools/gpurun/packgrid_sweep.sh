#!/bin/bash
# routed pack grid sweep at N=${NG:-2} (fused routing, pipelined)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NG=${NG:-2}
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $NG --steps 20 --warmup 5 > gpurun_out/sw_${NG}_$name.json 2> gpurun_out/sw_${NG}_$name.err
}
for g in 296 592 1184 2368; do run grid$g TM_PACK_GRID=$g; done
