#!/bin/bash
# fused routing: batch size sweep at N=${NG:-2}
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NG=${NG:-2}
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $NG --steps 20 --warmup 5 $EXTRA > gpurun_out/sw_${NG}_$name.json 2> gpurun_out/sw_${NG}_$name.err
}
EXTRA="--queries 8192" run q8k X=1
EXTRA="--queries 16384" run q16k X=1
EXTRA="--queries 16384 --no-pipeline" run q16k_nopipe X=1
