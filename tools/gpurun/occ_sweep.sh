#!/bin/bash
# routed walk CTAs per SM at N=${NG:-4}
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NG=${NG:-4}
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $NG --steps 20 --warmup 5 $EXTRA > gpurun_out/sw_${NG}_$name.json 2> gpurun_out/sw_${NG}_$name.err
}
for o in 6 7 8; do EXTRA="" run occ$o TM_WALK_OCC=$o; done
EXTRA="" run occ8_tail4 TM_WALK_OCC=8 TM_ROUTED_TAIL=4
