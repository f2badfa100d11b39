#!/bin/bash
# push routing knob sweep at N=${NG:-2}: one c5 bench line per setting
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NG=${NG:-2}
run() {  # name, env..., -- extra bench args
  local name=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $NG --steps 20 --warmup 5 $EXTRA > gpurun_out/sw_${NG}_$name.json 2> gpurun_out/sw_${NG}_$name.err
}
EXTRA="--routing push --no-pipeline" run nopipe X=1
EXTRA="--routing push" run occ3 TM_PUSH_WALK_OCC=3
EXTRA="--routing push" run occ4 TM_PUSH_WALK_OCC=4
EXTRA="--routing push" run grid296 TM_PACK_GRID=296
EXTRA="--routing push" run grid592_occ4 TM_PACK_GRID=592 TM_PUSH_WALK_OCC=4
EXTRA="--routing push" run grid2368 TM_PACK_GRID=2368
