#!/bin/bash
# fused routing knob sweep at N=${NG:-2}
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NG=${NG:-2}
T=$GRAFT_REPO_ROOT/paper_2508_11553_b200/libtmstore_tuning.so
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $NG --steps 20 --warmup 5 $EXTRA > gpurun_out/sw_${NG}_$name.json 2> gpurun_out/sw_${NG}_$name.err
}
EXTRA="--no-pipeline" run f_nopipe X=1
EXTRA="--no-pipeline" run f_nopipe_occ8 TM_WALK_OCC=8
EXTRA="--no-pipeline" run f_nopipe_occ4 TM_WALK_OCC=4
EXTRA="--no-pipeline" run f_nopipe_ring1 TM_LIB=$T TM_ROUTED_RING=1
EXTRA="--no-pipeline" run f_nopipe_ring2 TM_LIB=$T TM_ROUTED_RING=2
EXTRA="--no-pipeline" run f_nopipe_ring3 TM_LIB=$T TM_ROUTED_RING=3
EXTRA="" run f_pipe X=1
