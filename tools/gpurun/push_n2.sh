#!/bin/bash
# push vs fused routing at N=${NG:-2}: routed test worker, then c5 bench lines
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NG=${NG:-2}
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29561 tests/mp/routed_match.py > gpurun_out/push_test_$NG.log 2>&1
echo "test rc=$?" >> gpurun_out/push_test_$NG.log
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $NG --steps 20 --warmup 5 $EXTRA > gpurun_out/sw_${NG}_$name.json 2> gpurun_out/sw_${NG}_$name.err
}
EXTRA="--routing push" run push X=1
EXTRA="--routing push --no-pipeline" run push_nopipe X=1
EXTRA="--routing push" run push_g296 TM_PUSH_GRID=296
EXTRA="--routing push" run push_occ8 TM_PUSH_WALK_OCC=8
