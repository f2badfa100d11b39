#!/bin/bash
# routed walk with record look-ahead at N=${NG:-2}: test worker, bench lines, one trace
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NG=${NG:-2}
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29561 tests/mp/routed_match.py > gpurun_out/routed_test_$NG.log 2>&1
echo "test rc=$?" >> gpurun_out/routed_test_$NG.log
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $NG --steps 20 --warmup 5 $EXTRA > gpurun_out/sw_${NG}_$name.json 2> gpurun_out/sw_${NG}_$name.err
}
EXTRA="" run fused X=1
EXTRA="--no-pipeline" run fused_nopipe X=1
EXTRA="" run fused_tail8 TM_ROUTED_TAIL=8
bash tools/gpurun/trace_n2.sh
