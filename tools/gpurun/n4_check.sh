#!/bin/bash
# N=4 routed check: test worker at 4 ranks, c5 lines for short-end CTA settings; N=1 c5 line
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tests/mp/routed_match.py > gpurun_out/routed_test_4.log 2>&1
echo "test rc=$?" >> gpurun_out/routed_test_4.log
run() {  # ng, name, env...
  local ng=$1; local name=$2; shift; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $ng --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $ng --steps 20 --warmup 5 $EXTRA > gpurun_out/sw_${ng}_$name.json 2> gpurun_out/sw_${ng}_$name.err
}
for t in 0 8 16; do EXTRA="" run 4 tail$t TM_ROUTED_TAIL=$t; done
for t in 0 8; do EXTRA="--workload c5" run 1 tail$t TM_ROUTED_TAIL=$t; done
