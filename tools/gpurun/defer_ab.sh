#!/bin/bash
# deferred done-wait A/B at N=${NG:-2} (+ routed test worker)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NG=${NG:-2}
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29561 tests/mp/routed_match.py > gpurun_out/routed_test_$NG.log 2>&1
echo "test rc=$?" >> gpurun_out/routed_test_$NG.log
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $NG --steps 20 --warmup 5 $EXTRA > gpurun_out/sw_${NG}_$name.json 2> gpurun_out/sw_${NG}_$name.err
}
for r in 1 2; do
  EXTRA="" run defer_$r BENCH_DEFER_DONE=1
  EXTRA="" run nodefer_$r BENCH_DEFER_DONE=0
done
