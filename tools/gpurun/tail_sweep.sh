#!/bin/bash
# routed walk: short-end CTAs sweep at N=${NG:-2} (+ one trace with the default)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NG=${NG:-2}
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $NG --steps 20 --warmup 5 $EXTRA > gpurun_out/sw_${NG}_$name.json 2> gpurun_out/sw_${NG}_$name.err
}
for t in 0 4 8 16; do
  EXTRA="" run tail$t TM_ROUTED_TAIL=$t
done
EXTRA="--no-pipeline" run tail8_nopipe TM_ROUTED_TAIL=8
bash tools/gpurun/trace_n2.sh
