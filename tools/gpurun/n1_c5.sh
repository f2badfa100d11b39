#!/bin/bash
# N=1 c5 lines (plain python) for short-end CTA settings
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for t in 0 8; do
  TM_ROUTED_TAIL=$t timeout 400 python bench.py --workload c5 --steps 20 --warmup 5 > gpurun_out/sw_1_tail$t.json 2> gpurun_out/sw_1_tail$t.err
done
