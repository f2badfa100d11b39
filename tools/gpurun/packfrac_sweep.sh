#!/bin/bash
# e2e (c4, host-buffer C ABI) vs the share of tokens packed on the host (rest DMA'd raw)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for f in 1.0 0.95 0.9 0.85 0.8 0.7; do
  TM_H2D_PACK_FRAC=$f timeout 300 python bench.py --no-configs --no-c5 --no-cpu --steps 10 --warmup 3 --e2e-steps 8 > gpurun_out/pf_$f.json 2> gpurun_out/pf_$f.err
  python -c "import json; d=json.loads(open('gpurun_out/pf_$f.json').read().strip().splitlines()[-1]); print('$f', d['e2e'])" >> gpurun_out/pf_summary.txt
done
nproc >> gpurun_out/pf_summary.txt
