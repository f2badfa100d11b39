#!/bin/bash
# e2e knob sweep (packed share, host threads) on whatever box this is
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
echo "nproc $(nproc)" > gpurun_out/e2e24.txt
lscpu | grep -i "model name\|L3\|Core(s)\|Thread(s)" >> gpurun_out/e2e24.txt
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --no-configs --no-c5 --no-cpu --steps 10 --warmup 3 --e2e-steps 8 > gpurun_out/e24_$name.json 2> gpurun_out/e24_$name.err
  python -c "import json; d=json.loads(open('gpurun_out/e24_$name.json').read().strip().splitlines()[-1]); print('$name', round(d['e2e']['value']))" >> gpurun_out/e2e24.txt
}
for t in 8 12 14 16; do
  for f in 0.9 0.95; do run f${f}_t$t TM_H2D_PACK_FRAC=$f TM_HOST_THREADS=$t; done
done
