#!/bin/bash
# e2e vs H2D chunk size (tokens per copy)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
echo "nproc $(nproc)" > gpurun_out/chunk.txt
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --no-configs --no-c5 --no-cpu --steps 10 --warmup 3 --e2e-steps 8 > gpurun_out/ch_$name.json 2> gpurun_out/ch_$name.err
  python -c "import json; d=json.loads(open('gpurun_out/ch_$name.json').read().strip().splitlines()[-1]); print('$name', round(d['e2e']['value']))" >> gpurun_out/chunk.txt
}
for c in 12 24 48; do run iss_k$c TM_H2D_CHUNKS=$c; run noiss_k$c TM_H2D_CHUNKS=$c TM_H2D_ISSUER=0; done; run iss_k24_t17 TM_H2D_CHUNKS=24 TM_HOST_THREADS=17
