#!/bin/bash
# e2e (c4, host-buffer C ABI): packed staging through a ring of LLC-sized slots vs one
# full-size buffer, and the packed share; reference arm once for the box
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nproc > gpurun_out/rs_summary.txt
lscpu | grep -i "model name\|L3\|Socket\|NUMA node(s)" >> gpurun_out/rs_summary.txt
timeout 600 python -m pytest tests/test_h2d_pack_gpu.py -q > gpurun_out/rs_tests.log 2>&1; tail -1 gpurun_out/rs_tests.log >> gpurun_out/rs_summary.txt
run() {  # name, env...
  local name=$1; shift
  env "$@" timeout 300 python bench.py --no-configs --no-c5 --no-cpu --steps 10 --warmup 3 --e2e-steps 8 > gpurun_out/rs_$name.json 2> gpurun_out/rs_$name.err
  python -c "import json; d=json.loads(open('gpurun_out/rs_$name.json').read().strip().splitlines()[-1]); print('$name', round(d['e2e']['value']), d['e2e']['h2d_bytes_per_step'])" >> gpurun_out/rs_summary.txt
}
run full_f1 TM_H2D_RING=0 TM_H2D_PACK_FRAC=1.0
run full_f09 TM_H2D_RING=0 TM_H2D_PACK_FRAC=0.9
run ring8_f1 TM_H2D_RING=8 TM_H2D_PACK_FRAC=1.0
run ring8_f09 TM_H2D_RING=8 TM_H2D_PACK_FRAC=0.9
run ring16_f1 TM_H2D_RING=16 TM_H2D_PACK_FRAC=1.0
run ring4_1m_f1 TM_H2D_RING=4 TM_H2D_RING_TOKENS=1048576 TM_H2D_PACK_FRAC=1.0
run ring32_128k_f1 TM_H2D_RING=32 TM_H2D_RING_TOKENS=131072 TM_H2D_PACK_FRAC=1.0
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/rs_ref.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/rs_ref.json').read().strip().splitlines()[-1]); print('reference', round(d['value']), d['cpu_baseline']['cores'])" >> gpurun_out/rs_summary.txt
