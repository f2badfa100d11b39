#!/bin/bash
# per-call latency (tools/latency.py) with K2 shape variants (tuning build)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
T=$GRAFT_REPO_ROOT/paper_2508_11553_b200/libtmstore_tuning.so
for v in default tma3x256 tma2x128 t32x2x64 ws32x2x64; do
  echo "== $v" >> gpurun_out/lat_variants.txt
  TM_LIB=$T TM_RECORD_VARIANT=$v timeout 200 python tools/latency.py 2>/dev/null | head -2 >> gpurun_out/lat_variants.txt
done
