#!/bin/bash
# one ncu --set full capture of K2 on config 3 (after a clean run of the same command)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python tools/bench_paths.py --configs 3 --no-cpu --reps 2 > gpurun_out/c3_paths.jsonl 2> gpurun_out/c3_paths.err || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_record -c 1 -s 1 -o gpurun_out/c3_k_record \
  python tools/bench_paths.py --configs 3 --no-cpu --reps 1 > gpurun_out/c3_ncu.log 2>&1
