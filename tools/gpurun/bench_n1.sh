#!/bin/bash
# N=1 bench line + reference arm (the driver's order)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nproc > gpurun_out/bn1_nproc.txt
timeout 900 python bench.py --impl reference > gpurun_out/bn1_reference.json 2> gpurun_out/bn1_reference.err
timeout 1200 python bench.py > gpurun_out/bn1.json 2> gpurun_out/bn1.err
