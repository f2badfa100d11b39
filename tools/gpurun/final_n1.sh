#!/bin/bash
# round-end: GPU tests (2-GPU box), smoke, N=1 reference arm then N=1 bench line
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_gpu_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/final_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/final_smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/final_n1_reference.json 2> gpurun_out/final_n1_reference.err
timeout 1200 python bench.py > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err
