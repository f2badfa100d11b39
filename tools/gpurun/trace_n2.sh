#!/bin/bash
# routed-walk item timeline at N=${NG:-2} (TM_ROUTED_TRACE; synchronous, not a timing run)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
NG=${NG:-2}
rm -f gpurun_out/rtrace.*
TM_ROUTED_TRACE=gpurun_out/rtrace timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus $NG --steps 4 --warmup 3 --no-pipeline > gpurun_out/trace_bench.json 2> gpurun_out/trace_bench.err
python tools/routed_trace.py gpurun_out/rtrace > gpurun_out/rtrace_summary.txt 2>&1
rm -f gpurun_out/rtrace.*
