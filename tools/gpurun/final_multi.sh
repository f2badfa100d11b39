#!/bin/bash
# round-end multi-GPU bench lines: N=2 and N=4, reference arm first (as the driver does)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for ng in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $ng --master-addr 127.0.0.1 --master-port 29581 bench.py --impl reference --gpus $ng --steps 10 --warmup 3 > gpurun_out/final_n${ng}_reference.json 2> gpurun_out/final_n${ng}_reference.err
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $ng --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus $ng --steps 20 --warmup 5 > gpurun_out/final_n${ng}.json 2> gpurun_out/final_n${ng}.err
done
