# 4-GPU box: routed c5 at N = 2, 4 (pipelined default, and back to back) after the pipelining change
set -x
TM_PEER_TIMEOUT_MS=5000 timeout 400 python -m pytest tests/test_routing_gpu.py -q -x > gpurun_out/n4c_tests.log 2>&1; tail -2 gpurun_out/n4c_tests.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29520"
for n in 2 4; do
  timeout 300 $R --nproc-per-node $n bench.py --gpus $n --workload c5 --steps 20 > gpurun_out/n4c_c5_n$n.json 2> gpurun_out/n4c_c5_n$n.err
  timeout 300 $R --nproc-per-node $n bench.py --gpus $n --workload c5 --steps 20 --no-pipeline > gpurun_out/n4c_c5np_n$n.json 2> gpurun_out/n4c_c5np_n$n.err
done
echo done
