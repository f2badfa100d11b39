# 2-GPU check of the routed path (gpurun --gpus 2): routing tests, c5 at N=2 in all three exchange modes
set -x
python -m pytest tests/test_routing_gpu.py -q -x > gpurun_out/w_tests.log 2>&1; tail -3 gpurun_out/w_tests.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29514"
$R --nproc-per-node 2 bench.py --gpus 2 --workload c5 --steps 20 > gpurun_out/w_n2_c5.json 2> gpurun_out/w_n2_c5.err
$R --nproc-per-node 2 bench.py --gpus 2 --workload c5 --steps 20 --routing fused-nccl-barrier > gpurun_out/w_n2_c5_nb.json 2> gpurun_out/w_n2_c5_nb.err
$R --nproc-per-node 2 bench.py --gpus 2 --workload c5 --steps 10 --routing nccl > gpurun_out/w_n2_c5_nccl.json 2> gpurun_out/w_n2_c5_nccl.err
echo done
