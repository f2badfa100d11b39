# 2/4-GPU measurements (gpurun --gpus 4): weak-scaling c4 and the routed c5 path.
set -x
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29511"
$R --nproc-per-node 4 bench.py --gpus 4 > gpurun_out/n4_bench_c4.json 2> gpurun_out/n4_bench_c4.err
$R --nproc-per-node 4 bench.py --gpus 4 --impl reference --steps 3 > gpurun_out/n4_ref_c4.json 2> gpurun_out/n4_ref_c4.err
$R --nproc-per-node 4 bench.py --gpus 4 --workload c5 --steps 20 > gpurun_out/n4_bench_c5.json 2> gpurun_out/n4_bench_c5.err
$R --nproc-per-node 4 bench.py --gpus 4 --workload c5 --steps 20 --routing fused-nccl-barrier > gpurun_out/n4_bench_c5_ncclbar.json 2> gpurun_out/n4_bench_c5_ncclbar.err
$R --nproc-per-node 4 bench.py --gpus 4 --workload c5 --steps 10 --routing nccl > gpurun_out/n4_bench_c5_nccl.json 2> gpurun_out/n4_bench_c5_nccl.err
$R --nproc-per-node 2 bench.py --gpus 2 --workload c5 --steps 20 > gpurun_out/n2_bench_c5.json 2> gpurun_out/n2_bench_c5.err
$R --nproc-per-node 2 bench.py --gpus 2 > gpurun_out/n2_bench_c4.json 2> gpurun_out/n2_bench_c4.err
echo done
