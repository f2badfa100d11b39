# 4-GPU box (gpurun --gpus 4): GPU suite, one-GPU bench lines, 2/4-GPU c4 (host-routed) and c5 (routed) lines
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/n4b_tests.log 2>&1; tail -2 gpurun_out/n4b_tests.log
python bench.py > gpurun_out/n4b_c4_n1.json 2> gpurun_out/n4b_c4_n1.err
python bench.py --impl reference --steps 5 > gpurun_out/n4b_ref_n1.json 2> gpurun_out/n4b_ref_n1.err
python bench.py --workload c5 --steps 20 > gpurun_out/n4b_c5_n1.json 2> gpurun_out/n4b_c5_n1.err
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29518"
for n in 2 4; do
  timeout 600 $R --nproc-per-node $n bench.py --gpus $n > gpurun_out/n4b_c4_n$n.json 2> gpurun_out/n4b_c4_n$n.err
  timeout 300 $R --nproc-per-node $n bench.py --gpus $n --workload c5 --steps 20 > gpurun_out/n4b_c5_n$n.json 2> gpurun_out/n4b_c5_n$n.err
  timeout 300 $R --nproc-per-node $n bench.py --gpus $n --workload c5 --steps 20 --routing fused-nccl-barrier > gpurun_out/n4b_c5nb_n$n.json 2> gpurun_out/n4b_c5nb_n$n.err
  timeout 300 $R --nproc-per-node $n bench.py --gpus $n --workload c5 --steps 10 --routing nccl > gpurun_out/n4b_c5nccl_n$n.json 2> gpurun_out/n4b_c5nccl_n$n.err
done
timeout 600 $R --nproc-per-node 4 bench.py --gpus 4 --impl reference --steps 3 > gpurun_out/n4b_ref_n4.json 2> gpurun_out/n4b_ref_n4.err
echo done
