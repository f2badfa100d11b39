# 2-GPU verification (gpurun --gpus 2): GPU suite incl. world-2 routing, c4 N=1, routed c5 at N=2 packed vs raw
set -x
python -m pytest tests -m gpu -q -x > gpurun_out/v_tests.log 2>&1; tail -3 gpurun_out/v_tests.log
python bench.py > gpurun_out/v_bench_c4.json 2> gpurun_out/v_bench_c4.err
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29513"
$R --nproc-per-node 2 bench.py --gpus 2 --workload c5 --steps 20 > gpurun_out/v_n2_c5.json 2> gpurun_out/v_n2_c5.err
TM_ROUTE_PACK=0 $R --nproc-per-node 2 bench.py --gpus 2 --workload c5 --steps 20 > gpurun_out/v_n2_c5_nopack.json 2> gpurun_out/v_n2_c5_nopack.err
python tools/route_pack_probe.py > gpurun_out/v_pack_probe.txt 2>&1
echo done
