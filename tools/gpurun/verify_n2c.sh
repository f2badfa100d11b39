# 2-GPU box: routed tests + c5 N=2 (faster k_route / pack), then a one-GPU e2e sweep of TM_H2D_PACK_FRAC
set -x
python -m pytest tests/test_routing_gpu.py tests/test_h2d_pack_gpu.py -q -x > gpurun_out/x_tests.log 2>&1; tail -3 gpurun_out/x_tests.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29515"
$R --nproc-per-node 2 bench.py --gpus 2 --workload c5 --steps 20 > gpurun_out/x_n2_c5.json 2> gpurun_out/x_n2_c5.err
for f in 1.0 0.9 0.8 0.7 0.6; do
  TM_H2D_PACK_FRAC=$f python bench.py --steps 5 --no-cpu --e2e-steps 6 > gpurun_out/x_e2e_$f.json 2> gpurun_out/x_e2e_$f.err
  tail -1 gpurun_out/x_e2e_$f.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('frac=$f', round(d['value']/1e6,2), 'Mq/s e2e', round(d['e2e']['value']/1e3), 'kq/s h2d', d['e2e']['h2d_bytes_per_step'])"
done
echo done
