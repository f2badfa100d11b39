# e2e (host-buffer path) with and without packed H2D at N=2 and N=4 (gpurun --gpus 4)
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29512"
for n in 2 4; do
  for mode in 0 -1; do
    for thr in 16 8 4; do
      [ "$mode" = "-1" ] && [ "$thr" != "16" ] && continue
      TM_H2D_PACK_MIN=$mode TM_HOST_THREADS=$thr $R --nproc-per-node $n bench.py --gpus $n --steps 5 --e2e-steps 3 > gpurun_out/ps_$n_$mode_$thr.json 2>/dev/null
      tail -1 gpurun_out/ps_$n_$mode_$thr.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$n pack_min=$mode threads=$thr', round(d['value']/1e6,1), 'Mq/s e2e', round(d['e2e']['value']/1e3), 'kq/s')"
    done
  done
done
