#!/bin/bash
# The scaling curve the driver measures, for a maintainer with one node of N B200s:
# N = 1 (c4 headline), then N = 2, 4, 8 under torchrun (routed c5 headline + c4 / c2 / c3
# shards), each preceded by the reference arm as the driver runs it.  Lines go to
# scale_out/bench_n<N>.json and scale_out/bench_n<N>_reference.json.
#   tools/scale.sh [max_gpus] [steps] [warmup]
set -u
cd "$(dirname "$0")/.."
MAX=${1:-8}
STEPS=${2:-20}
WARM=${3:-5}
mkdir -p scale_out
NGPU=$(python -c "import torch; print(torch.cuda.device_count())")
for n in 1 2 4 8; do
  [ "$n" -gt "$MAX" ] || [ "$n" -gt "$NGPU" ] && break
  if [ "$n" -eq 1 ]; then
    python bench.py --impl reference --steps "$STEPS" --warmup "$WARM" > scale_out/bench_n1_reference.json
    python bench.py --steps "$STEPS" --warmup "$WARM" > scale_out/bench_n1.json
  else
    for impl in reference b200; do
      suffix=$([ "$impl" = reference ] && echo "_reference" || echo "")
      python -m torch.distributed.run --nnodes=1 --nproc-per-node "$n" --master-addr 127.0.0.1 \
        --master-port $((29600 + n)) bench.py --impl "$impl" --gpus "$n" --steps "$STEPS" --warmup "$WARM" \
        > "scale_out/bench_n${n}${suffix}.json"
    done
  fi
  python -c "import json,sys; d=json.loads(open('scale_out/bench_n$n.json').read().strip().splitlines()[-1]); print('N=$n', d['metric'], round(d['value'] / 1e6, 2), 'M', d['unit'])"
done
