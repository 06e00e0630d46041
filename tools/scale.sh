#!/bin/bash
# Scaling curve on one 8-GPU node: bench.py at 1/2/4/8
# ranks (torchrun, NCCL over NVLink), one JSON line per N under
# gpurun_out/scale/, plus NCCL_DEBUG=INFO logs (look for NVLS / ring setup).
#   tools/scale.sh [config ...]     (default: c3 c5)
set -u
O=gpurun_out/scale; mkdir -p $O
CONFIGS=${@:-c3 c5}
NGPU=$(nvidia-smi -L | wc -l)
for c in $CONFIGS; do
  for n in 1 2 4 8; do
    [ "$n" -gt "$NGPU" ] && continue
    if [ "$n" -eq 1 ]; then
      timeout 1800 python bench.py --config $c --no-cpu-baseline --steps 20 --warmup 3 > $O/${c}_n$n.json 2> $O/${c}_n$n.err
    else
      NCCL_DEBUG=INFO timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
        --master-addr 127.0.0.1 --master-port $((29500 + n)) bench.py --gpus $n --config $c --no-cpu-baseline \
        --steps 20 --warmup 3 > $O/${c}_n$n.json 2> $O/${c}_n$n.err
    fi
  done
done
echo done
