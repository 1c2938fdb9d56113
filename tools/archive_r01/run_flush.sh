#!/bin/bash
# A/B of the drain flush size at N (synthetic checkpointed step), alternating runs.
cd "$(dirname "$0")/.."
N=$1; TAG=${2:-fl}; OUT=gpurun_out; F=$OUT/${TAG}_flush_n$N.jsonl; rm -f $F
if [ "$N" = "1" ]; then B="python"; else B="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29781"; fi
for fb in 0 8388608 67108864 0 8388608 67108864; do
  CM_DRAIN_FLUSH_BYTES=$fb timeout 400 $B bench.py --gpus $N --steps 20 --warmup 5 --no-model --no-baseline --no-e2e --no-variants | sed "s/^{/{\"flush\": $fb, /" >> $F 2>> $OUT/${TAG}_flush_n$N.err
done
