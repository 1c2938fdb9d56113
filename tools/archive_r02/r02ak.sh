#!/bin/bash
# Model mode at N GPUs: the all-reduce kernel choice (hybrid bulk-copy vs per-thread) in a real
# training step (the bulk-copy kernel holds shared memory on every SM while backward runs).
cd "$(dirname "$0")/.."
N=${1:-2}; TAG=${2:-r02ak}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_model_n$N.jsonl; : > $F
port=32400
for rep in 1 2 3; do
  for impl in -1 0; do
    port=$((port + 1))
    CM_AR_IMPL=$impl timeout 900 $RUN --master-port $port tools/model_mode.py --steps 20 --warmup 5 --arms nccl,ours_nockpt,ours_ckpt >> $F 2>> $OUT/${TAG}.err
  done
done
