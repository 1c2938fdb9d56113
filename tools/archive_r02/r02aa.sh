#!/bin/bash
# Model mode at N GPUs: the step's tail after backward with and without per-bucket optimizer steps.
cd "$(dirname "$0")/.."
N=${1:-2}; TAG=${2:-r02aa}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_model_tail_n$N.jsonl; : > $F
port=31900
for rep in 1 2; do
  for bs in 1 0; do
    port=$((port + 1))
    CM_BUCKET_STEP=$bs timeout 900 $RUN --master-port $port tools/model_mode.py --steps 20 --warmup 5 >> $F 2>> $OUT/${TAG}.err
  done
done
