#!/bin/bash
# Model mode at N GPUs: per-bucket steps on the comm stream vs on a lowest-priority stream.
cd "$(dirname "$0")/.."
N=${1:-1}; TAG=${2:-r02ab}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_model_n$N.jsonl; : > $F
port=32000
for rep in 1 2; do
  for cfg in "CM_BUCKET_STREAM=comm" "CM_BUCKET_STREAM=low" "CM_BUCKET_STEP=0"; do
    port=$((port + 1))
    env $cfg timeout 900 $RUN --master-port $port tools/model_mode.py --steps 20 --warmup 5 --arms nccl,ours_nockpt,ours_ckpt >> $F 2>> $OUT/${TAG}.err
  done
done
