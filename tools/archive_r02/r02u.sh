#!/bin/bash
# n=1 model mode A/B: shadow step after the training optimizer vs after the last all-reduce,
# with and without per-bucket steps.
cd "$(dirname "$0")/.."
TAG=${1:-r02u}; OUT=gpurun_out
F=$OUT/${TAG}_model_n1.jsonl; : > $F
for rep in 1 2; do
  for cfg in "CM_SHADOW_AFTER_TRAIN=0" "CM_SHADOW_AFTER_TRAIN=1" "CM_SHADOW_AFTER_TRAIN=1 CM_BUCKET_STEP=0"; do
    env $cfg timeout 900 python tools/model_mode.py --steps 20 --warmup 5 --arms nccl,ours_ckpt >> $F 2>> $OUT/${TAG}.err
  done
done
