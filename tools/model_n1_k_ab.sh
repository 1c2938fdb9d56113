#!/bin/bash
# 1 GPU: GPT-2 model mode, snapshot every K = 8 (D = 16) vs K = 16 (D = 17), alternating.
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r02bn}
for rep in 1 2; do
  timeout 600 python tools/model_mode.py --steps 100 --warmup 10 --arms nccl,ours_ckpt --persist-every 8 --ring-depth 16 >> $OUT/${TAG}_model_n1_k.jsonl 2>> $OUT/${TAG}.err
  timeout 600 python tools/model_mode.py --steps 100 --warmup 10 --arms nccl,ours_ckpt --persist-every 16 --ring-depth 17 >> $OUT/${TAG}_model_n1_k.jsonl 2>> $OUT/${TAG}.err
done
