#!/bin/bash
# n=1 model mode: host snapshot every K=8 vs K=16 steps (ring depth 16 both), two reps.
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r01s_k}
F=$OUT/${TAG}.jsonl; : > $F
for rep in 1 2; do
  for k in 8 16; do
    echo "{\"persist_every\": $k}" >> $F
    timeout 600 python tools/model_mode.py --steps 20 --warmup 5 --persist-every $k --ring-depth 16 --arms nccl,ours_ckpt >> $F 2>> $OUT/${TAG}.err
  done
done
