#!/bin/bash
# 1 GPU: GPT-2 model mode, 4 repetitions of (NCCL DDP, ours no-ckpt, ours ckpt) at 40 timed
# iterations each -- the n=1 checkpoint overhead with its run-to-run spread.
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r02be}
for rep in 1 2 3 4; do
  timeout 600 python tools/model_mode.py --steps 40 --warmup 5 >> $OUT/${TAG}_model_n1_reps.jsonl 2>> $OUT/${TAG}_model_n1_reps.err
done
