#!/bin/bash
# 1 GPU: GPT-2 model mode cost decomposition of the checkpoint (2 repetitions).
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r02bf}
for rep in 1 2; do
  timeout 900 python tools/model_mode.py --steps 40 --warmup 5 \
    --arms ours_nockpt,ours_tap_nodrain,nockpt_d2hload,nockpt_d2hpaced,ours_tap_only,ours_ckpt \
    >> $OUT/${TAG}_model_n1_decomp.jsonl 2>> $OUT/${TAG}_model_n1_decomp.err
done
