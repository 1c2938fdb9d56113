#!/bin/bash
# n=1 model mode: does a low-intensity shadow AdamW (few CTAs on the lowest-priority stream)
# hide under the training step better than the full-grid one?  Two alternating reps.
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r01m_sb}
F=$OUT/${TAG}.jsonl; : > $F
for rep in 1 2; do
  timeout 600 python tools/model_mode.py --steps 20 --warmup 5 --arms nccl,ours_nockpt >> $F 2>> $OUT/${TAG}.err
  for sb in 296 32 8; do
    echo "{\"shadow_blocks\": $sb}" >> $F
    CM_SHADOW_BLOCKS=$sb timeout 600 python tools/model_mode.py --steps 20 --warmup 5 --arms ours_ckpt >> $F 2>> $OUT/${TAG}.err
  done
done
