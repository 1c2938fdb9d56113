#!/bin/bash
# n=1 model mode: the tap's bytes as one plain copy-engine D2H per iteration vs the same
# bytes in small chunks released from forward pre-hooks (paced) -- is the copy engine's
# interference with the training step a matter of saturation bursts?
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r01m_paced}
F=$OUT/${TAG}.jsonl; : > $F
for rep in 1 2; do
  timeout 600 python tools/model_mode.py --steps 20 --warmup 5 --arms ours_nockpt,nockpt_d2hload,nockpt_d2hpaced >> $F 2>> $OUT/${TAG}.err
done
