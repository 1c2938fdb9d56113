#!/bin/bash
# 1 GPU: --set full of the training AdamW (the dominant kernel at n=1) and of the shadow's
# AdamW, GPT-2 size, after the same target exited 0 without ncu.
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r02bd}
TGT="python tools/prof_target.py --steps 3 --ring-depth 16 --persist-every 8"
$TGT > $OUT/${TAG}_prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:adamw_wt -s 2 -c 2 -o $OUT/${TAG}_adamw $TGT > $OUT/${TAG}_ncu_adamw.log 2>&1
echo "adamw rc=$?" >> $OUT/${TAG}_ncu_adamw.log
