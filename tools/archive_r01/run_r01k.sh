#!/bin/bash
# Final 1-GPU evidence: GPU suite, smoke, bench; then an ncu full set of the bf16-grad
# AdamW after the zero-operand fast path (after its plain run exited 0).
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r01k}
bash tools/run_r01e.sh 1 $TAG
T5="python tools/prof_target.py --steps 2 --dtype bf16"
$T5 > $OUT/prof_plain_bf16_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:adamw_wt -s 0 -c 1 -o $OUT/prof_adamw_bf16_$TAG $T5 > $OUT/ncu_adamw_bf16_$TAG.log 2>&1
echo "adamw bf16 rc=$?" >> $OUT/ncu_adamw_bf16_$TAG.log
