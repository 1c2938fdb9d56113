#!/bin/bash
# Round-1d: AdamW microbench (fp32 / bf16 grads), the bench launch list of the current code,
# and full sets of adamw_wt (fp32 and bf16 grads).  Each ncu command runs only after the
# same command exited 0 without ncu.
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r01d}
timeout 300 python tools/microbench.py adamw_wt adamw_bf16_wt adamw_bf16_vec > $OUT/mb_adamw_$TAG.jsonl 2> $OUT/mb_adamw_$TAG.err
BENCH="python bench.py --steps 2 --warmup 3 --no-baseline --no-e2e --no-model --cpu-sample-s 0.2"
$BENCH > $OUT/ncu_bench_plain_$TAG.json 2> $OUT/ncu_bench_plain_$TAG.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $OUT/launches_$TAG.csv $BENCH > $OUT/ncu_launches_$TAG.log 2>&1
echo "launch list rc=$?" >> $OUT/ncu_launches_$TAG.log
T3="python tools/prof_target.py --steps 2"
$T3 > $OUT/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:adamw_wt -s 0 -c 1 -o $OUT/prof_adamw_$TAG $T3 > $OUT/ncu_adamw_$TAG.log 2>&1
echo "adamw rc=$?" >> $OUT/ncu_adamw_$TAG.log
T5="python tools/prof_target.py --steps 2 --dtype bf16"
$T5 > $OUT/prof_plain_bf16_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:adamw_wt -s 0 -c 1 -o $OUT/prof_adamw_bf16_$TAG $T5 > $OUT/ncu_adamw_bf16_$TAG.log 2>&1
echo "adamw bf16 rc=$?" >> $OUT/ncu_adamw_bf16_$TAG.log
