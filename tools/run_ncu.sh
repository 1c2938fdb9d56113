#!/bin/bash
# ncu evidence on one GPU (never a multi-rank command).  Each ncu command runs only after
# the identical command exited 0 without ncu.  Usage: tools/run_ncu.sh <tag>
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r01b}
BENCH="python bench.py --steps 2 --warmup 1 --no-baseline --no-e2e --no-model --cpu-sample-s 0.2"
$BENCH > $OUT/ncu_bench_plain_$TAG.json 2> $OUT/ncu_bench_plain_$TAG.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $OUT/launches_$TAG.csv $BENCH > $OUT/ncu_launches_$TAG.log 2>&1
echo "launch list rc=$?" >> $OUT/ncu_launches_$TAG.log
TGT="python tools/prof_target.py --steps 2"
$TGT > $OUT/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:adamw_wt -s 0 -c 1 -o $OUT/prof_adamw_$TAG $TGT > $OUT/ncu_adamw_$TAG.log 2>&1
echo "adamw rc=$?" >> $OUT/ncu_adamw_$TAG.log
ncu --set full --clock-control none --import-source on -k regex:rs_tap_ag -s 2 -c 1 -o $OUT/prof_rs_tap_ag_$TAG $TGT > $OUT/ncu_ar_$TAG.log 2>&1
echo "ar rc=$?" >> $OUT/ncu_ar_$TAG.log
TGT8="python tools/prof_target.py --steps 2 --n 4"
$TGT8 > $OUT/prof_plain4_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rs_tap_ag -s 10 -c 1 -o $OUT/prof_rs_tap_ag_v4_$TAG $TGT8 > $OUT/ncu_ar4_$TAG.log 2>&1
echo "ar4 rc=$?" >> $OUT/ncu_ar4_$TAG.log
