#!/bin/bash
# ncu evidence on one GPU (never a multi-rank command).  Each ncu command runs only after
# the identical command exited 0 without ncu.
cd "$(dirname "$0")/.."
OUT=gpurun_out
BENCH="python bench.py --steps 2 --warmup 1 --no-baseline --no-e2e --cpu-sample-s 0.2"
$BENCH > $OUT/ncu_bench_plain.json 2> $OUT/ncu_bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches.csv $BENCH > $OUT/ncu_launches.log 2>&1
echo "launch list rc=$?" >> $OUT/ncu_launches.log
TGT="python tools/prof_target.py --steps 2"
$TGT > $OUT/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:adamw_wt -s 0 -c 1 -o $OUT/prof_adamw $TGT > $OUT/ncu_adamw.log 2>&1
echo "adamw rc=$?" >> $OUT/ncu_adamw.log
ncu --set full --clock-control none --import-source on -k regex:rs_tap_ag -s 2 -c 1 -o $OUT/prof_rs_tap_ag $TGT > $OUT/ncu_ar.log 2>&1
echo "ar rc=$?" >> $OUT/ncu_ar.log
TGT8="python tools/prof_target.py --steps 2 --n 8"
$TGT8 > $OUT/prof_plain8.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rs_tap_ag -s 20 -c 1 -o $OUT/prof_rs_tap_ag_v8 $TGT8 > $OUT/ncu_ar8.log 2>&1
echo "ar8 rc=$?" >> $OUT/ncu_ar8.log
