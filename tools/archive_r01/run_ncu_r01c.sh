#!/bin/bash
# ncu evidence for the round-1c kernels on one GPU (each ncu command only after the same
# command exited 0 without ncu): the bench launch list, full sets of sgd_wt_kernel and the
# SM drain_kernel, and a refreshed adamw_wt_kernel / rs_tap_ag full set.
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r01c}
BENCH="python bench.py --steps 2 --warmup 3 --no-baseline --no-e2e --no-model --cpu-sample-s 0.2"
$BENCH > $OUT/ncu_bench_plain_$TAG.json 2> $OUT/ncu_bench_plain_$TAG.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $OUT/launches_$TAG.csv $BENCH > $OUT/ncu_launches_$TAG.log 2>&1
echo "launch list rc=$?" >> $OUT/ncu_launches_$TAG.log
T1="python tools/prof_target.py --steps 2 --opt sgd"
$T1 > $OUT/prof_plain_sgd_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sgd_wt -s 0 -c 1 -o $OUT/prof_sgd_$TAG $T1 > $OUT/ncu_sgd_$TAG.log 2>&1
echo "sgd rc=$?" >> $OUT/ncu_sgd_$TAG.log
T2="python tools/prof_target.py --steps 2 --drain-ctas 1"
$T2 > $OUT/prof_plain_drain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:drain_kernel -s 2 -c 1 -o $OUT/prof_drain_$TAG $T2 > $OUT/ncu_drain_$TAG.log 2>&1
echo "drain rc=$?" >> $OUT/ncu_drain_$TAG.log
T3="python tools/prof_target.py --steps 2"
$T3 > $OUT/prof_plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:adamw_wt -s 0 -c 1 -o $OUT/prof_adamw_$TAG $T3 > $OUT/ncu_adamw_$TAG.log 2>&1
echo "adamw rc=$?" >> $OUT/ncu_adamw_$TAG.log
T4="python tools/prof_target.py --steps 2 --n 4"
$T4 > $OUT/prof_plain4_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rs_tap_ag -s 10 -c 1 -o $OUT/prof_rs_tap_ag_v4_$TAG $T4 > $OUT/ncu_ar4_$TAG.log 2>&1
echo "ar4 rc=$?" >> $OUT/ncu_ar4_$TAG.log
