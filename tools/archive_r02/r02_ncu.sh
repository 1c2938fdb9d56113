#!/bin/bash
# ncu evidence on one GPU for the current kernels (never a multi-rank command; each ncu command
# runs only after the same command exited 0 without ncu):
#   1. the bench's launch list (gpu__time_duration, cold-cache, serialised: shares)
#   2. DRAM bytes + duration of every launch of 3 GPT-2 iterations (bench shadow config K=8, D=16)
#      -> profiles/traffic.json via tools/traffic_from_ncu.py
#   3. --set full of the training AdamW, one all-reduce (staged tap) and one shadow AdamW
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r02g}
BENCH="python bench.py --steps 2 --warmup 1 --no-baseline --no-e2e --no-model --cpu-sample-s 0"
$BENCH > $OUT/${TAG}_bench_plain.json 2> $OUT/${TAG}_bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $OUT/${TAG}_launches.csv $BENCH > $OUT/${TAG}_launches.log 2>&1
echo "launch list rc=$?" >> $OUT/${TAG}_launches.log
TGT="python tools/prof_target.py --steps 3 --ring-depth 16 --persist-every 8"
$TGT > $OUT/${TAG}_prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"rs_tap_ag|adamw_wt|gen_grads" --csv --log-file $OUT/${TAG}_dram.csv $TGT > $OUT/${TAG}_dram.log 2>&1
echo "dram rc=$?" >> $OUT/${TAG}_dram.log
ncu --set full --clock-control none --import-source on -k regex:adamw_wt -s 1 -c 1 -o $OUT/${TAG}_adamw $TGT > $OUT/${TAG}_ncu_adamw.log 2>&1
echo "adamw rc=$?" >> $OUT/${TAG}_ncu_adamw.log
ncu --set full --clock-control none --import-source on -k regex:rs_tap_ag -s 18 -c 1 -o $OUT/${TAG}_ar $TGT > $OUT/${TAG}_ncu_ar.log 2>&1
echo "ar rc=$?" >> $OUT/${TAG}_ncu_ar.log
ncu --set full --clock-control none --import-source on -k regex:adamw_wt -s 2 -c 1 -o $OUT/${TAG}_shadow $TGT > $OUT/${TAG}_ncu_shadow.log 2>&1
echo "shadow rc=$?" >> $OUT/${TAG}_ncu_shadow.log
