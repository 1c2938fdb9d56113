#!/bin/bash
# Final-tree ncu evidence on one GPU (each ncu command after the same command exited 0):
#   1. the default bench's launch list (shares), 2. DRAM bytes per launch of 3 GPT-2
#   iterations in the bench's shadow config (profiles/traffic.json), 3. --set full of the
#   bulk-copy all-reduce (rs_tap_ag_tma_kernel, 2 virtual ranks on one GPU).
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r02av}
BENCH="python bench.py --steps 2 --warmup 1 --no-baseline --no-e2e --no-model --cpu-sample-s 0"
$BENCH > $OUT/${TAG}_bench_plain.json 2> $OUT/${TAG}_bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $OUT/${TAG}_launches.csv $BENCH > $OUT/${TAG}_launches.log 2>&1
echo "launch list rc=$?" >> $OUT/${TAG}_launches.log
TGT="python tools/prof_target.py --steps 3 --ring-depth 16 --persist-every 8"
$TGT > $OUT/${TAG}_prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"rs_tap_ag|adamw_wt|gen_grads" --csv --log-file $OUT/${TAG}_dram.csv $TGT > $OUT/${TAG}_dram.log 2>&1
echo "dram rc=$?" >> $OUT/${TAG}_dram.log
TGT2="python tools/prof_target.py --n 2 --steps 2 --ring-depth 4 --persist-every 2"
$TGT2 > $OUT/${TAG}_prof2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rs_tap_ag_tma -s 20 -c 1 -o $OUT/${TAG}_ar_tma $TGT2 > $OUT/${TAG}_ncu_ar_tma.log 2>&1
echo "ar tma rc=$?" >> $OUT/${TAG}_ncu_ar_tma.log
