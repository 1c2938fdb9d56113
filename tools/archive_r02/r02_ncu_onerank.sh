#!/bin/bash
# ncu NVLink counters for ONE profiled rank of a 2-rank run: rank 0 under ncu (few metrics,
# kernel replay: the replayed barrier passes at once, epochs are ">="), rank 1 plain.
cd "$(dirname "$0")/.."
TAG=${1:-r02h}; OUT=gpurun_out; Z=${2:-}
M=gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
export MASTER_ADDR=127.0.0.1 MASTER_PORT=30911 WORLD_SIZE=2 CM_PDL=0
RANK=1 LOCAL_RANK=1 timeout 600 python tools/ncu_target_mp.py --steps 2 $Z > $OUT/${TAG}_onerank_r1$Z.log 2>&1 &
P1=$!
RANK=0 LOCAL_RANK=0 timeout 600 ncu --metrics $M --clock-control none -k regex:"rs_tap_ag|adamw_zero1" -c 40 --csv \
   --log-file $OUT/${TAG}_onerank$Z.csv python tools/ncu_target_mp.py --steps 2 $Z > $OUT/${TAG}_onerank_r0$Z.log 2>&1
echo "rank0 rc=$?" >> $OUT/${TAG}_onerank_r0$Z.log
wait $P1; echo "rank1 rc=$?" >> $OUT/${TAG}_onerank_r1$Z.log
