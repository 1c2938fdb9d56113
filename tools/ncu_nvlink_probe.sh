#!/bin/bash
# ncu NVLink counters of the all-reduce kernels (one process, 2 GPUs, barriers off) and of the
# ZeRO-1 AdamW + parameter all-gather.  The plain command first, then ncu.
cd "$(dirname "$0")/.."
TAG=${1:-r02ao}; OUT=gpurun_out
M=gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
for impl in -1 0; do
  P="python tools/ncu_nvlink_probe.py --n 2 --impl $impl"
  timeout 300 $P > $OUT/${TAG}_plain_impl$impl.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -k regex:"rs_tap_ag" --csv --log-file $OUT/${TAG}_nvl_impl$impl.csv $P > $OUT/${TAG}_ncu_impl$impl.log 2>&1
  echo "rc=$?" >> $OUT/${TAG}_ncu_impl$impl.log
done
P="python tools/ncu_nvlink_probe.py --n 2 --zero1"
timeout 300 $P > $OUT/${TAG}_plain_zero1.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -k regex:"rs_tap_ag|adamw_zero1" --csv --log-file $OUT/${TAG}_nvl_zero1.csv $P > $OUT/${TAG}_ncu_zero1.log 2>&1
echo "rc=$?" >> $OUT/${TAG}_ncu_zero1.log
