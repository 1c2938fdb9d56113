#!/bin/bash
# NVLink evidence from ncu for the all-reduce (rs_tap_ag) and the ZeRO-1 AdamW + parameter
# all-gather (adamw_zero1) at N GPUs: one multi-rank command under ncu --target-processes all,
# a few counters only (nvlrx/nvltx bytes, duration, DRAM bytes).  The kernels' cross-GPU
# barriers pass under replay (epoch flags are ">="), and a barrier that never completes traps
# after ~30 s instead of hanging.  The same command first runs without ncu.
cd "$(dirname "$0")/.."
N=${1:-2}; TAG=${2:-r02e}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
M=gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,nvltx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
for z in "" "--zero1"; do
  zt=${z:+_zero1}
  CMD="tools/ncu_target_mp.py --steps 2 $z"
  timeout 300 $RUN --master-port 30711 $CMD > $OUT/${TAG}_nvl_plain_n${N}${zt}.log 2>&1
  echo "plain rc=$?" >> $OUT/${TAG}_nvl_plain_n${N}${zt}.log
  timeout 900 ncu --target-processes all --metrics $M --clock-control none -k regex:"rs_tap_ag|adamw_zero1" \
     --csv --log-file $OUT/${TAG}_nvl_n${N}${zt}.csv $RUN --master-port 30712 $CMD > $OUT/${TAG}_nvl_ncu_n${N}${zt}.log 2>&1
  echo "ncu rc=$?" >> $OUT/${TAG}_nvl_ncu_n${N}${zt}.log
done
