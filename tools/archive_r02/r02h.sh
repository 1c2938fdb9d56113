#!/bin/bash
# 2 GPUs: multi-process suite, NVML NVLink counters (two-shot and ZeRO-1), one-rank ncu NVLink counters.
cd "$(dirname "$0")/.."
N=${1:-2}; TAG=${2:-r02h}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q > $OUT/${TAG}_mp_tests_n$N.log 2>&1
echo "mp tests rc=$?" >> $OUT/${TAG}_mp_tests_n$N.log
timeout 300 $RUN --master-port 30931 tools/nvlink_counters.py --steps 20 > $OUT/${TAG}_nvml_n$N.json 2> $OUT/${TAG}_nvml_n$N.err
timeout 300 $RUN --master-port 30932 tools/nvlink_counters.py --steps 20 --zero1 > $OUT/${TAG}_nvml_n${N}_zero1.json 2>> $OUT/${TAG}_nvml_n$N.err
if [ "$N" = "2" ]; then
  bash tools/r02_ncu_onerank.sh $TAG
  bash tools/r02_ncu_onerank.sh $TAG --zero1
fi
