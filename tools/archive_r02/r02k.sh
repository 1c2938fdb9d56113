#!/bin/bash
# 1 GPU: the round-2 GPU tests after the device-word report, the shadow/training AdamW per-launch
# durations, and the bench default line.
cd "$(dirname "$0")/.."
TAG=${1:-r02k}; OUT=gpurun_out
timeout 1800 python -m pytest tests/test_gpu_edge.py tests/test_gpu_bucket_step.py tests/test_gpu_checkpoint.py tests/test_gpu_ddp.py -q > $OUT/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> $OUT/${TAG}_tests.log
TGT="python tools/prof_target.py --steps 3 --ring-depth 16 --persist-every 8"
$TGT > $OUT/${TAG}_prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"rs_tap_ag|adamw_wt|gen_grads" --csv --log-file $OUT/${TAG}_dram.csv $TGT > $OUT/${TAG}_dram.log 2>&1
echo "dram rc=$?" >> $OUT/${TAG}_dram.log
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench rc=$?" >> $OUT/${TAG}_bench.err
