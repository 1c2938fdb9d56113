#!/bin/bash
# n=1 model mode A/B: the staging copy by a copy engine (n1_copy_engine) and K=16 snapshots.
cd "$(dirname "$0")/.."
TAG=${1:-r02r}; OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_checkpoint.py -q -k "n1_copy_engine" > $OUT/${TAG}_test.log 2>&1
echo "rc=$?" >> $OUT/${TAG}_test.log
F=$OUT/${TAG}_model_n1.jsonl; : > $F
for rep in 1 2; do
  CM_N1_COPY_ENGINE=0 timeout 900 python tools/model_mode.py --steps 20 --warmup 5 >> $F 2>> $OUT/${TAG}.err
  CM_N1_COPY_ENGINE=1 timeout 900 python tools/model_mode.py --steps 20 --warmup 5 >> $F 2>> $OUT/${TAG}.err
  CM_N1_COPY_ENGINE=1 timeout 900 python tools/model_mode.py --steps 20 --warmup 5 --persist-every 16 --ring-depth 17 \
    --arms ours_ckpt >> $F 2>> $OUT/${TAG}.err
done
