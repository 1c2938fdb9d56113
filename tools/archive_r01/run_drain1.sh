#!/bin/bash
cd "$(dirname "$0")/.."
TAG=${1:-dr}; OUT=gpurun_out; F=$OUT/${TAG}_drain_n1.json; rm -f $F
timeout 600 python tools/model_mode.py --steps 20 --warmup 5 --arms nccl,ours_nockpt >> $F 2> $OUT/${TAG}.err
for k in 0 1 2 3; do
  timeout 400 python tools/model_mode.py --steps 20 --warmup 5 --arms ours_ckpt --drain-ctas $k >> $F 2>> $OUT/${TAG}.err
done
