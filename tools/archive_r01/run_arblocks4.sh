#!/bin/bash
# All-reduce grid cap A/B at 4 GPUs: default vs one 512-thread block per SM, 16-128 MiB.
cd "$(dirname "$0")/.."
OUT=gpurun_out; F=$OUT/r01t_arblocks_n4.jsonl; : > $F
RUN="python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1"
port=30400
for ab in 0 148; do
  port=$((port + 1))
  timeout 300 $RUN --master-port $port tools/sweep_allreduce.py --mode ours --min-mib 16 --max-mib 128 --burst 8 --reps 8 --ar-blocks $ab >> $F 2>> $OUT/r01t_arblocks_n4.err
done
