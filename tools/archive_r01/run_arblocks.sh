#!/bin/bash
# All-reduce grid cap A/B on GPT-2-sized buckets (16-64 MiB), bursts of 8 launches, N GPUs.
cd "$(dirname "$0")/.."
N=${1:-2}; TAG=${2:-r01t_arblocks}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_n$N.jsonl; : > $F
port=30300
for rep in 1 2; do
  for ab in 0 148 296 444; do
    port=$((port + 1))
    timeout 300 $RUN --master-port $port tools/sweep_allreduce.py --mode ours --min-mib 16 --max-mib 64 --burst 8 --reps 10 --ar-blocks $ab >> $F 2>> $OUT/${TAG}_n$N.err
  done
done
