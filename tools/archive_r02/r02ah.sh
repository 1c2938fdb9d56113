#!/bin/bash
# n=2: bulk-copy tile 16 KiB (default) vs 8 KiB vs the per-thread kernel, in-step pattern.
cd "$(dirname "$0")/.."
N=${1:-2}; TAG=${2:-r02ah}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_sweep_n$N.jsonl; : > $F
port=32300
for rep in 1 2; do
for cfg in "CM_AR_IMPL=0" "CM_AR_IMPL=2" "CM_AR_IMPL=2 CM_AR_TMA_TILE=8192" "CM_AR_IMPL=2 CM_AR_TMA_TILE=4096"; do
  port=$((port + 1))
  env $cfg CM_LAZY_EXIT_SWEEP=1 timeout 600 $RUN --master-port $port tools/sweep_allreduce.py --mode ours --multi-bucket \
    --min-mib 8 --max-mib 128 --reps 10 --burst 8 --tag "$cfg" >> $F 2>> $OUT/${TAG}_sweep.err
done
done
