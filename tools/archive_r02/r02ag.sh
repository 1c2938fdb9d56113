#!/bin/bash
# Bulk-copy all-reduce tuning at N GPUs: parity of the variants (virtual ranks, 1 GPU of the box)
# then the in-step-pattern sweep (8 buckets per iteration, lazy exits, PDL) per (stages, tile).
cd "$(dirname "$0")/.."
N=${1:-4}; TAG=${2:-r02ag}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
for cfg in "CM_AR_TMA_STAGES=3" "CM_AR_TMA_TILE=4096" "CM_AR_TMA_STAGES=3 CM_AR_TMA_TILE=16384"; do
  env $cfg timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "pipelined_allreduce and -2]" >> $OUT/${TAG}_parity.log 2>&1
  echo "$cfg rc=$?" >> $OUT/${TAG}_parity.log
done
F=$OUT/${TAG}_sweep_n$N.jsonl; : > $F
port=32200
for cfg in "CM_AR_IMPL=0" "CM_AR_IMPL=2" "CM_AR_IMPL=2 CM_AR_TMA_STAGES=3" "CM_AR_IMPL=2 CM_AR_TMA_TILE=16384" \
           "CM_AR_IMPL=2 CM_AR_TMA_STAGES=3 CM_AR_TMA_TILE=16384" "CM_AR_IMPL=2 CM_AR_TMA_TILE=8192" \
           "CM_AR_IMPL=2 CM_AR_TMA_STAGES=3 CM_AR_TMA_TILE=8192"; do
  port=$((port + 1))
  env $cfg CM_LAZY_EXIT_SWEEP=1 timeout 600 $RUN --master-port $port tools/sweep_allreduce.py --mode ours --multi-bucket \
    --min-mib 8 --max-mib 256 --reps 10 --burst 8 --tag "$cfg" >> $F 2>> $OUT/${TAG}_sweep.err
done
