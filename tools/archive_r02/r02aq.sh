#!/bin/bash
# n=4: bulk-copy tile 8 KiB (default) vs 4 KiB: step-pattern sweep and the lockstep GPT-2 chain.
cd "$(dirname "$0")/.."
N=${1:-4}; TAG=${2:-r02aq}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_sweep_n$N.jsonl; : > $F
port=32500
for cfg in "CM_AR_TMA_TILE=8192" "CM_AR_TMA_TILE=4096" "CM_AR_TMA_TILE=6144"; do
  port=$((port + 1))
  env $cfg CM_AR_IMPL=2 CM_LAZY_EXIT_SWEEP=1 timeout 600 $RUN --master-port $port tools/sweep_allreduce.py --mode ours --multi-bucket \
    --min-mib 8 --max-mib 64 --reps 10 --burst 8 --tag "$cfg" >> $F 2>> $OUT/${TAG}_sweep.err
done
for rep in 1 2; do
  for tile in 8192 4096; do
    port=$((port + 1))
    CM_AR_TMA_TILE=$tile timeout 600 $RUN --master-port $port bench.py --gpus $N --steps 20 --warmup 5 --no-model --no-e2e \
      --no-variants --cpu-sample-s 0 > $OUT/${TAG}_bench_tile${tile}_$rep.json 2>> $OUT/${TAG}_bench.err
  done
done
