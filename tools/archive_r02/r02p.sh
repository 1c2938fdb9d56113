#!/bin/bash
# PDL trigger point A/B at n=2: lockstep chain (bench nockpt) and multi-bucket sweeps with exit
# barriers on and off, mode 0 (trigger after the entry barrier) vs 2 (after the data phase).
cd "$(dirname "$0")/.."
TAG=${1:-r02p}; OUT=gpurun_out; N=2
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
port=31500
for rep in 1 2; do
  for mode in 0 2; do
    port=$((port + 1))
    CM_PDL_MODE=$mode timeout 600 $RUN --master-port $port bench.py --gpus $N --steps 20 --warmup 5 --no-model --no-e2e \
      --no-variants --cpu-sample-s 0 > $OUT/${TAG}_bench_mode${mode}_$rep.json 2>> $OUT/${TAG}_bench.err
  done
done
F=$OUT/${TAG}_sweep.jsonl; : > $F
for lz in 1 0; do
  for mode in 2; do
    port=$((port + 1))
    echo "== lazy=$lz mode=$mode" >> $OUT/${TAG}_sweep.err
    CM_PDL_MODE=$mode CM_LAZY_EXIT_SWEEP=$lz timeout 400 $RUN --master-port $port tools/sweep_allreduce.py --mode ours --multi-bucket \
      --min-mib 1 --max-mib 256 --reps 10 --burst 8 --tag "lazy=$lz mode=$mode" >> $F 2>> $OUT/${TAG}_sweep.err
    echo "rc=$?" >> $OUT/${TAG}_sweep.err
  done
done
