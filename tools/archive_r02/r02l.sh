#!/bin/bash
# N GPUs: C5 kill points (incl. before the reduce-scatter and mid shadow step), then the C3
# bucket sweep with the current kernels (ours without tap, ours with the staged tap, NCCL).
cd "$(dirname "$0")/.."
N=${1:-2}; TAG=${2:-r02l}; OUT=gpurun_out
bash tools/run_c5_points.sh $N ${TAG}_c5
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_sweep_n$N.jsonl; : > $F
port=31200
for mode in ours ours_tap nccl; do
  port=$((port + 1))
  timeout 900 $RUN --master-port $port tools/sweep_allreduce.py --mode $mode --min-mib 1 --max-mib 1024 --reps 10 --burst 8 \
    --tag "r02 $mode" >> $F 2>> $OUT/${TAG}_sweep_n$N.err
done
# one iteration of 8 different buckets per timed rep (the in-step pattern: PDL overlap)
port=$((port + 1))
timeout 900 $RUN --master-port $port tools/sweep_allreduce.py --mode ours --multi-bucket --min-mib 1 --max-mib 512 \
  --reps 10 --burst 8 --tag "r02 ours multi-bucket" >> $F 2>> $OUT/${TAG}_sweep_n$N.err
