#!/bin/bash
# C3 bucket sweep with the current kernels at N GPUs: ours without tap, ours with the staged
# tap, NCCL default -- fp32 and bf16.
cd "$(dirname "$0")/.."
N=${1:-2}; TAG=${2:-r01q}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_sweep_n$N.jsonl; : > $F
port=30200
for dt in f32 bf16; do
  for mode in ours ours_tap nccl; do
    port=$((port + 1))
    timeout 600 $RUN --master-port $port tools/sweep_allreduce.py --mode $mode --dtype $dt --max-mib 1024 --reps 10 >> $F 2>> $OUT/${TAG}_sweep_n$N.err
  done
done
