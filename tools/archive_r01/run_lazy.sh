#!/bin/bash
# Lazy all-reduce exits at N: multi-process parity, then the no-checkpoint step A/B.
cd "$(dirname "$0")/.."
N=$1; TAG=${2:-lz}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > $OUT/${TAG}_mp_n$N.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_mp_n$N.log
for lz in 1 0 1; do
  CM_LAZY_EXIT=$lz timeout 600 $RUN --master-port 2973$lz bench.py --gpus $N --steps 30 --warmup 5 --no-model --no-variants --no-e2e > $OUT/${TAG}_bench_lz${lz}_n$N.json 2>> $OUT/${TAG}_bench_n$N.err
  cat $OUT/${TAG}_bench_lz${lz}_n$N.json >> $OUT/${TAG}_bench_all_n$N.jsonl
done
