#!/bin/bash
# Two-shot kernel variants at N: parity (multi-process) with ar_impl=1, then the bucket sweep
# (exit barriers on, as complete collectives) for ar_impl 0 / 1 (148 and 296 blocks).
cd "$(dirname "$0")/.."
N=$1; TAG=${2:-ai}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
CM_AR_IMPL=1 timeout 600 python -m pytest tests/test_gpu_multiproc.py -x -q -k "parity_f32 or parity_bf16 or zero1" > $OUT/${TAG}_mp_n$N.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_mp_n$N.log
F=$OUT/${TAG}_sweep_n$N.jsonl; rm -f $F
for cfg in "0 148" "1 148" "1 296"; do
  set -- $cfg
  CM_AR_IMPL=$1 CM_AR_PIPE_BLOCKS=$2 timeout 400 $RUN --master-port 29761 tools/sweep_allreduce.py --mode ours --min-kib 2048 --max-kib 262144 --reps 10 --burst 10 --oneshot-max 0 | sed "s/^{/{\"ar_impl\": $1, \"pipe_blocks\": $2, /" >> $F 2>> $OUT/${TAG}_sweep_n$N.err
done
