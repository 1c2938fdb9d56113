#!/bin/bash
# Llama-3-8B-shaped ZeRO-1 with a calibrated compute filler, T_tok sweep at N
# GPUs (NCCL no-ckpt, ours no-ckpt, ours + per-iteration checkpoint; host shadow K=8, D=9).
cd "$(dirname "$0")/.."
N=${1:-4}; TAG=${2:-r01f_c4}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_sweep_n$N.jsonl; : > $F
port=29950
for T in ${TOKENS:-4096 8192 16384 32768}; do
  port=$((port + 1))
  timeout 1200 $RUN --master-port $port tools/filler_mode.py --tokens $T --steps 3 --warmup 2 --ring-depth 9 --persist-every 8 >> $F 2>> $OUT/${TAG}_sweep_n$N.err
done
# A/B at 16k tokens: one optimizer kernel after the last bucket (round 1) vs per-bucket steps
port=$((port + 1))
CM_BUCKET_STEP=0 timeout 1200 $RUN --master-port $port tools/filler_mode.py --tokens 16384 --steps 3 --warmup 2 --ring-depth 9 --persist-every 8 >> $F 2>> $OUT/${TAG}_sweep_n$N.err
