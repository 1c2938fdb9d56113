#!/bin/bash
# GPT-2 model mode at N GPUs, alternating A/B arms: per-bucket optimizer step on/off, and the
# single device->host queue (persist_queue) on/off.  Usage: tools/r02_model_ab.sh N TAG [REPS]
cd "$(dirname "$0")/.."
N=${1:-1}; TAG=${2:-r02f}; REPS=${3:-2}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_model_n$N.jsonl; : > $F
port=30800
for rep in $(seq $REPS); do
  for cfg in "CM_BUCKET_STEP=1 CM_PERSIST_QUEUE=0" "CM_BUCKET_STEP=0 CM_PERSIST_QUEUE=0" "CM_BUCKET_STEP=1 CM_PERSIST_QUEUE=1"; do
    port=$((port + 1))
    env $cfg timeout 900 $RUN --master-port $port tools/model_mode.py --steps 20 --warmup 5 >> $F 2>> $OUT/${TAG}_model_n$N.err
  done
done
