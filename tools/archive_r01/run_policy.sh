#!/bin/bash
# The drain auto policy at N: GPT-2 model mode and the C4 Llama filler, all arms.
cd "$(dirname "$0")/.."
N=$1; TAG=${2:-po}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 $RUN --master-port 29701 tools/model_mode.py --steps 20 --warmup 5 --arms nccl,ours_nockpt,ours_ckpt > $OUT/${TAG}_model_n$N.json 2> $OUT/${TAG}_model_n$N.err
timeout 1200 $RUN --master-port 29702 tools/filler_mode.py --tokens 16384 --steps 5 --warmup 2 --ring-depth 8 --persist-every 8 > $OUT/${TAG}_filler_n$N.json 2> $OUT/${TAG}_filler_n$N.err
