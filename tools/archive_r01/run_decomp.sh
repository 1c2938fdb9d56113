#!/bin/bash
# Checkpoint-cost decomposition in GPT-2 model mode at N: nccl, ours_nockpt, nockpt + a plain
# D2H load of the tap's bytes, tap without drain, tap only, full checkpoint (K=8, K=16).
cd "$(dirname "$0")/.."
N=$1; TAG=${2:-dc}; OUT=gpurun_out
if [ "$N" = "1" ]; then RUN="python"; else RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29651"; fi
timeout 1200 $RUN tools/model_mode.py --steps 20 --warmup 5 --arms ${ARMS:-nccl,ours_nockpt,nockpt_d2hload,ours_tap_nodrain,ours_tap_only,ours_ckpt} > $OUT/${TAG}_decomp_n$N.json 2> $OUT/${TAG}_decomp_n$N.err
timeout 600 $RUN tools/model_mode.py --steps 20 --warmup 5 --arms ours_ckpt --persist-every 16 --ring-depth 16 >> $OUT/${TAG}_decomp_n$N.json 2>> $OUT/${TAG}_decomp_n$N.err
