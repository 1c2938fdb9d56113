#!/bin/bash
# C4 filler runs at N: auto drain (all arms), then ours_ckpt with 1 and 2 SM-drain CTAs and K=16.
cd "$(dirname "$0")/.."
N=$1; TAG=${2:-c4}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_filler_n$N.jsonl; rm -f $F
timeout 900 $RUN --master-port 29691 tools/filler_mode.py --tokens 16384 --steps 5 --warmup 2 --ring-depth 8 --persist-every 8 >> $F 2> $OUT/${TAG}_filler_n$N.err
timeout 600 $RUN --master-port 29692 tools/filler_mode.py --tokens 16384 --steps 5 --warmup 2 --ring-depth 8 --persist-every 8 --arms ours_ckpt --drain-ctas 2 >> $F 2>> $OUT/${TAG}_filler_n$N.err
timeout 600 $RUN --master-port 29693 tools/filler_mode.py --tokens 16384 --steps 5 --warmup 2 --ring-depth 16 --persist-every 16 --arms ours_ckpt >> $F 2>> $OUT/${TAG}_filler_n$N.err
