#!/bin/bash
cd "$(dirname "$0")/.."
N=$1; TAG=${2:-c4}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
ARMS=nccl,ours_nockpt,nockpt_d2hload,ours_tap_nodrain,ours_tap_only,ours_ckpt timeout 1000 tools/run_decomp.sh $N $TAG
timeout 1500 $RUN --master-port 29643 tools/filler_mode.py --tokens 16384 --steps 5 --warmup 2 --ring-depth 8 --persist-every 8 > $OUT/${TAG}_filler_n$N.json 2> $OUT/${TAG}_filler_n$N.err
echo "rc=$?" >> $OUT/${TAG}_filler_n$N.err
