#!/bin/bash
# Model-mode checkpoint overhead with the copy-engine drain vs the SM drain (1, 2, 4 CTAs).
cd "$(dirname "$0")/.."
N=$1; TAG=${2:-dr}; OUT=gpurun_out
if [ "$N" = "1" ]; then RUN="python"; else RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29661"; fi
F=$OUT/${TAG}_drain_n$N.json; rm -f $F
timeout 600 $RUN tools/model_mode.py --steps 20 --warmup 5 --arms nccl,ours_nockpt,ours_ckpt >> $F 2> $OUT/${TAG}_drain_n$N.err
for k in 1 2 4; do
  timeout 400 $RUN tools/model_mode.py --steps 20 --warmup 5 --arms ours_tap_only,ours_ckpt --drain-ctas $k >> $F 2>> $OUT/${TAG}_drain_n$N.err
done
timeout 600 $RUN tools/model_mode.py --steps 20 --warmup 5 --arms nccl,ours_ckpt >> $F 2>> $OUT/${TAG}_drain_n$N.err
