#!/bin/bash
# Checkpoint-cost decomposition in GPT-2 model mode, the C4 Llama filler run, and a quick
# bench line at N.  Usage: tools/run_n4_model.sh N TAG
cd "$(dirname "$0")/.."
N=$1; TAG=${2:-mm}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 $RUN --master-port 29641 tools/model_mode.py --steps 20 --warmup 5 --arms nccl,ours_nockpt,ours_tap_only,ours_ckpt > $OUT/${TAG}_model_n$N.json 2> $OUT/${TAG}_model_n$N.err
timeout 600 $RUN --master-port 29642 tools/model_mode.py --steps 20 --warmup 5 --arms ours_ckpt --persist-every 16 --ring-depth 16 > $OUT/${TAG}_model_k16_n$N.json 2>> $OUT/${TAG}_model_n$N.err
timeout 1500 $RUN --master-port 29643 tools/filler_mode.py --tokens 16384 --steps 5 --warmup 2 --ring-depth 8 --persist-every 8 > $OUT/${TAG}_filler_n$N.json 2> $OUT/${TAG}_filler_n$N.err
echo "rc=$?" >> $OUT/${TAG}_filler_n$N.err
timeout 600 $RUN --master-port 29644 bench.py --gpus $N --steps 20 --warmup 5 --no-model --no-variants > $OUT/${TAG}_bench_n$N.json 2> $OUT/${TAG}_bench_n$N.err
