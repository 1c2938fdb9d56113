#!/bin/bash
# GPU-timed step period for the drain policy, at N GPUs: link diagnosis (default), then the
# full bench line (model mode included).
cd "$(dirname "$0")/.."
N=${1:-4}; TAG=${2:-r01h}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_link_n$N.jsonl; : > $F
B="bench.py --gpus $N --steps 30 --warmup 5 --no-model --no-baseline --no-e2e --no-variants --cpu-sample-s 0.2"
timeout 600 $RUN --master-port 30041 $B >> $F 2>> $OUT/${TAG}_link_n$N.err
timeout 1200 $RUN --master-port 30042 bench.py --gpus $N --steps 20 --warmup 5 > $OUT/${TAG}_bench_n$N.json 2> $OUT/${TAG}_bench_n$N.err
