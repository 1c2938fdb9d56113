#!/bin/bash
# Llama-3-8B-shaped synthetic bench line at N GPUs (BASELINE configs[3]), ZeRO-1, host shadow.
cd "$(dirname "$0")/.."
N=${1:-4}; OUT=gpurun_out; TAG=${2:-r01l}
timeout 1800 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 30071 bench.py --gpus $N --workload llama8b --steps 5 --warmup 3 --ring-depth 8 --persist-every 8 --no-e2e --zero1 --no-model > $OUT/${TAG}_llama_n$N.json 2> $OUT/${TAG}_llama_n$N.err
