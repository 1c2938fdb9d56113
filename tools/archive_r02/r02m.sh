#!/bin/bash
# 4 GPUs: C4 Llama-3-8B-shaped ZeRO-1 + compute filler T sweep (per-bucket steps; A/B at 16k),
# then the Llama synthetic bench line (BASELINE configs[3]).
cd "$(dirname "$0")/.."
N=${1:-4}; TAG=${2:-r02m}; OUT=gpurun_out
free -g > $OUT/${TAG}_mem.txt 2>&1
bash tools/run_c4_sweep.sh $N ${TAG}_c4
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1500 $RUN --master-port 31301 bench.py --gpus $N --workload llama8b --zero1 --steps 5 --warmup 3 --ring-depth 9 \
  --persist-every 8 --no-e2e --no-model --cpu-sample-s 0 > $OUT/${TAG}_llama_n$N.json 2> $OUT/${TAG}_llama_n$N.err
echo "rc=$?" >> $OUT/${TAG}_llama_n$N.err
