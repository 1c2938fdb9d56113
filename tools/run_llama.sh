#!/bin/bash
# C4: Llama-3-8B-shaped gradients (bf16 grads, fp32 AdamW state, 226 buckets), host shadow.
cd "$(dirname "$0")/.."
N=$1; OUT=gpurun_out
free -g > $OUT/llama_n$N.mem; nvidia-smi --query-gpu=memory.total --format=csv >> $OUT/llama_n$N.mem
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1500 $RUN --master-port 29621 bench.py --gpus $N --workload llama8b --steps 5 --warmup 2 --ring-depth 5 --persist-every 4 --no-e2e --cpu-sample-s 2 > $OUT/llama_n$N.json 2> $OUT/llama_n$N.err
echo "rc=$?" >> $OUT/llama_n$N.err
