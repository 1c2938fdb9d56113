#!/bin/bash
# Fresh multi-GPU evidence at N: host facts, full bench.py (model mode, ZeRO-1 variant),
# then the C4 Llama-3-8B-shaped synthetic step (ZeRO-1, host shadow).  Usage: N TAG
cd "$(dirname "$0")/.."
N=$1; TAG=${2:-r}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
{ free -g; nproc; nvidia-smi topo -m; } > $OUT/${TAG}_host_n$N.txt 2>&1
timeout 1200 $RUN --master-port 29631 bench.py --gpus $N --steps 20 --warmup 5 > $OUT/${TAG}_bench_n$N.json 2> $OUT/${TAG}_bench_n$N.err
echo "rc=$?" >> $OUT/${TAG}_bench_n$N.err
timeout 1500 $RUN --master-port 29632 bench.py --gpus $N --workload llama8b --steps 5 --warmup 3 --ring-depth 4 --persist-every 4 --no-e2e --zero1 --no-model > $OUT/${TAG}_llama_n$N.json 2> $OUT/${TAG}_llama_n$N.err
echo "rc=$?" >> $OUT/${TAG}_llama_n$N.err
