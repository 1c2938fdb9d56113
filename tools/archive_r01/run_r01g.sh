#!/bin/bash
# Drain policy with the backlog rule, at N GPUs: link diagnosis (default x2, device shadow),
# then the full bench line (model mode included).
cd "$(dirname "$0")/.."
N=${1:-4}; TAG=${2:-r01g}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_link_n$N.jsonl; : > $F
B="bench.py --gpus $N --steps 30 --warmup 5 --no-model --no-baseline --no-e2e --no-variants --cpu-sample-s 0.2"
port=30010
run() { port=$((port + 1)); local v=$1; shift; echo "{\"variant\": \"$v\"}" >> $F; timeout 600 $RUN --master-port $port $B "$@" >> $F 2>> $OUT/${TAG}_link_n$N.err; }
run default
run default_again
run device_shadow --shadow device
timeout 1200 $RUN --master-port 30031 bench.py --gpus $N --steps 20 --warmup 5 > $OUT/${TAG}_bench_n$N.json 2> $OUT/${TAG}_bench_n$N.err
