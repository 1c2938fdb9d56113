#!/bin/bash
# Host-link diagnosis of the checkpointed synthetic step at N GPUs: busy time and per-copy
# rate of the tap drains and snapshot persists (kernels.host_link_busy), for the default
# configuration and three variations.
cd "$(dirname "$0")/.."
N=${1:-4}; TAG=${2:-r01f_link}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_n$N.jsonl; : > $F
B="bench.py --gpus $N --steps 30 --warmup 5 --no-model --no-baseline --no-e2e --no-variants --cpu-sample-s 0.2"
port=29990
run() { port=$((port + 1)); local v=$1; local e=$2; shift 2; echo "{\"variant\": \"$v\"}" >> $F; env $e timeout 600 $RUN --master-port $port $B "$@" >> $F 2>> $OUT/${TAG}_n$N.err; }
run default X=1
run flush64 CM_DRAIN_FLUSH_BYTES=67108864
run device_shadow X=1 --shadow device
run k16 X=1 --persist-every 16 --ring-depth 32
