#!/bin/bash
# Multi-GPU ZeRO-1 session: multi-process tests, bench.py --zero1 (with model mode).
cd "$(dirname "$0")/.."
N=$1; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > $OUT/mp_tests_n${N}_z.log 2>&1
echo "mp tests rc=$?" >> $OUT/mp_tests_n${N}_z.log
timeout 900 $RUN --master-port 29631 bench.py --gpus $N --steps 20 --warmup 5 --zero1 > $OUT/bench_n${N}_zero1.json 2> $OUT/bench_n${N}_zero1.err
timeout 1500 $RUN --master-port 29632 bench.py --gpus $N --workload llama8b --steps 5 --warmup 2 --ring-depth 4 --persist-every 4 --no-e2e --zero1 > $OUT/llama_n${N}_zero1.json 2>> $OUT/bench_n${N}_zero1.err
