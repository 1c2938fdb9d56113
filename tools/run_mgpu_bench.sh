#!/bin/bash
# Multi-GPU bench session (no sweep): multi-process tests, bench.py (with model mode) at N.
cd "$(dirname "$0")/.."
N=$1; TAG=${2:-}
OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > $OUT/mp_tests_n$N$TAG.log 2>&1
echo "mp tests rc=$?" >> $OUT/mp_tests_n$N$TAG.log
timeout 900 $RUN --master-port 29613 bench.py --gpus $N --steps 20 --warmup 5 > $OUT/bench_n$N$TAG.json 2> $OUT/bench_n$N$TAG.err
timeout 600 $RUN --master-port 29614 bench.py --gpus $N --steps 20 --warmup 5 --no-model --no-e2e --no-baseline --shadow device > $OUT/bench_n${N}${TAG}_dev.json 2>> $OUT/bench_n$N$TAG.err
free -g > $OUT/host_mem_n$N$TAG.txt; nvidia-smi topo -m >> $OUT/host_mem_n$N$TAG.txt
timeout 600 $RUN --master-port 29616 tools/restore_bench.py phase1 cmrb$N 7 > $OUT/restore_n$N$TAG.log 2>&1
timeout 900 $RUN --master-port 29617 tools/restore_bench.py phase2 cmrb$N 7 100 > $OUT/restore_n$N$TAG.json 2>> $OUT/restore_n$N$TAG.log
