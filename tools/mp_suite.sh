#!/bin/bash
# N GPUs: multi-process suite + the full default bench line (model mode, ZeRO-1 variant).
cd "$(dirname "$0")/.."
N=${1:-2}; TAG=${2:-r02s}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1800 python -m pytest tests/test_gpu_multiproc.py -q > $OUT/${TAG}_mp_tests_n$N.log 2>&1
echo "mp tests rc=$?" >> $OUT/${TAG}_mp_tests_n$N.log
timeout 1200 $RUN --master-port 31601 bench.py --gpus $N > $OUT/${TAG}_bench_n$N.json 2> $OUT/${TAG}_bench_n$N.err
echo "bench rc=$?" >> $OUT/${TAG}_bench_n$N.err
