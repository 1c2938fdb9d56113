#!/bin/bash
# Multi-GPU session: multi-process parity tests, C3 bucket sweep (ours with/without tap,
# NCCL default and NVLS off), and bench.py at N GPUs.  Usage: tools/run_mgpu.sh N [max_mib]
cd "$(dirname "$0")/.."
N=$1; MAXMIB=${2:-1024}
OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_multiproc.py -x -q > $OUT/mp_tests_n$N.log 2>&1
echo "mp tests rc=$?" >> $OUT/mp_tests_n$N.log
for mode in ours_tap ours nccl; do
  timeout 600 $RUN --master-port 29611 tools/sweep_allreduce.py --mode $mode --max-mib $MAXMIB >> $OUT/sweep_n$N.jsonl 2>> $OUT/sweep_n$N.err
done
NCCL_NVLS_ENABLE=0 timeout 600 $RUN --master-port 29612 tools/sweep_allreduce.py --mode nccl --max-mib $MAXMIB >> $OUT/sweep_n$N.jsonl 2>> $OUT/sweep_n$N.err
timeout 600 $RUN --master-port 29613 bench.py --gpus $N --steps 10 --warmup 3 > $OUT/bench_n$N.json 2> $OUT/bench_n$N.err
timeout 600 $RUN --master-port 29614 bench.py --gpus $N --steps 10 --warmup 3 --shadow device --no-e2e > $OUT/bench_n${N}_dev.json 2>> $OUT/bench_n$N.err
