#!/bin/bash
# ar_impl 2 (bulk-copy pipeline): parity on one GPU first (virtual ranks), then at N GPUs the
# multi-process parity with ar_impl 2, the bucket sweep (in-step pattern) and the lockstep chain A/B.
cd "$(dirname "$0")/.."
N=${1:-2}; TAG=${2:-r02ac}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "pipelined_allreduce" > $OUT/${TAG}_parity.log 2>&1
echo "rc=$?" >> $OUT/${TAG}_parity.log
grep -q "rc=0" $OUT/${TAG}_parity.log || exit 1
CM_AR_IMPL=2 timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -k "parity_f32 or parity_bf16 or parity_zero1 and not oneshot" > $OUT/${TAG}_mp.log 2>&1
echo "rc=$?" >> $OUT/${TAG}_mp.log
F=$OUT/${TAG}_sweep.jsonl; : > $F
port=32100
for impl in 0 2; do
  port=$((port + 1))
  CM_AR_IMPL=$impl CM_LAZY_EXIT_SWEEP=1 timeout 600 $RUN --master-port $port tools/sweep_allreduce.py --mode ours --multi-bucket \
    --min-mib 4 --max-mib 256 --reps 10 --burst 8 --tag "impl=$impl multi" >> $F 2>> $OUT/${TAG}_sweep.err
  port=$((port + 1))
  CM_AR_IMPL=$impl timeout 600 $RUN --master-port $port tools/sweep_allreduce.py --mode ours \
    --min-mib 64 --max-mib 1024 --reps 10 --burst 4 --tag "impl=$impl single" >> $F 2>> $OUT/${TAG}_sweep.err
done
for impl in 0 2; do
  port=$((port + 1))
  CM_AR_IMPL=$impl timeout 600 $RUN --master-port $port bench.py --gpus $N --steps 20 --warmup 5 --no-model --no-e2e \
      --no-variants --cpu-sample-s 0 > $OUT/${TAG}_bench_impl$impl.json 2>> $OUT/${TAG}_bench.err
done
