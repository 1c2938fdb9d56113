#!/bin/bash
# ZeRO-1 with bulk-copy parameter all-gather (zero1_impl 2): parity on one GPU (virtual ranks)
# and across 4 GPUs (multi-process, NVLink), then an A/B of the kernel inside the GPT-2
# ZeRO-1 bench step (impl 1 vs 2, two reps).
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r01o}; N=${2:-4}
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "zero1" > $OUT/${TAG}_tests.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_tests.log
CM_ZERO1_IMPL=2 timeout 600 python -m pytest tests/test_gpu_sgd.py tests/test_gpu_parity.py -m gpu -x -q -k "zero1" > $OUT/${TAG}_tests_env2.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_tests_env2.log
grep -q "rc=0" $OUT/${TAG}_tests.log && grep -q "rc=0" $OUT/${TAG}_tests_env2.log || exit 1
CM_ZERO1_IMPL=2 timeout 900 python -m pytest tests/test_gpu_multiproc.py -m gpu -x -q -k "zero1" > $OUT/${TAG}_mp.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_mp.log
grep -q "rc=0" $OUT/${TAG}_mp.log || exit 1
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
for rep in 1 2; do
  for z in 1 2; do
    CM_ZERO1_IMPL=$z timeout 600 $RUN --master-port $((30100 + rep * 10 + z)) bench.py --gpus $N --zero1 --steps 20 --warmup 5 --no-model --no-e2e --no-variants --cpu-sample-s 0.2 > $OUT/${TAG}_z${z}_r${rep}.json 2> $OUT/${TAG}_z${z}_r${rep}.err
  done
done
