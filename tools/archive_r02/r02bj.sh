#!/bin/bash
# 4 GPUs: balanced bulk-copy partition -- multi-process parity with the bulk-copy kernel on
# every bucket, then the lockstep all-reduce at n=4 and n=2 (bench, no model / e2e).
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r02bj}
CM_AR_TMA_MIN_BYTES=0 timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -x \
  -k "parity_f32 or parity_bf16 or parity_zero1 or model_parity" > $OUT/${TAG}_mp_tma_tests.log 2>&1
echo "rc=$?" >> $OUT/${TAG}_mp_tma_tests.log
B="bench.py --steps 20 --warmup 5 --no-model --no-e2e --no-variants --cpu-sample-s 0"
timeout 400 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 31790 $B --gpus 4 > $OUT/${TAG}_bench_n4.json 2> $OUT/${TAG}_bench_n4.err
timeout 400 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 31791 $B --gpus 2 > $OUT/${TAG}_bench_n2.json 2> $OUT/${TAG}_bench_n2.err
