#!/bin/bash
# Round-1d A/B on a 4-GPU box: AdamW single-tile variant (impl 3) vs warp-tiled pairs
# (impl 2), ZeRO-1 AdamW+AG with two groups per thread in flight (zero1_impl 1) vs one (0);
# parity of both first.
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r01d_ab}; N=${2:-4}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_numa.py -m gpu -x -q -k "implementations or zero1 or numa" > $OUT/${TAG}_tests.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_tests.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -m gpu -x -q -k "zero1" > $OUT/${TAG}_mp_tests.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_mp_tests.log
timeout 300 python tools/microbench.py adamw_wt adamw_wt1 adamw_bf16_wt adamw_bf16_wt1 adamw_wt adamw_wt1 adamw_bf16_wt adamw_bf16_wt1 > $OUT/${TAG}_mb.jsonl 2> $OUT/${TAG}_mb.err
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
for rep in 1 2; do
  for z in 0 1; do
    CM_ZERO1_IMPL=$z timeout 600 $RUN --master-port $((29800 + rep * 10 + z)) bench.py --gpus $N --zero1 --steps 20 --warmup 5 --no-model --no-e2e --no-variants --cpu-sample-s 0.2 > $OUT/${TAG}_z${z}_r${rep}.json 2> $OUT/${TAG}_z${z}_r${rep}.err
  done
done
