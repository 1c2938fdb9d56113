#!/bin/bash
# Round-1d: zero-operand fast path of the AdamW divisions (parity + microbench), and the
# bench line with the prefetched e2e inputs.
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r01d_z}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sgd.py -m gpu -x -q > $OUT/${TAG}_tests.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_tests.log
timeout 300 python tools/microbench.py adamw_wt adamw_bf16_wt adamw_wt adamw_bf16_wt > $OUT/${TAG}_mb.jsonl 2> $OUT/${TAG}_mb.err
timeout 1200 python bench.py --steps 20 --warmup 5 > $OUT/${TAG}_bench_n1.json 2> $OUT/${TAG}_bench_n1.err; echo "rc=$?" >> $OUT/${TAG}_bench_n1.err
