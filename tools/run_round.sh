#!/bin/bash
# Full evidence pass at N GPUs: GPU test suite, bench.py (default flags), model-mode decomposition.
cd "$(dirname "$0")/.."
N=$1; TAG=${2:-rr}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/${TAG}_tests.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_tests.log
if [ "$N" = "1" ]; then B="python"; else B="$RUN --master-port 29671"; fi
timeout 1200 $B bench.py --gpus $N --steps 20 --warmup 5 > $OUT/${TAG}_bench_n$N.json 2> $OUT/${TAG}_bench_n$N.err
echo "rc=$?" >> $OUT/${TAG}_bench_n$N.err
if [ "$N" = "1" ]; then M="python"; else M="$RUN --master-port 29672"; fi
timeout 900 $M tools/model_mode.py --steps 20 --warmup 5 --arms nccl,ours_nockpt,ours_tap_only,ours_ckpt > $OUT/${TAG}_model_n$N.json 2> $OUT/${TAG}_model_n$N.err
