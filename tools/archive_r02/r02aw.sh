#!/bin/bash
# 1 GPU: PDL for the n=1 staging copies -- parity files, then bench A/B of the isolated chain.
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r02aw}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_checkpoint.py tests/test_gpu_edge.py \
  tests/test_gpu_bucket_step.py tests/test_gpu_ddp.py tests/test_gpu_serving.py -q -x > $OUT/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> $OUT/${TAG}_tests.log
B="python bench.py --steps 20 --warmup 5 --no-baseline --no-e2e --no-model --cpu-sample-s 0"
for rep in 1 2; do
  CM_PDL=0 timeout 300 $B > $OUT/${TAG}_pdl0_$rep.json 2>> $OUT/${TAG}_bench.err
  CM_PDL=1 timeout 300 $B > $OUT/${TAG}_pdl1_$rep.json 2>> $OUT/${TAG}_bench.err
  CM_PDL=1 CM_AR_BLOCKS=296 timeout 300 $B > $OUT/${TAG}_pdl1_b296_$rep.json 2>> $OUT/${TAG}_bench.err
done
