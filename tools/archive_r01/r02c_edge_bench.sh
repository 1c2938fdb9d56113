#!/bin/bash
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r02c}
timeout 900 python -m pytest tests/test_gpu_edge.py -q > $OUT/${TAG}_edge.log 2>&1
echo "edge rc=$?" >> $OUT/${TAG}_edge.log
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench rc=$?" >> $OUT/${TAG}_bench.err
