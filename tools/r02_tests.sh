#!/bin/bash
# GPU suite on one B200: the new checkpoint/edge tests first, then everything.
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r02b}
timeout 1200 python -m pytest tests/test_gpu_edge.py tests/test_gpu_checkpoint.py -q -x > $OUT/${TAG}_new_tests.log 2>&1
echo "new tests rc=$?" >> $OUT/${TAG}_new_tests.log
timeout 2400 python -m pytest tests -m gpu -q > $OUT/${TAG}_tests.log 2>&1
echo "gpu suite rc=$?" >> $OUT/${TAG}_tests.log
