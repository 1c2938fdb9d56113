#!/bin/bash
# Last check of the final tree on one GPU: the GPU suite and smoke.
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r01r}
timeout 1200 python -m pytest tests -m gpu -q > $OUT/${TAG}_tests_n1.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_tests_n1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_smoke.log
