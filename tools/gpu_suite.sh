#!/bin/bash
# 1 GPU, current tree: the whole GPU suite, smoke, the default bench line.
cd "$(dirname "$0")/.."
TAG=${1:-r02v}; OUT=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $OUT/${TAG}_tests.log 2>&1
echo "gpu suite rc=$?" >> $OUT/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/${TAG}_smoke.log
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench rc=$?" >> $OUT/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/${TAG}_ref.json 2> $OUT/${TAG}_ref.err
echo "ref rc=$?" >> $OUT/${TAG}_ref.err
