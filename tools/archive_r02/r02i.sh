#!/bin/bash
# 1 GPU: whole GPU suite, smoke, the ncu recipe (launch list, per-launch DRAM, --set full),
# bench default line, model-mode A/B (per-bucket step, single D2H queue).
cd "$(dirname "$0")/.."
TAG=${1:-r02i}; OUT=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $OUT/${TAG}_tests.log 2>&1
echo "gpu suite rc=$?" >> $OUT/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/${TAG}_smoke.log
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench rc=$?" >> $OUT/${TAG}_bench.err
bash tools/r02_ncu.sh $TAG
python tools/traffic_from_ncu.py $OUT/${TAG}_dram.csv $OUT/${TAG}_traffic.json > $OUT/${TAG}_traffic.log 2>&1
bash tools/r02_model_ab.sh 1 $TAG 2
