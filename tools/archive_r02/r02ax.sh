#!/bin/bash
# 1 GPU: n=1 staging-copy chain with and without PDL (bench isolated pass, chain timing)
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r02ax}
B="python bench.py --steps 20 --warmup 5 --no-baseline --no-e2e --no-model --cpu-sample-s 0"
for rep in 1 2; do
  CM_PDL=0 timeout 300 $B > $OUT/${TAG}_pdl0_$rep.json 2>> $OUT/${TAG}_bench.err
  CM_PDL=1 timeout 300 $B > $OUT/${TAG}_pdl1_$rep.json 2>> $OUT/${TAG}_bench.err
done
