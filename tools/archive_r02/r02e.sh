#!/bin/bash
# n GPUs: new multi-process tests, the lockstep PDL A/B (bench), NVLink ncu counters.
cd "$(dirname "$0")/.."
N=${1:-2}; TAG=${2:-r02e}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q > $OUT/${TAG}_mp_tests_n$N.log 2>&1
echo "mp tests rc=$?" >> $OUT/${TAG}_mp_tests_n$N.log
port=30600
for rep in 1 2; do
  for pdl in 0 1; do
    port=$((port + 1))
    CM_PDL=$pdl timeout 600 $RUN --master-port $port bench.py --gpus $N --steps 20 --warmup 5 --no-model --no-e2e \
      --no-variants --cpu-sample-s 0 > $OUT/${TAG}_bench_n${N}_pdl${pdl}_$rep.json 2>> $OUT/${TAG}_bench_n$N.err
  done
done
bash tools/r02_nvlink_ncu.sh $N $TAG
