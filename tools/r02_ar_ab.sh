#!/bin/bash
# All-reduce A/B on N GPUs: PDL on/off x size-dependent grid on/off (bursts of 8 launches,
# 8-128 MiB, exit barriers on), then the lockstep GPT-2 no-checkpoint step (bench nockpt_ours)
# with PDL on/off, then the multi-process parity suite.  Usage: tools/r02_ar_ab.sh N TAG
cd "$(dirname "$0")/.."
N=${1:-2}; TAG=${2:-r02d}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x > $OUT/${TAG}_mp_tests_n$N.log 2>&1
echo "mp tests rc=$?" >> $OUT/${TAG}_mp_tests_n$N.log
F=$OUT/${TAG}_arab_n$N.jsonl; : > $F
port=30500
for rep in 1 2; do
  for pdl in 0 1; do
    for sw in 0 50331648; do
      port=$((port + 1))
      CM_PDL=$pdl CM_AR_GRID_SWITCH_BYTES=$sw timeout 300 $RUN --master-port $port tools/sweep_allreduce.py --mode ours \
        --min-mib 8 --max-mib 128 --burst 8 --reps 10 --tag "pdl=$pdl,switch=$sw" >> $F 2>> $OUT/${TAG}_arab_n$N.err
    done
  done
done
for rep in 1 2; do
  for pdl in 0 1; do
    port=$((port + 1))
    CM_PDL=$pdl timeout 600 $RUN --master-port $port bench.py --gpus $N --steps 20 --warmup 5 --no-model --no-e2e \
      --no-variants --cpu-sample-s 0 > $OUT/${TAG}_bench_n${N}_pdl${pdl}_$rep.json 2>> $OUT/${TAG}_bench_n$N.err
  done
done
echo done >> $OUT/${TAG}_arab_n$N.err
