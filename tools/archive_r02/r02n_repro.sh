#!/bin/bash
# Regression of the PDL + exit-barrier deadlock (n=2, multi-bucket sweep at 8 MiB): the forced
# PDL case (pdl=2) must not trap with monotone barrier announcements; default pdl skips exits.
cd "$(dirname "$0")/.."
TAG=${1:-r02n}; OUT=gpurun_out; N=2
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
F=$OUT/${TAG}_repro.jsonl; : > $F
port=31400
for cfg in "CM_PDL=2" "CM_PDL=1" "CM_PDL=1 CM_LAZY_EXIT_SWEEP=1"; do
  port=$((port + 1))
  echo "== $cfg $(date +%s)" >> $OUT/${TAG}_repro.err
  env $cfg timeout 150 $RUN --master-port $port tools/sweep_allreduce.py --mode ours --multi-bucket --min-mib 1 --max-mib 64 \
    --reps 5 --burst 8 --tag "$cfg" >> $F 2>> $OUT/${TAG}_repro.err
  echo "rc=$? $(date +%s)" >> $OUT/${TAG}_repro.err
done
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -k "parity_f32 or parity_bf16 or parity_zero1 or restore_soft or model_parity" > $OUT/${TAG}_mp.log 2>&1
echo "mp rc=$?" >> $OUT/${TAG}_mp.log
for rep in 1; do
  port=$((port + 1))
  timeout 600 $RUN --master-port $port bench.py --gpus $N --steps 20 --warmup 5 --no-model --no-e2e \
      --no-variants --cpu-sample-s 0 > $OUT/${TAG}_bench.json 2>> $OUT/${TAG}_bench.err
done
