#!/bin/bash
# f2 session at N GPUs: multi-process parity of the one-shot path, then the small-bucket
# sweep (16 KiB - 4 MiB) two-shot vs one-shot vs NCCL.  Usage: tools/run_oneshot.sh N [tag]
cd "$(dirname "$0")/.."
N=$1; TAG=${2:-os}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
[ -z "$3" ] && timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -k "oneshot or sgd or nvls" > $OUT/${TAG}_mp_n$N.log 2>&1
echo "mp tests rc=$?" >> $OUT/${TAG}_mp_n$N.log
F=$OUT/${TAG}_sweep_n$N.jsonl; rm -f $F
for dt in f32 bf16; do
  timeout 300 $RUN --master-port 29621 tools/sweep_allreduce.py --mode ours --dtype $dt --min-kib 16 --max-kib 4096 --oneshot-max 0 --reps 20 --burst 50 >> $F 2>> $OUT/${TAG}_sweep_n$N.err
  timeout 300 $RUN --master-port 29622 tools/sweep_allreduce.py --mode ours --dtype $dt --min-kib 16 --max-kib 1024 --oneshot-max 1048576 --reps 20 --burst 50 >> $F 2>> $OUT/${TAG}_sweep_n$N.err
  timeout 300 $RUN --master-port 29625 tools/sweep_allreduce.py --mode ours --nvls --dtype $dt --min-kib 16 --max-kib 1024 --oneshot-max 1048576 --reps 20 --burst 50 >> $F 2>> $OUT/${TAG}_sweep_n$N.err
  timeout 300 $RUN --master-port 29623 tools/sweep_allreduce.py --mode ours_tap --dtype $dt --min-kib 16 --max-kib 1024 --oneshot-max 1048576 --reps 20 --burst 50 >> $F 2>> $OUT/${TAG}_sweep_n$N.err
  timeout 300 $RUN --master-port 29624 tools/sweep_allreduce.py --mode nccl --dtype $dt --min-kib 16 --max-kib 4096 --reps 20 --burst 50 >> $F 2>> $OUT/${TAG}_sweep_n$N.err
done
echo done >> $OUT/${TAG}_sweep_n$N.err
