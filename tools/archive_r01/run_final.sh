#!/bin/bash
# Round-end evidence at N GPUs: C5 restore (hard kill at k=11, restore, 100 more steps
# bit-exact), the full bench line, and (N >= 4) the C4 Llama-8B-shaped synthetic bench line.
cd "$(dirname "$0")/.."
N=$1; TAG=${2:-fin}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
timeout 600 $RUN --master-port 29751 tools/restore_bench.py phase1 cmrb${TAG}$N 11 > $OUT/${TAG}_restore_n$N.log 2>&1
timeout 900 $RUN --master-port 29752 tools/restore_bench.py phase2 cmrb${TAG}$N 11 100 > $OUT/${TAG}_restore_n$N.json 2>> $OUT/${TAG}_restore_n$N.log
if [ "$N" = "1" ]; then B="python"; else B="$RUN --master-port 29753"; fi
timeout 1200 $B bench.py --gpus $N --steps 20 --warmup 5 > $OUT/${TAG}_bench_n$N.json 2> $OUT/${TAG}_bench_n$N.err
if [ "$N" -ge 4 ]; then
  timeout 1500 $RUN --master-port 29754 bench.py --gpus $N --workload llama8b --steps 5 --warmup 3 --ring-depth 8 --persist-every 8 --no-e2e --zero1 --no-model > $OUT/${TAG}_llama_n$N.json 2> $OUT/${TAG}_llama_n$N.err
fi
