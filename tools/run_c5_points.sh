#!/bin/bash
# SURVEY 8.d C5 kill points at N GPUs (GPT-2, K=8, D=16): hard kill after k in {1, 7, 50}
# whole iterations, after iteration k's all-reduces (before its optimizer step), and in the
# middle of a restore (SIGKILL 5 ms / 30 ms / 80 ms into cm_restore); every case then restores
# and runs 100 more iterations, sampled bit-exact vs the oracle's uninterrupted run.
cd "$(dirname "$0")/.."
N=${1:-2}; TAG=${2:-r01e_c5}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
: > $OUT/${TAG}_n$N.jsonl
port=29900
one() {   # name k point [kill-delay]
  local name=$1 k=$2 point=$3 delay=$4
  port=$((port + 3))
  CM_KILL_POINT=$point timeout 600 $RUN --master-port $port tools/restore_bench.py phase1 $name $k 100 $point >> $OUT/${TAG}_n$N.log 2>&1
  if [ -n "$delay" ]; then
    timeout 300 $RUN --master-port $((port + 1)) tools/restore_bench.py phase2kill $name $k 100 $delay >> $OUT/${TAG}_n$N.log 2>&1
    point="${point}+restore_killed_${delay}s"
  fi
  CM_KILL_POINT=$point timeout 900 $RUN --master-port $((port + 2)) tools/restore_bench.py phase2 $name $k 100 >> $OUT/${TAG}_n$N.jsonl 2>> $OUT/${TAG}_n$N.log
  rm -f /dev/shm/$name.r*
}
one c5a$N 1 step
one c5g$N 7 before_rs
one c5b$N 7 after_ar
one c5h$N 16 mid_shadow
one c5c$N 50 step
one c5d$N 11 step 0.005
one c5e$N 11 step 0.03
one c5f$N 11 step 0.08
