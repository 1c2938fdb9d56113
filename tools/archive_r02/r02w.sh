#!/bin/bash
# C5 at Llama-3-8B scale (4 GPUs, ZeRO-1, bf16 grads, host shadow K=8 D=9): hard kill after 10
# iterations (shadow one step behind: the last iteration's shadow step still in flight), new
# processes attach, restore (wall time), 5 more iterations sampled bit-exact vs the oracle;
# then the same with a kill 5 ms into a restore.
cd "$(dirname "$0")/.."
N=${1:-4}; TAG=${2:-r02w}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
export CM_RESTORE_WORKLOAD=llama8b
: > $OUT/${TAG}_c5_llama_n$N.jsonl
timeout 900 $RUN --master-port 31801 tools/restore_bench.py phase1 c5ll$N 10 5 step >> $OUT/${TAG}_c5_llama_n$N.log 2>&1
CM_KILL_POINT=step timeout 900 $RUN --master-port 31802 tools/restore_bench.py phase2 c5ll$N 10 5 >> $OUT/${TAG}_c5_llama_n$N.jsonl 2>> $OUT/${TAG}_c5_llama_n$N.log
rm -f /dev/shm/c5ll$N.r*
timeout 900 $RUN --master-port 31803 tools/restore_bench.py phase1 c5lm$N 13 5 step >> $OUT/${TAG}_c5_llama_n$N.log 2>&1
timeout 600 $RUN --master-port 31804 tools/restore_bench.py phase2kill c5lm$N 13 5 0.05 >> $OUT/${TAG}_c5_llama_n$N.log 2>&1
CM_KILL_POINT="step+restore_killed_0.05s" timeout 900 $RUN --master-port 31805 tools/restore_bench.py phase2 c5lm$N 13 5 >> $OUT/${TAG}_c5_llama_n$N.jsonl 2>> $OUT/${TAG}_c5_llama_n$N.log
rm -f /dev/shm/c5lm$N.r*
