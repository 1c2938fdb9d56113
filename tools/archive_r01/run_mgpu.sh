#!/bin/bash
# Multi-GPU session: multi-process parity tests, C3 bucket sweep (ours without tap, ours
# with the staged and the direct tap, NCCL default and NVLS off), bench.py and the GPT-2
# model mode at N GPUs.  Usage: tools/run_mgpu.sh N [max_mib] [skip_tests]
cd "$(dirname "$0")/.."
N=$1; MAXMIB=${2:-1024}
OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
if [ -z "$3" ]; then
  timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > $OUT/mp_tests_n$N.log 2>&1
  echo "mp tests rc=$?" >> $OUT/mp_tests_n$N.log
fi
rm -f $OUT/sweep_n$N.jsonl
for mode in ours ours_tap ours_tap_direct nccl; do
  timeout 600 $RUN --master-port 29611 tools/sweep_allreduce.py --mode $mode --max-mib $MAXMIB >> $OUT/sweep_n$N.jsonl 2>> $OUT/sweep_n$N.err
done
NCCL_NVLS_ENABLE=0 timeout 600 $RUN --master-port 29612 tools/sweep_allreduce.py --mode nccl --max-mib $MAXMIB >> $OUT/sweep_n$N.jsonl 2>> $OUT/sweep_n$N.err
timeout 600 $RUN --master-port 29613 bench.py --gpus $N --steps 10 --warmup 3 > $OUT/bench_n$N.json 2> $OUT/bench_n$N.err
timeout 900 $RUN --master-port 29614 tools/model_mode.py --steps 12 --warmup 4 > $OUT/model_n$N.json 2> $OUT/model_n$N.err
timeout 900 $RUN --master-port 29615 tools/model_mode.py --steps 12 --warmup 4 --tap direct --arms ours_ckpt > $OUT/model_n${N}_direct.json 2>> $OUT/model_n$N.err
