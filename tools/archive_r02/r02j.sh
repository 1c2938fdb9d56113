#!/bin/bash
# N GPUs: multi-process suite, full bench line (model mode), model-mode A/B (per-bucket step),
# an nvidia-smi NVLink counter probe.
cd "$(dirname "$0")/.."
N=${1:-4}; TAG=${2:-r02j}; OUT=gpurun_out
RUN="python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1"
nvidia-smi topo -m > $OUT/${TAG}_topo.txt 2>&1
( nvidia-smi nvlink -s -i 0; nvidia-smi nvlink -gt d -i 0; nvidia-smi nvlink -gt r -i 0 ) > $OUT/${TAG}_nvlink_probe0.txt 2>&1
timeout 1800 python -m pytest tests/test_gpu_multiproc.py -q > $OUT/${TAG}_mp_tests_n$N.log 2>&1
echo "mp tests rc=$?" >> $OUT/${TAG}_mp_tests_n$N.log
( nvidia-smi nvlink -gt d -i 0 ) > $OUT/${TAG}_nvlink_probe1.txt 2>&1
timeout 1200 $RUN --master-port 31001 bench.py --gpus $N > $OUT/${TAG}_bench_n$N.json 2> $OUT/${TAG}_bench_n$N.err
echo "bench rc=$?" >> $OUT/${TAG}_bench_n$N.err
F=$OUT/${TAG}_model_n$N.jsonl; : > $F
port=31010
for cfg in "CM_BUCKET_STEP=1" "CM_BUCKET_STEP=0" "CM_BUCKET_STEP=1" "CM_BUCKET_STEP=0"; do
  port=$((port + 1))
  env $cfg timeout 900 $RUN --master-port $port tools/model_mode.py --steps 20 --warmup 5 >> $F 2>> $OUT/${TAG}_model_n$N.err
done
