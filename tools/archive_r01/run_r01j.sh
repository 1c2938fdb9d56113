#!/bin/bash
# Final 2-GPU evidence: multi-process suite at n=2, then the full bench line.
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r01j}
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -m gpu -q -k "not llama" > $OUT/${TAG}_mp_tests_n2.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_mp_tests_n2.log
timeout 1200 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 30061 bench.py --gpus 2 --steps 20 --warmup 5 > $OUT/${TAG}_bench_n2.json 2> $OUT/${TAG}_bench_n2.err
