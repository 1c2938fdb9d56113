#!/bin/bash
# Round-1 final evidence. N=1: full GPU suite, smoke, bench. N>1: multi-process suite, bench.
cd "$(dirname "$0")/.."
OUT=gpurun_out; N=${1:-1}; TAG=${2:-r01e}
if [ "$N" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > $OUT/${TAG}_tests_n1.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_tests_n1.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_smoke.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_smoke.log
  timeout 1200 python bench.py --steps 20 --warmup 5 > $OUT/${TAG}_bench_n1.json 2> $OUT/${TAG}_bench_n1.err; echo "rc=$?" >> $OUT/${TAG}_bench_n1.err
else
  timeout 1500 python -m pytest tests/test_gpu_multiproc.py -m gpu -q > $OUT/${TAG}_mp_tests_n$N.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_mp_tests_n$N.log
  timeout 1200 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29871 bench.py --gpus $N --steps 20 --warmup 5 > $OUT/${TAG}_bench_n$N.json 2> $OUT/${TAG}_bench_n$N.err; echo "rc=$?" >> $OUT/${TAG}_bench_n$N.err
fi
