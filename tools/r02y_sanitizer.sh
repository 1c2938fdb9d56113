#!/bin/bash
# compute-sanitizer over the smoke path and selected parity tests (1 GPU, virtual ranks):
# memcheck (out-of-bounds / misaligned / leaks of device memory), racecheck (shared-memory
# hazards: the TMA-staged kernels), synccheck (barrier misuse).
cd "$(dirname "$0")/.."
TAG=${1:-r02y}; OUT=gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $CS --tool memcheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_memcheck_smoke.log 2>&1
echo "rc=$?" >> $OUT/${TAG}_memcheck_smoke.log
timeout 1500 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_edge.py tests/test_gpu_bucket_step.py -q -x \
  -k "edge_values_full_path_bit_exact or nonfinite_is_refused or bucket_steps_bit_exact and 2-0" > $OUT/${TAG}_memcheck_tests.log 2>&1
echo "rc=$?" >> $OUT/${TAG}_memcheck_tests.log
timeout 900 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_checkpoint.py -q -x -k "single_bit_flip" > $OUT/${TAG}_memcheck_verify.log 2>&1
echo "rc=$?" >> $OUT/${TAG}_memcheck_verify.log
timeout 900 $CS --tool racecheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -q -x -k "adamw_implementations_bit_exact or zero1_bit_exact and 2-0-2" > $OUT/${TAG}_racecheck.log 2>&1
echo "rc=$?" >> $OUT/${TAG}_racecheck.log
timeout 900 $CS --tool synccheck --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${TAG}_synccheck_smoke.log 2>&1
echo "rc=$?" >> $OUT/${TAG}_synccheck_smoke.log
