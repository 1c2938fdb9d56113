#!/bin/bash
# Restore source-snapshot fix: the new test passes with the fixed library and fails with the
# library built before the fix (tools/exp/libcm_before_restore_fix.so: nvcc of cm_runtime.cu as
# of 4c5fc53^, the parent of the fix commit, with build.py's flags; not kept in the tree), then
# the restore tests.
cd "$(dirname "$0")/.."
OUT=gpurun_out; TAG=${1:-r01e_restore}
K="source_snapshot"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$K" > $OUT/${TAG}_fixed.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_fixed.log
cp paper_2507_13522_b200/libcm.so /tmp/libcm_fixed.so
cp tools/exp/libcm_before_restore_fix.so paper_2507_13522_b200/libcm.so
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "$K" > $OUT/${TAG}_before_fix.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_before_fix.log
cp /tmp/libcm_fixed.so paper_2507_13522_b200/libcm.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sgd.py -m gpu -q -k "restore or consolidation or lagging" > $OUT/${TAG}_restore_tests.log 2>&1; echo "rc=$?" >> $OUT/${TAG}_restore_tests.log
