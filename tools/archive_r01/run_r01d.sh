cd $GRAFT_REPO_ROOT
OUT=gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/r01d_tests.log 2>&1; echo "rc=$?" >> $OUT/r01d_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r01d_smoke.log 2>&1; echo "rc=$?" >> $OUT/r01d_smoke.log
timeout 1200 python bench.py --steps 20 --warmup 5 > $OUT/r01d_bench_n1.json 2> $OUT/r01d_bench_n1.err; echo "rc=$?" >> $OUT/r01d_bench_n1.err
