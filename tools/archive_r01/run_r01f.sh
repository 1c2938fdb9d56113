bash tools/run_r01e_restore.sh r01e_restore
bash tools/run_c5_points.sh 2 r01e_c5
timeout 900 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29981 bench.py --gpus 2 --steps 20 --warmup 5 --no-model > gpurun_out/r01f_bench_n2.json 2> gpurun_out/r01f_bench_n2.err
