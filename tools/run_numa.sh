#!/bin/bash
# NUMA placement probe of the host shadow segment (N GPUs): topology + D2H into node-bound pinned memory.
cd "$(dirname "$0")/.."
N=$1; OUT=gpurun_out
(lscpu | grep -i -E "numa|socket|model name"; nvidia-smi topo -m; numactl -H 2>/dev/null; cat /sys/devices/system/node/node*/meminfo | grep MemTotal) > $OUT/numa_topo_n$N.txt 2>&1
timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29761 tools/numa_probe.py > $OUT/numa_probe_n$N.jsonl 2> $OUT/numa_probe_n$N.err
echo "rc=$?" >> $OUT/numa_probe_n$N.err
