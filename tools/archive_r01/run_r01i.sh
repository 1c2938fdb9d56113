#!/bin/bash
# Link-bound threshold 12.5 GB/s: C4 filler at T=8k and T=16k tokens/GPU (N GPUs).
cd "$(dirname "$0")/.."
N=${1:-4}
TOKENS="8192 16384" bash tools/run_c4_sweep.sh $N r01i_c4
