#!/bin/bash
# A/B of the latency-bound shapes (C2 modes, N3 env step) for kernel build variants:
#   scripts/ab_latency.sh <name>:<so> ...   (runs on the GPU box)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  name=${v%%:*}; so=${v#*:}
  echo "== $name" >> gpurun_out/ab_latency.txt
  LOB_LIB_OVERRIDE=$so timeout 300 python scripts/rl_shape.py >> gpurun_out/ab_latency.txt 2>&1
  LOB_LIB_OVERRIDE=$so timeout 300 python scripts/env_bench.py >> gpurun_out/ab_latency.txt 2>&1
done
cat gpurun_out/ab_latency.txt
