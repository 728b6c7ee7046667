#!/bin/bash
# A/B timing of kernel build variants: scripts/variants.sh <name>:<so> ... (runs on the GPU box)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  name=${v%%:*}; so=${v#*:}
  LOB_LIB_OVERRIDE=$so timeout 600 python bench.py --steps 10 --e2e-steps 0 --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/var_$name.json 2> gpurun_out/var_$name.err
  python -c "import json,sys; d=json.load(open('gpurun_out/var_$name.json')); print('$name', '%.4g msg/s'%d['value'], 'kernel %.3f ms'%d['roofline']['kernel_ms'])" >> gpurun_out/variants.txt 2>&1
done
cat gpurun_out/variants.txt
