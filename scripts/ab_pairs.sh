#!/bin/bash
# A/B of build variants without the GPU test suite: each argument is "CONFIG:var1,var2,...";
# REPS rounds, interleaved.   usage: scripts/ab_pairs.sh "C4:base,v1" "C5_512:base,v2"
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/ab.txt
for rep in $(seq 1 ${REPS:-2}); do
for spec in "$@"; do
  c=${spec%%:*}; vs=${spec#*:}
  for v in ${vs//,/ }; do
    LOB_LIB_OVERRIDE=variants/$v.so timeout 600 python bench.py --config $c --steps ${STEPS:-10} --e2e-steps 0 --no-cpu-baseline --parity-books ${PARITY:-64} > gpurun_out/ab_${c}_$v.json 2> gpurun_out/ab_${c}_$v.err
    python -c "import json; d=json.load(open('gpurun_out/ab_${c}_$v.json')); print('$c', '$v', '%.4g msg/s'%d['value'], 'kernel %.4f ms'%d['roofline']['kernel_ms'], 'parity', d['parity']['bit_exact'])" >> gpurun_out/ab.txt 2>&1 || echo "$c $v failed" >> gpurun_out/ab.txt
  done
done
done
cat gpurun_out/ab.txt
