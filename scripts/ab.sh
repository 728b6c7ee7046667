#!/bin/bash
# One gpurun call for a kernel change: GPU parity tests on the in-tree build, then
# A/B of build variants (variants/<name>.so) on the given configs.
#   scripts/ab.sh "C4 C2" base v14a v14b
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cfgs=$1; shift
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)" > gpurun_out/ab.txt
for rep in $(seq 1 ${REPS:-2}); do
for c in $cfgs; do
  for v in "$@"; do
    LOB_LIB_OVERRIDE=variants/$v.so timeout 600 python bench.py --config $c --steps ${STEPS:-10} --e2e-steps 0 --no-cpu-baseline > gpurun_out/ab_${c}_$v.json 2> gpurun_out/ab_${c}_$v.err
    python -c "import json; d=json.load(open('gpurun_out/ab_${c}_$v.json')); print('$c', '$v', '%.4g msg/s'%d['value'], 'kernel %.4f ms'%d['roofline']['kernel_ms'])" >> gpurun_out/ab.txt 2>&1 || echo "$c $v failed" >> gpurun_out/ab.txt
  done
done
done
cat gpurun_out/ab.txt
