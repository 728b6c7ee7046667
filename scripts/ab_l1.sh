#!/bin/bash
# A/B of the L1-trace build (bench.py --l1, C4) across variants/<name>.so.  usage: scripts/ab_l1.sh v1 v2 ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/ab_l1.txt
for rep in 1 2; do for v in "$@"; do
  LOB_LIB_OVERRIDE=variants/$v.so timeout 600 python bench.py --l1 --steps 10 --e2e-steps 0 --no-cpu-baseline --parity-books 64 > gpurun_out/abl1_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/abl1_$v.json').read().strip().splitlines()[-1]); print('L1', '$v', '%.4g msg/s'%d['value'], 'parity', d['parity']['bit_exact'])" >> gpurun_out/ab_l1.txt 2>&1 || echo "$v failed" >> gpurun_out/ab_l1.txt
done; done
cat gpurun_out/ab_l1.txt
