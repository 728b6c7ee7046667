#!/bin/bash
# side-split experiments: wait counters, then C2 A/B (variants/*.so; nosplit = base with LOB_SPLIT_BPS=0)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
LOB_LIB_OVERRIDE=variants/splitstats.so timeout 120 python scripts/split_stats.py ${CFG:-C2} > gpurun_out/split_stats.json 2>&1
cat gpurun_out/split_stats.json
for rep in 1 2; do
for v in ${VARS:-base relaxed nosplit}; do
  so=$v; env=""
  [ $v = nosplit ] && { so=base; env="LOB_SPLIT_BPS=0"; }
  env $env LOB_LIB_OVERRIDE=variants/$so.so timeout 120 python bench.py --config ${CFG:-C2} --steps 10 --e2e-steps 0 --no-cpu-baseline --parity-books 64 > gpurun_out/sab_$v.json 2> gpurun_out/sab_$v.err
  python -c "import json; d=json.load(open('gpurun_out/sab_$v.json')); print('$v', '%.4g msg/s'%d['value'], 'kernel %.4f ms'%d['roofline']['kernel_ms'], 'parity', d['parity']['bit_exact'])" || echo "$v failed"
done
done
