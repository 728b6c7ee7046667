#!/bin/bash
# bench every BASELINE config once (device-resident value only) -> gpurun_out/sweep.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in ${CONFIGS:-C1 C2 C3 C4 C5_32 C5_100 C5_512 C5_2048}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/sweep_$c.json 2> gpurun_out/sweep_$c.err
  python -c "import json; d=json.load(open('gpurun_out/sweep_$c.json')); r=d['roofline']; print('$c', '%.4g msg/s'%d['value'], '%.3f ns/msg'%d['ns_per_message'], 'kernel %.3f ms'%r['kernel_ms'], 'B/msg %.1f'%r['alg_bytes_per_msg'], 'hbm %.2f%%'%(100*r['frac']))" >> gpurun_out/sweep.txt 2>&1 || echo "$c failed" >> gpurun_out/sweep.txt
done
cat gpurun_out/sweep.txt
