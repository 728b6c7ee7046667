#!/bin/bash
# K sweep on C4: books per GPU from 1 to 262,144, device-resident,
# one line per K -> gpurun_out/k_sweep.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/k_sweep.txt
for K in 1 16 148 592 1184 4736 16384 65536 262144; do
  timeout 600 python bench.py --config C4 --books $K --steps ${STEPS:-5} --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/k_$K.json 2> gpurun_out/k_$K.err
  python -c "import json; d=json.loads(open('gpurun_out/k_$K.json').read().strip().splitlines()[-1]); r=d['roofline']; print('K=$K', '%.4g msg/s'%d['value'], '%.3f ns/msg'%d['ns_per_message'], 'kernel %.4f ms'%r['kernel_ms'], 'step %.4f ms'%d['ms_per_step'], 'hbm %.2f%%'%(100*r['frac']))" >> gpurun_out/k_sweep.txt 2>&1 || echo "K=$K failed" >> gpurun_out/k_sweep.txt
done
cat gpurun_out/k_sweep.txt
