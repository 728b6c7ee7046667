#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lob_step_split -s 3 -c 1 -o gpurun_out/prof_split_${CFG:-C2} -f \
    python bench.py --config ${CFG:-C2} --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --parity-books 0 > gpurun_out/ncu_split.log 2>&1
echo "ncu rc=$?"
