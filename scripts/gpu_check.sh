#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + full capture of the step kernel.
# usage: scripts/gpu_check.sh [tests|bench|ncu|all]...
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
what="${*:-all}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
for w in $what; do
  case $w in
    tests|all)
      timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/status.txt
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt ;;&
    bench|all)
      timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/status.txt ;;&
    launches|all)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv \
         python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu-launch rc=$?" >> gpurun_out/status.txt ;;&
    ncu|all)
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:lob_step -s 3 -c 1 -o gpurun_out/prof_step -f \
         python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu-full rc=$?" >> gpurun_out/status.txt ;;
  esac
done
cat gpurun_out/status.txt
