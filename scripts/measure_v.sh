#!/bin/bash
# One gpurun call of round evidence for the in-tree build: GPU tests + smoke, default
# bench line, ncu launch list of the bench command, one ncu --set full capture of the
# C4 step kernel (+ explicit pipe counters).   usage: scripts/measure_v.sh <tag>
cd "$(dirname "$0")/.."
tag=${1:-v}
mkdir -p gpurun_out
: > gpurun_out/measure_$tag.txt
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)" >> gpurun_out/measure_$tag.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$? $(tail -1 gpurun_out/smoke.log)" >> gpurun_out/measure_$tag.txt
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?" >> gpurun_out/measure_$tag.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$tag.csv \
   python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch_$tag.log 2>&1; echo "ncu-launch rc=$?" >> gpurun_out/measure_$tag.txt
timeout 1200 ncu --set full --metrics sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_lsu.sum,sm__inst_executed_pipe_cbu.sum,sm__inst_executed_pipe_adu.sum,sm__inst_executed_pipe_uniform.sum \
   --clock-control none --import-source on -k regex:lob_step -s 3 -c 1 -o gpurun_out/prof_c4_$tag -f \
   python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_$tag.log 2>&1; echo "ncu-full rc=$?" >> gpurun_out/measure_$tag.txt
# summaries here, the report itself stays on the box (gpurun_out is capped at 64 MiB)
python scripts/ncu_summary.py full gpurun_out/prof_c4_$tag.ncu-rep 65536000 > gpurun_out/step_ncu_full_$tag.txt 2>&1
python scripts/sass_hotspots.py gpurun_out/prof_c4_$tag.ncu-rep _ZN4lobk8lob_stepILi4ELi1ELi4ELi3EEEvNS_6ParamsENS_9EnvParamsE 40 > gpurun_out/step_hotspots_$tag.txt 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_$tag.csv > gpurun_out/launches_$tag.txt 2>&1
mkdir -p /tmp/ncu_reps && mv gpurun_out/*.ncu-rep /tmp/ncu_reps/ 2>/dev/null
cat gpurun_out/measure_$tag.txt
