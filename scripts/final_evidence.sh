#!/bin/bash
# All round evidence for the in-tree build in one gpurun call.
#   scripts/final_evidence.sh <tag>
cd "$(dirname "$0")/.."
tag=${1:-final}
mkdir -p gpurun_out
bash scripts/measure_v.sh $tag
bash scripts/ncu_configs.sh $tag C2 C3 C5_512 C5_2048 > gpurun_out/ncu_configs_$tag.txt 2>&1
CFG=C2 bash scripts/ncu_split.sh > /dev/null 2>&1
python scripts/ncu_summary.py full gpurun_out/prof_split_C2.ncu-rep 10000000 > gpurun_out/step_split_C2_ncu_full_$tag.txt 2>&1
python scripts/sass_hotspots.py gpurun_out/prof_split_C2.ncu-rep _ZN4lobk14lob_step_splitILi4ELi2EEEvNS_6ParamsE 40 > gpurun_out/step_split_C2_hotspots_$tag.txt 2>&1
mkdir -p /tmp/ncu_reps && mv gpurun_out/prof_split_C2.ncu-rep /tmp/ncu_reps/ 2>/dev/null
CONFIGS="C1 C2 C3 C4 C5_32 C5_100 C5_256 C5_512 C5_1024 C5_2048" bash scripts/config_sweep.sh > /dev/null
timeout 300 python scripts/rl_shape.py > gpurun_out/rl_shape_$tag.json 2>&1
timeout 600 python scripts/env_bench.py > gpurun_out/env_bench_$tag.json 2>&1
timeout 300 python scripts/session_overhead.py > gpurun_out/session_overhead_$tag.json 2>&1
LOB_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_gloo2_$tag.json 2> gpurun_out/bench_gloo2_$tag.err
timeout 300 python bench.py --l1 --steps 5 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_l1_$tag.json 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$tag.json 2>&1
timeout 300 python scripts/paper_tables.py > gpurun_out/paper_tables_$tag.json 2>&1
timeout 300 taskset -c 0 python scripts/oracle_1core.py > gpurun_out/oracle_1core_$tag.json 2>&1
bash scripts/k_sweep.sh > /dev/null
[ -n "$SKIP_SAN" ] || bash scripts/sanitize_all.sh > gpurun_out/sanitize_$tag.txt   # (compute-sanitizer may be closed on the pool)
bash scripts/split_sweep.sh > /dev/null
cat gpurun_out/measure_$tag.txt gpurun_out/ncu_configs_$tag.txt gpurun_out/sweep.txt gpurun_out/k_sweep.txt gpurun_out/split_sweep.txt
