#!/bin/bash
# ncu --set full (+ explicit pipe and local-memory counters) of ONE lob_step launch per
# config, in-tree build.   usage: scripts/ncu_configs.sh <tag> C5_512 C5_2048 C2 ...
cd "$(dirname "$0")/.."
tag=$1; shift
mkdir -p gpurun_out
for c in "$@"; do
  timeout 900 ncu --set full --metrics sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_lsu.sum,sm__inst_executed_pipe_cbu.sum,sm__inst_executed_pipe_adu.sum,sm__inst_executed_pipe_uniform.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum \
    --clock-control none --import-source on -k regex:lob_step -s 3 -c 1 -o gpurun_out/prof_${c}_$tag -f \
    python bench.py --config $c --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline --parity-books 0 > gpurun_out/ncu_${c}_$tag.log 2>&1
  echo "$c ncu rc=$?"
  case $c in C2) n=10000000;; C3) n=16384000;; C4) n=65536000;; C1) n=1000;; *) n=4096000;; esac
  python scripts/ncu_summary.py full gpurun_out/prof_${c}_$tag.ncu-rep $n > gpurun_out/step_${c}_ncu_full_$tag.txt 2>&1
  [ -n "$KEEP_REPS" ] || { mkdir -p /tmp/ncu_reps && mv gpurun_out/prof_${c}_$tag.ncu-rep /tmp/ncu_reps/; }
done
