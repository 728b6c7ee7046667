#!/bin/bash
# One gpurun call: GPU tests + smoke + bench (N=1), then the self-spawned 2-rank bench
# (gloo, both ranks on the one GPU).   usage: scripts/check_all.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
bash scripts/gpu_check.sh tests bench > /dev/null
LOB_DIST_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_gloo2.json 2> gpurun_out/bench_gloo2.err; echo "gloo2 rc=$?" >> gpurun_out/status.txt
cat gpurun_out/status.txt; tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json
