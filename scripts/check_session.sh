#!/bin/bash
# One gpurun call: session tests, GPU test suite, smoke; A/B variants (args: ab_pairs specs).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_session.py -x -q -p no:cacheprovider > gpurun_out/pytest_session.log 2>&1; echo "session rc=$? $(tail -1 gpurun_out/pytest_session.log)" > gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)" >> gpurun_out/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/status.txt
if [ $# -gt 0 ]; then REPS=${REPS:-2} bash scripts/ab_pairs.sh "$@" > /dev/null; fi
cat gpurun_out/status.txt gpurun_out/ab.txt 2>/dev/null; tail -30 gpurun_out/pytest_session.log
