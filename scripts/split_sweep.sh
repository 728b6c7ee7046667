#!/bin/bash
# side-split build vs lob_step on latency-bound shapes (few books): C1, C2, and C4 /
# C5 batches of K books; LOB_SPLIT_BPS forces the choice -> gpurun_out/split_sweep.txt
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/split_sweep.txt
run() {  # label env... -- bench args
  local lab=$1; shift
  env "$@" timeout 300 python bench.py $BARGS --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --parity-books 64 > gpurun_out/ss.json 2> gpurun_out/ss.err
  python -c "import json; d=json.loads(open('gpurun_out/ss.json').read().strip().splitlines()[-1]); print('$lab', '%.4g msg/s'%d['value'], 'kernel %.4f ms'%d['roofline']['kernel_ms'], 'parity', d['parity']['bit_exact'])" >> gpurun_out/split_sweep.txt 2>&1 || echo "$lab failed" >> gpurun_out/split_sweep.txt
}
for spec in "C1:0" "C2:0" "C4:148" "C4:592" "C4:1184" "C4:2368" "C4:4736" "C5_100:1184" "C5_256:592" "C5_512:296" "C5_512:1184"; do
  c=${spec%%:*}; k=${spec#*:}
  BARGS="--config $c"; [ $k != 0 ] && BARGS="$BARGS --books $k"
  run "$c K=$k split" LOB_SPLIT_BPS=100000 LOB_SPLIT_MIN_MSGS=0
  run "$c K=$k step " LOB_SPLIT_BPS=0
done
cat gpurun_out/split_sweep.txt
