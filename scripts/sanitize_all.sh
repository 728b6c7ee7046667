#!/bin/bash
# compute-sanitizer over scripts/sanitize.py: default grid, a 1-CTA grid (LOB_GRID_CAP=1)
# so the dynamic book scheduler runs under racecheck/synccheck, the many-wave build and the
# side-split build.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  for cap in 0 1; do
    LOB_GRID_CAP=$cap timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/san_${tool}_cap$cap.txt 2>&1
    echo "$tool cap=$cap rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san_${tool}_cap$cap.txt | tail -1)"
  done
  # the many-wave build (predicated single-writer stores) forced on the small batches
  LOB_FORCE_WIDE=1 LOB_GRID_CAP=1 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/san_${tool}_wide.txt 2>&1
  echo "$tool wide rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san_${tool}_wide.txt | tail -1)"
  # the side-split build (lob_split.cuh) forced on every one-warp batch
  LOB_SPLIT_BPS=100000 LOB_SPLIT_MIN_MSGS=0 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/san_${tool}_split.txt 2>&1
  echo "$tool split rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san_${tool}_split.txt | tail -1)"
done
