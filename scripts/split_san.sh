#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  LOB_SPLIT_BPS=100000 LOB_SPLIT_MIN_MSGS=0 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize.py > gpurun_out/san_${tool}_split.txt 2>&1
  echo "$tool split rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/san_${tool}_split.txt | tail -1)"
done
