#!/bin/bash
# compute-sanitizer over tools/sanitize.py; summaries into gpurun_out/sanitize_<tool>.txt
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $tool  \
    --print-limit 20 python tools/sanitize.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize_$tool.txt | tail -2 | tr '\n' ' ')"
done
