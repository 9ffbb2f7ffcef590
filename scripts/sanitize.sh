#!/bin/bash
# compute-sanitizer memcheck / synccheck / racecheck over scripts/sanitize_small.py
mkdir -p gpurun_out
CS=${CS:-/usr/local/cuda/bin/compute-sanitizer}
for tool in memcheck synccheck racecheck; do
  echo "== $tool"
  timeout 1200 $CS --tool $tool --print-limit 20 python scripts/sanitize_small.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|sanitize run ok|Traceback|Error:" gpurun_out/sanitize_$tool.log | head -20
done
