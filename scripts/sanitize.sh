#!/bin/bash
# compute-sanitizer memcheck / synccheck / racecheck over scripts/sanitize_small.py
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  echo "== $tool"
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_small.py 2>&1 | grep -E "COMPUTE-SANITIZER|ERROR SUMMARY|sanitize run ok|Error|Race|hazard" | head -40
done
