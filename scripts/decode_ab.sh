#!/bin/bash
# A/B of the decode kernel launch modes (graph of back-to-back launches).
for cfg in "" "ISB_NO_PDL=1" "ISB_DECODE_PAD=20000" "ISB_DECODE_PAD=20000 ISB_NO_PDL=1" "ISB_NO_DECODE=1"; do
  echo "== $cfg"
  env $cfg python scripts/launch_modes.py 2>&1 | grep graph
done
