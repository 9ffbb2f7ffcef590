#!/bin/bash
# A/B of compile-time variants: ISB_LIB_PATH points the ctypes binding at each build.
for f in exp_libs/*.so; do
  for d in ${DBG:-1 25}; do
    echo "== $f dbg=$d"
    ISB_LIB_PATH=$f ISB_DECODE_DBG=$d BIG=1 timeout 60 python scripts/launch_modes.py
  done
done
