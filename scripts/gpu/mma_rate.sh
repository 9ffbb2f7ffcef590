#!/bin/bash
for m in 16 32 64; do timeout 300 python scripts/group_knobs.py $m; done
timeout 900 python -m pytest tests/test_gpu_group.py -q -x 2>&1 | tail -2
