#!/bin/bash
for m in 16 32 64; do timeout 300 python scripts/group_knobs.py $m 65536; done
