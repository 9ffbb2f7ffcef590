#!/bin/bash
timeout 120 python scripts/pf_time.py 2048 0 32 0 32
timeout 100 python scripts/pair_quick.py 2048 2>&1 | grep -v "== ss: True" | head -4
