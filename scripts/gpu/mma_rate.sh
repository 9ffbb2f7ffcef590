#!/bin/bash
timeout 120 python scripts/pf_time.py 2048 0 64 0 64
timeout 100 python scripts/pair_quick.py 2048 64 2>&1 | grep -v "== ss: True" | head -4
