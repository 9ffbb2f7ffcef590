#!/bin/bash
timeout 120 python scripts/pf_time.py 2048 0 64 0 64 2112
