#!/bin/bash
timeout 120 python scripts/pf_time.py 2048 0
timeout 900 python -m pytest tests/test_gpu_group.py tests/test_gpu_scale.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
