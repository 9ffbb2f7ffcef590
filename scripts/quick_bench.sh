#!/bin/bash
# quick GPU check: parity subset + K3/K4 kernel timings at decode shapes
set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "integer_scale_bit_exact or float_scale or workspace or random_instances" > gpurun_out/quick_tests.log 2>&1; echo rc=$? >> gpurun_out/quick_tests.log
timeout 300 python bench.py --steps 500 --warmup 20 --no-cpu --sweep 1 16 64 256 2048 > gpurun_out/quick_bench.json 2> gpurun_out/quick_bench.err
