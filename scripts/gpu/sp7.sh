timeout 100 python scripts/pair_quick.py 2048 2>&1 | grep -v "== ss: True"; timeout 200 python -m pytest tests/test_gpu_scale.py -q -x -k "prefill_fold or pair_kernel or full_size" 2>&1 | tail -2
ISB_AB_FLAG=0 timeout 60 python scripts/trace_pair.py 2048 4096 22016 0 2>&1 | grep "epilogue chunk\|issue-to-issue\|^tile [0-2]"
