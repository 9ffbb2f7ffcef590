timeout 600 python -m pytest tests/test_gpu_group.py -x -q 2>&1 | tail -3
timeout 300 python scripts/group_fold_ab.py 1 16 32 64
