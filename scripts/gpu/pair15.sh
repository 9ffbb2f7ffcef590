ISB_PAIR_CFG=2562 timeout 100 python scripts/pair_quick.py 2048 1048576 1048592 1048580 2>&1
