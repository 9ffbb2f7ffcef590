ISB_AB_FLAG=4194304 timeout 100 python scripts/pair_quick.py 2048 8 4 2>&1
