ISB_AB_FLAG=4194304 timeout 60 python scripts/trace_pair.py 2048 4096 22016 0 2>&1 | grep -v "Warn\|_methods\|ret = " | grep -v "^[0-9]* "
ISB_AB_FLAG=4194304 timeout 100 python scripts/pair_quick.py 2048 512 8 2>&1 | grep -v "pair == ss: True"
