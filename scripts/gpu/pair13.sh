ISB_PAIR_CFG=2563 timeout 100 python scripts/pair_quick.py 2048 4 1 2 55 2>&1 | grep -v "pair == ss: True"
ISB_PAIR_CFG=2563 timeout 60 python scripts/trace_pair.py 2048 4096 22016 0 2>&1 | grep -v "Warn\|_methods\|ret = "
ISB_PAIR_CFG=2563 timeout 60 python scripts/trace_pair.py 2048 4096 22016 4 2>&1 | grep -v "Warn\|_methods\|ret = "
