ISB_AB_FLAG=4194304 timeout 60 python scripts/trace_pair.py 2048 4096 22016 0 2>&1 | grep -v "Warn\|_methods\|ret = "
ISB_AB_FLAG=4194304 timeout 60 python scripts/trace_pair.py 2048 4096 22016 4 2>&1 | grep -v "Warn\|_methods\|ret = "
