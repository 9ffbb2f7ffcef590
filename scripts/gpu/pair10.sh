ISB_PAIR_CFG=256 timeout 300 python scripts/pair_quick.py 2048 4 1 3 55 2>&1 | grep -v "pair == ss: True" > gpurun_out/pair10.txt 2>&1
ISB_PAIR_CFG=256 timeout 120 python scripts/trace_pair.py 2048 4096 22016 0 2>&1 | grep -v "Warn\|_methods\|ret = " >> gpurun_out/pair10.txt 2>&1
ISB_PAIR_CFG=256 timeout 120 python scripts/trace_pair.py 2048 4096 22016 4 2>&1 | grep -v "Warn\|_methods\|ret = " >> gpurun_out/pair10.txt 2>&1
cat gpurun_out/pair10.txt
