for c in 2561 256; do
ISB_PAIR_CFG=$c timeout 300 python scripts/pair_quick.py 2048 4 2>&1 | grep -v "pair == ss: True"
ISB_PAIR_CFG=$c timeout 120 python scripts/trace_pair.py 2048 4096 22016 0 2>&1 | grep -v "Warn\|_methods\|ret = "
ISB_PAIR_CFG=$c timeout 120 python scripts/trace_pair.py 2048 4096 22016 4 2>&1 | grep -v "Warn\|_methods\|ret = "
done > gpurun_out/pair12.txt 2>&1
cat gpurun_out/pair12.txt
