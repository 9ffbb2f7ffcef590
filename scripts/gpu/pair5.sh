for c in 2562 192 256; do
  echo "== ISB_PAIR_CFG=$c"
  ISB_PAIR_CFG=$c timeout 300 python scripts/pair_quick.py 2048 4 3 64 48 55 2>&1 | grep -v "^  first"
done > gpurun_out/pair5.txt 2>&1
ISB_PAIR_CFG=192 timeout 120 python scripts/trace_pair.py 2048 4096 22016 0 >> gpurun_out/pair5.txt 2>&1
ISB_PAIR_CFG=2562 timeout 120 python scripts/trace_pair.py 2048 4096 22016 0 >> gpurun_out/pair5.txt 2>&1
cat gpurun_out/pair5.txt
