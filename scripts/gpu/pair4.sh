for c in 256 2562 192; do
  echo "== ISB_PAIR_CFG=$c"
  ISB_PAIR_CFG=$c timeout 300 python scripts/pair_quick.py 2048 64 3 67 55 119 2>&1 | grep -v "^  first"
done > gpurun_out/pair4.txt 2>&1
ISB_PAIR_CFG=192 timeout 120 python scripts/trace_pair.py 2048 4096 22016 64 >> gpurun_out/pair4.txt 2>&1
cat gpurun_out/pair4.txt
