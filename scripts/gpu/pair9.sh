for c in 256 192; do
  echo "== ISB_PAIR_CFG=$c"
  ISB_PAIR_CFG=$c timeout 300 python scripts/pair_quick.py 2048 4 128 256 1 3 55 2>&1 | grep -v "pair == ss: True"
done > gpurun_out/pair9.txt 2>&1
ISB_PAIR_CFG=256 timeout 120 python scripts/trace_pair.py 2048 4096 22016 0 >> gpurun_out/pair9.txt 2>&1
ISB_PAIR_CFG=256 timeout 120 python scripts/trace_pair.py 2048 4096 22016 4 >> gpurun_out/pair9.txt 2>&1
cat gpurun_out/pair9.txt
