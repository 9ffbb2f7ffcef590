for c in 2562 192; do
  echo "== ISB_PAIR_CFG=$c"
  ISB_PAIR_CFG=$c timeout 300 python scripts/pair_quick.py 2048 4 8 128 136 52 2>&1 | grep -v "pair == ss: True"
done > gpurun_out/pair7.txt 2>&1
cat gpurun_out/pair7.txt
