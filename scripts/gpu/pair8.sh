for c in 256 2562 192; do
  echo "== ISB_PAIR_CFG=$c"
  ISB_PAIR_CFG=$c timeout 300 python scripts/pair_quick.py 2048 4 8 128 256 55 2>&1
done > gpurun_out/pair8.txt 2>&1
cat gpurun_out/pair8.txt
