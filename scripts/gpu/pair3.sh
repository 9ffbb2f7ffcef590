for c in 2562 192; do
  for f in 0 55; do
    echo "== ISB_PAIR_CFG=$c flags=$f"
    ISB_PAIR_CFG=$c timeout 120 python scripts/trace_pair.py 2048 4096 22016 $f
  done
done > gpurun_out/pair3.txt 2>&1
cat gpurun_out/pair3.txt
