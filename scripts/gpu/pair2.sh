# pair kernel configs x measurement knobs (M=2048 LLaMA-2-7B layer)
for c in 256 2562 192; do
  echo "== ISB_PAIR_CFG=$c"
  ISB_PAIR_CFG=$c timeout 300 python scripts/pair_quick.py 2048 1 2 3 4 16 32 48 7 55 2>&1 | grep -v "^  first"
done > gpurun_out/pair2.txt 2>&1
cat gpurun_out/pair2.txt
