#!/bin/bash
# Prefill kernel ring-depth A/B: grouped LLaMA-2-7B layer at M=2048 per library variant.
cat > /tmp/pf.py <<'PY'
import sys; sys.argv=['x']; import torch, bench, paper_2405_14597_b200 as isb
dev=torch.device('cuda:0'); layers,_=bench.build_layers(isb,16,dev,1234)
xq=[isb.quantize_per_token(torch.randn((2048,k),device=dev)) for _,k,_ in bench.LAYER]
ops=sum(2*2048*k*n for _,k,n in bench.LAYER)
for r in range(3):
    us,_=bench.grouped_prefill_us(isb,layers,xq); print(f'  grouped prefill M=2048: {us:.1f} us = {ops/us/1e6:.0f} TOPS', flush=True)
PY
for v in default scripts/_var/sp_12_6.so scripts/_var/sp_12_7.so scripts/_var/sp_9_9.so; do
  echo "== $v"
  if [ $v = default ]; then unset ISB_LIB_PATH; else export ISB_LIB_PATH=$PWD/$v; fi
  timeout 120 python /tmp/pf.py
  timeout 100 python scripts/pair_quick.py 2048 2>&1 | grep -v "== ss: True"
done
unset ISB_LIB_PATH
timeout 60 python scripts/trace_pair.py 2048 4096 22016 0 2>&1 | grep "issue-to-issue\|transform warp\|a_full after"
