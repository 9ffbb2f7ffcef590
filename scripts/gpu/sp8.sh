timeout 100 python scripts/pair_quick.py 2048 2>&1 | grep -v "== ss: True"
ISB_AB_FLAG=0 timeout 60 python scripts/trace_pair.py 2048 4096 22016 0 2>&1 | grep "epilogue chunk\|issue-to-issue\|a_full after"
timeout 300 python -c "
import sys; sys.argv=['x']; import torch, bench, paper_2405_14597_b200 as isb
dev=torch.device('cuda:0'); layers,_=bench.build_layers(isb,16,dev,1234)
xq=[isb.quantize_per_token(torch.randn((2048,k),device=dev)) for _,k,_ in bench.LAYER]
us,_=bench.grouped_prefill_us(isb,layers,xq); ops=sum(2*2048*k*n for _,k,n in bench.LAYER)
print(f'grouped prefill M=2048: {us:.1f} us = {ops/us/1e6:.0f} TOPS')"
