"""Grouped prefill launch of the LLaMA-2-7B layer (pre-quantized inputs, M from argv[1]):
the CTA-pair fold kernel over all four linears' tiles, for ncu:
ncu -k regex:gemm_w4a8_sp -s 2 -c 1 python scripts/prefill_group_profile.py 2048"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14597_b200 as isb  # noqa: E402
from bench import LAYER, build_layers  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
dev = torch.device("cuda:0")
layers, _ = build_layers(isb, 16, dev, seed=1234)
xq = [isb.quantize_per_token(torch.randn((m, k), device=dev)) for _, k, _ in LAYER]
plan = isb.GroupedGemm([{"weight": l[3], "xq": q, "sa": sa} for l, (q, sa) in zip(layers[0], xq)])
for _ in range(4):
    plan.run()
torch.cuda.synchronize()
print("done", plan.grid, plan.tile_tokens)
