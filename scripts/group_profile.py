"""Eager back-to-back grouped layer launches (LLaMA-2-7B, M from argv[1], weights
rotated over 3 replicas) for ncu: ncu -k regex:gemm_w4a8_group -s 6 -c 1 ..."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14597_b200 as isb  # noqa: E402
from bench import REPLICAS, build_layers  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
path = sys.argv[2] if len(sys.argv) > 2 else "integer-scale"
dev = torch.device("cuda:0")
layers, xs = build_layers(isb, m, dev, seed=1234)
plans = [isb.GroupedGemm([{"weight": l[3], "x": x} for l, x in zip(layers[r], xs)], path=path)
         for r in range(REPLICAS)]
for i in range(12):
    plans[i % REPLICAS].run()
torch.cuda.synchronize()
print("done", plans[0].grid)
