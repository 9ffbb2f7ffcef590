"""Grouped decode launch (LLaMA-2-7B layer) with measurement knobs (isb_debug_set_flags,
gemm_group.cu: 1 no A stores, 2 no epilogue TMEM loads, 4 no MMAs, 256 no epilogue
stores / piece reduction): us per layer. python group_knobs.py M [flags...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402
from paper_2405_14597_b200 import _lib  # noqa: E402

dev = torch.device("cuda:0")
lib = _lib.load()
layers, _ = bench.build_layers(isb, 16, dev, 1234)
m = int(sys.argv[1])
xs = [torch.randn((m, k), device=dev) for _, k, _ in bench.LAYER]
for fl in [0] + [int(a) for a in sys.argv[2:]]:
    lib.isb_debug_set_flags(fl)
    us, _ = bench.grouped_layer_us(isb, layers, xs, "integer-scale")
    lib.isb_debug_set_flags(0)
    print(f"M={m} flags={fl}: {us:.2f} us", flush=True)
