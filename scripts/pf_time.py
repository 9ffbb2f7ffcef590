"""Grouped prefill launch of the LLaMA-2-7B layer's 4 linears at M (default 2048):
us per layer for each debug-knob value given (isb_debug_set_flags), 3 repeats each.
python pf_time.py [M] [flags...]   (ISB_LIB_PATH selects a library variant)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402
from paper_2405_14597_b200 import _lib  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
flags = [int(a) for a in sys.argv[2:]] or [0]
dev = torch.device("cuda:0")
lib = _lib.load()
layers, _ = bench.build_layers(isb, 16, dev, 1234)
xq = [isb.quantize_per_token(torch.randn((m, k), device=dev)) for _, k, _ in bench.LAYER]
ops = sum(2 * m * k * n for _, k, n in bench.LAYER)
for fl in flags:
    lib.isb_debug_set_flags(fl)
    r = [bench.grouped_prefill_us(isb, layers, xq)[0] for _ in range(3)]
    lib.isb_debug_set_flags(0)
    print(f"M={m} flags={fl}: " + " ".join(f"{u:.1f}" for u in r) + f" us = {ops / min(r) / 1e6:.0f} TOPS", flush=True)
