"""Grouped decode launch, LLaMA-2-7B layer: integer vs float scale, us per layer at several M."""
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
for m in [int(a) for a in sys.argv[1:]] or [1, 16, 32, 64]:
    xs = [torch.randn((m, k), device=dev) for _, k, _ in bench.LAYER]
    it, _ = bench.grouped_layer_us(isb, layers, xs, "integer-scale")
    fl, _ = bench.grouped_layer_us(isb, layers, xs, "float-scale")
    print(f"M={m}: int {it:.2f} us, float {fl:.2f} us, int/float speedup {fl / it:.3f}", flush=True)
