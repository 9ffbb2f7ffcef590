"""gate_up prefill K3 time with measurement knobs (isb_debug_set_flags): python prefill_dbg.py M flags..."""
import ctypes as C
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402
from paper_2405_14597_b200 import _lib  # noqa: E402

dev = torch.device("cuda:0")
m = int(sys.argv[1])
layers, _ = bench.build_layers(isb, 16, dev, 1)
lib = _lib.load()
for fl in [int(a) for a in sys.argv[2:]] or [0]:
    lib.isb_debug_set_flags(fl)
    xq = [isb.quantize_per_token(torch.randn((m, k), device=dev)) for _, k, _ in bench.LAYER]
    ti = bench.gemm_kernel_timing(isb, layers, xq, m, "int", iters=10)
    print(f"flags={fl} M={m}", " ".join(f"{r['linear']}={r['us']:.1f}" for r in ti),
          f"layer={sum(r['us'] for r in ti):.1f}")
lib.isb_debug_set_flags(0)
