"""Prefill fold: the CTA-pair kernel (gemm_sp.cu, default at M >= 512) vs the 1-CTA SS kernel
(gemm_fold.cu, forced with debug flag 1<<22) on the LLaMA-2-7B layer at M (default 2048): bit-identical outputs
(int32 / bf16) and per-linear kernel times. python pair_quick.py [M] [extra flags...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402
from paper_2405_14597_b200 import _lib  # noqa: E402

SS = 1 << 22
PAIR = 0
dev = torch.device("cuda:0")
m = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
extra = [int(a) for a in sys.argv[2:]]
layers, _ = bench.build_layers(isb, 16, dev, 1)
lib = _lib.load()
torch.manual_seed(1)
xq = [isb.quantize_per_token(torch.randn((m, k), device=dev)) for _, k, _ in bench.LAYER]
ws = [t[3] for t in layers[0]]
for dt in (torch.int32, torch.bfloat16):
    for (q, sa), w, (name, k, n) in zip(xq, ws, bench.LAYER):
        lib.isb_debug_set_flags(SS)
        a = isb.gemm_integer_scale(q, sa, w, out_dtype=dt)
        lib.isb_debug_set_flags(PAIR)
        b = isb.gemm_integer_scale(q, sa, w, out_dtype=dt)
        torch.cuda.synchronize()
        same = torch.equal(a, b)
        print(f"{name} {dt}: pair == ss: {same}", flush=True)
        if not same:
            d = (a != b).nonzero()
            print("  first diffs", d[:8].tolist(), "count", d.shape[0])
for fl in [SS, PAIR] + [PAIR | e for e in extra]:
    lib.isb_debug_set_flags(fl)
    ti = bench.gemm_kernel_timing(isb, layers, xq, m, "int", iters=20)
    tot = sum(r["us"] for r in ti)
    ops = sum(2 * m * k * n for _, k, n in bench.LAYER)
    print(f"flags={fl:#x} M={m}", " ".join(f"{r['linear']}={r['us']:.1f}" for r in ti),
          f"layer={tot:.1f} us = {ops / tot / 1e6:.0f} TOPS", flush=True)
lib.isb_debug_set_flags(0)
