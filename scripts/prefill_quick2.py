"""Prefill M=2048 LLaMA-2-7B layer: folded K3 vs per-group K3 (same skeleton as K4) vs
K4, alpha 1024 and 8192; us per layer (graph of launches, weights rotated)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14597_b200 as isb  # noqa: E402
from bench import LAYER, llama_like_weight  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
dev = torch.device("cuda:0")
gen = torch.Generator(device=dev)
gen.manual_seed(5)
res = {}
for amp in (1024, 8192):
    ws = []
    for _, k, n in LAYER:
        wf = llama_like_weight(k, n, gen, dev)
        codes, scales = isb.quantize_weight(wf, 128, 4)
        si = isb.integerize_scales(scales.cpu().numpy(), amp)
        ws.append(isb.PackedWeight.from_codes(codes, 128, scales, si.int_scales, amp))
    xq = [isb.quantize_per_token(torch.randn((m, k), device=dev)) for _, k, _ in LAYER]
    outs = [torch.empty((m, n), dtype=torch.bfloat16, device=dev) for _, _, n in LAYER]
    for name, f in (("int", isb.gemm_integer_scale), ("float", isb.gemm_float_scale)):
        def run():
            for (q, sa), w, o in zip(xq, ws, outs):
                f(q, sa, w, out=o)
        run()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for _ in range(4):
                    run()
        torch.cuda.current_stream().wait_stream(s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 4
        ops = sum(2 * m * k * n for _, k, n in LAYER)
        print(f"alpha={amp} {name}: {us:.1f} us/layer  {ops / us / 1e6:.0f} TOPS "
              f"(max k_g {max(w.info["max_int_scale"] for w in ws)})",
              flush=True)
