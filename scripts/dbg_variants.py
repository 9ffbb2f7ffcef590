"""Time the tcgen05 GEMM with debug knobs that skip pieces of the pipeline."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402
from paper_2405_14597_b200 import _lib  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda:0")
gen = torch.Generator(device=dev)
gen.manual_seed(0)
for (m, k, n) in [(16, 4096, 4096), (16, 4096, 22016)]:
    ws = []
    for _ in range(3):
        wf = bench.llama_like_weight(k, n, gen, dev)
        codes, scales = isb.quantize_weight(wf, 128, 4)
        s = isb.integerize_scales(scales.cpu().numpy(), 1024)
        ws.append(isb.PackedWeight.from_codes(codes, 128, scales, s.int_scales, 1024))
    q, sa = isb.quantize_per_token(torch.randn((m, k), device=dev))
    out = torch.empty((m, n), dtype=torch.bfloat16, device=dev)
    wsp = isb.Workspace()
    for flags in [0, 1, 2, 4, 3, 7]:
        lib.isb_debug_set_flags(flags)
        for i in range(3):
            isb.gemm_integer_scale(q, sa, ws[i % 3], out=out, workspace=wsp)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i in range(30):
                isb.gemm_integer_scale(q, sa, ws[i % 3], out=out, workspace=wsp)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"M={m} K={k} N={n} flags={flags}: {e0.elapsed_time(e1) * 1000 / 30:.2f} us/launch")
    lib.isb_debug_set_flags(0)
