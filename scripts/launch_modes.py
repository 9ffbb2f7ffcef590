"""Per-launch time of K3 back-to-back: eager vs CUDA graph (PDL on/off via env)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402

dev = torch.device("cuda:0")
gen = torch.Generator(device=dev)
gen.manual_seed(0)
shapes = [(16, 4096, 4096), (16, 4096, 22016)] + ([(16, 4096, 131072)] if os.environ.get('BIG') else [])
for (m, k, n) in shapes:
    ws = []
    for _ in range(3):
        wf = bench.llama_like_weight(k, n, gen, dev)
        codes, scales = isb.quantize_weight(wf, 128, 4)
        s = isb.integerize_scales(scales.cpu().numpy(), 1024)
        ws.append(isb.PackedWeight.from_codes(codes, 128, scales, s.int_scales, 1024))
    q, sa = isb.quantize_per_token(torch.randn((m, k), device=dev))
    out = torch.empty((m, n), dtype=torch.bfloat16, device=dev)
    for i in range(3):
        isb.gemm_integer_scale(q, sa, ws[i % 3], out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(60):
        isb.gemm_integer_scale(q, sa, ws[i % 3], out=out)
    e1.record()
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) * 1000 / 60
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(60):
            isb.gemm_integer_scale(q, sa, ws[i % 3], out=out)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) * 1000 / 60
    gb = (n * k // 2 + 4 * n * k // 128) / graph / 1e3
    print(f"{gb:.0f} GB/s PDL={os.environ.get('ISB_NO_PDL') != '1'} M={m} K={k} N={n}: eager {eager:.2f} us, graph {graph:.2f} us")
