"""Per-launch time (CUDA graph, weights rotated) of the fused act-quant GEMM vs K1 + K3."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2405_14597_b200 as isb
dev = torch.device("cuda:0")
gen = torch.Generator(device=dev); gen.manual_seed(0)

def graph_time(fn, iters=30):
    fn(0); torch.cuda.synchronize()
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(iters):
                fn(i)
    torch.cuda.current_stream().wait_stream(s)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / iters

for (m, k, n) in [(16, 4096, 4096), (16, 4096, 22016), (16, 11008, 4096)]:
    ws = []
    for _ in range(3):
        wf = bench.llama_like_weight(k, n, gen, dev)
        codes, scales = isb.quantize_weight(wf, 128, 4)
        s = isb.integerize_scales(scales.cpu().numpy(), 1024)
        ws.append(isb.PackedWeight.from_codes(codes, 128, scales, s.int_scales, 1024))
    x = torch.randn((m, k), device=dev)
    q = torch.empty((m, k), dtype=torch.int8, device=dev); sa = torch.empty((m,), dtype=torch.float64, device=dev)
    out = torch.empty((m, n), dtype=torch.bfloat16, device=dev)
    wsp = isb.Workspace()
    t_f = graph_time(lambda i: isb.gemm_act_fused(x, ws[i % 3], out=out, sa_out=sa, workspace=wsp))
    t_u = graph_time(lambda i: (isb.quantize_per_token(x, codes=q, scales=sa), isb.gemm_integer_scale(q, sa, ws[i % 3], out=out, workspace=wsp)))
    t_g = graph_time(lambda i: isb.gemm_integer_scale(q, sa, ws[i % 3], out=out, workspace=wsp))
    t_q = graph_time(lambda i: isb.quantize_per_token(x, codes=q, scales=sa))
    print(f"M={m} K={k} N={n}: fused {t_f:.2f} us | K1+K3 {t_u:.2f} us | K3 only {t_g:.2f} | K1 only {t_q:.2f}")
