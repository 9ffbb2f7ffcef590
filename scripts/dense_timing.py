"""Layer time of the dense fp16 baseline (isb_gemm_dense) vs cuBLAS (torch.matmul) for
the LLaMA-2-7B linears at decode and prefill M; CUDA graphs, 3 rotating weight replicas."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402

dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
ws = [[(torch.randn((n, k), device=dev) * 0.02).half() for _, k, n in bench.LAYER] for _ in range(3)]


def timed(body, reps):
    body()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                body()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1000 / reps)
    return best


for m in [int(a) for a in (sys.argv[1:] or ["16", "2048"])]:
    xs = [torch.randn((m, k), device=dev).half() for _, k, _ in bench.LAYER]
    outs = [torch.empty((m, n), device=dev, dtype=torch.float16) for _, _, n in bench.LAYER]
    res = {}
    for name, fn in (("isb_dense", lambda r, i: isb.gemm_dense(xs[i], ws[r][i], out=outs[i])),
                     ("cublas", lambda r, i: torch.matmul(xs[i], ws[r][i].t(), out=outs[i]))):
        per = []
        for i in range(4):
            per.append(timed(lambda: [fn(r, i) for r in range(3)], 4 if m > 256 else 10) / 3)
        res[name] = [round(v, 2) for v in per] + [round(sum(per), 2)]
    flops = sum(2 * m * k * n for _, k, n in bench.LAYER)
    print(f"M={m}", {k: (v, round(flops / v[-1] / 1e6, 1)) for k, v in res.items()}, "(us per linear, layer, TFLOP/s)")
