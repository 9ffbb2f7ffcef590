"""Quick A/B of the grouped layer launch vs K1 + K3 per linear (LLaMA-2-7B layer,
weights rotated over 3 replicas). Prints us/layer for M in argv (default 1 16 64)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14597_b200 as isb  # noqa: E402
from bench import LAYER, REPLICAS, alg_bytes, build_layers  # noqa: E402


def graph_time(fn, iters=60, reps=5):
    fn(0)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(iters):
                fn(i)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / iters)
    return sorted(ts)[len(ts) // 2]


def main():
    dev = torch.device("cuda:0")
    ms = [int(a) for a in sys.argv[1:]] or [1, 16, 64]
    for m in ms:
        layers, xs = build_layers(isb, m, dev, seed=1234)
        byts = sum(alg_bytes(m, k, n) for _, k, n in LAYER)
        plans = {}
        for path in ("integer-scale", "float-scale"):
            plans[path] = [isb.GroupedGemm([{"weight": l[3], "x": x} for l, x in zip(layers[r], xs)],
                                           path=path) for r in range(REPLICAS)]
        q = [torch.empty((m, k), dtype=torch.int8, device=dev) for _, k, _ in LAYER]
        sa = [torch.empty((m,), dtype=torch.float64, device=dev) for _ in LAYER]
        outs = [torch.empty((m, n), dtype=torch.bfloat16, device=dev) for _, _, n in LAYER]

        def unfused(i, f=isb.gemm_integer_scale):
            for j, l in enumerate(layers[i % REPLICAS]):
                isb.quantize_per_token(xs[j], codes=q[j], scales=sa[j])
                f(q[j], sa[j], l[3], out=outs[j])

        t_g = graph_time(lambda i: plans["integer-scale"][i % REPLICAS].run())
        t_gf = graph_time(lambda i: plans["float-scale"][i % REPLICAS].run())
        t_u = graph_time(unfused)
        t_uf = graph_time(lambda i: unfused(i, isb.gemm_float_scale))
        p = plans["integer-scale"][0]
        print(f"M={m}: grouped int {t_g:.2f} us ({byts / t_g / 1e3:.0f} GB/s)  float {t_gf:.2f} us "
              f"| K1+K3 {t_u:.2f} us  K1+K4 {t_uf:.2f} us | grid {p.grid} C={p.cluster} "
              f"MT={p.tile_tokens} makespan {p.makespan_steps:.1f}", flush=True)


if __name__ == "__main__":
    main()
