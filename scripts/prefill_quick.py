"""Per-linear K3 / K4 timings of the LLaMA-2-7B layer at prefill sizes (graph-timed)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402

dev = torch.device("cuda:0")
ms = [int(a) for a in sys.argv[1:]] or [2048]
layers, _ = bench.build_layers(isb, 16, dev, 1)
for m in ms:
    xq = [isb.quantize_per_token(torch.randn((m, k), device=dev)) for _, k, _ in bench.LAYER]
    ti = bench.gemm_kernel_timing(isb, layers, xq, m, "int", iters=10)
    tf = bench.gemm_kernel_timing(isb, layers, xq, m, "float", iters=10)
    for a, b in zip(ti, tf):
        print(f"M={m} {a['linear']:8s} int {a['us']:8.2f} us {a['tops']:7.1f} TOPS | float {b['us']:8.2f} us"
              f" {b['tops']:7.1f} TOPS | speedup {b['us'] / a['us']:.3f}")
    ui, uf = sum(r["us"] for r in ti), sum(r["us"] for r in tf)
    ops = sum(2 * m * k * n for _, k, n in bench.LAYER)
    print(f"M={m} layer int {ui:.1f} us ({ops / ui / 1e6:.0f} TOPS)  float {uf:.1f} us  speedup {uf / ui:.3f}")
