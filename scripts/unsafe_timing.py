"""Unsafe layer timing: LLaMA-2-70B down_proj shape (K = 28672, N = 8192, llama-like weights) with alpha = 32768 (argv[1])
(static bound > int32): the K-chunked exact tensor-core path (isb_gemm_integer_scale) vs
the scalar int64 checked kernel and the float-scale path. python unsafe_timing.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402

dev = torch.device("cuda:0")
K, N = 28672, 8192
AMP = int(sys.argv[1]) if len(sys.argv) > 1 else 32768  # alpha: 32768 makes this layer unsafe
g = torch.Generator(device=dev)
g.manual_seed(5)
wf = bench.llama_like_weight(K, N, g, dev)  # heavy-tailed channels, as the bench's weights
codes, scales = isb.quantize_weight(wf, 128, 4)
s = isb.integerize_scales(scales.cpu().numpy(), AMP)
pw = isb.PackedWeight.from_codes(codes, 128, scales, s.int_scales, AMP)
info = isb.overflow_analyzer(K, 128, 8, 4, s)
print(f"static bound {info['static_bound']} ({info['static_bound'] / 2**31:.2f} x int32), safe={info['safe']}")


def t(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


for m in (16, 2048):
    xq, sa = isb.quantize_per_token(torch.randn((m, K), device=dev))
    ti = t(lambda: isb.gemm_integer_scale(xq, sa, pw, out_dtype=torch.bfloat16))
    tf = t(lambda: isb.gemm_float_scale(xq, sa, pw, out_dtype=torch.bfloat16))
    tc = t(lambda: isb.gemm_checked("integer-scale", xq, sa, pw), iters=2)
    ops = 2 * m * K * N
    print(f"M={m}: integer (K-chunked exact) {ti:.1f} us ({ops / ti / 1e6:.0f} TOPS), "
          f"float-scale {tf:.1f} us, scalar checked {tc:.1f} us ({tc / ti:.0f}x)")
