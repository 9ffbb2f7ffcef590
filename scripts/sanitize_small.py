"""Small invocations of every kernel family for compute-sanitizer runs
(scripts/sanitize.sh runs memcheck, synccheck and racecheck over it)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_14597_b200 as isb  # noqa: E402
from oracle import oracle as O  # noqa: E402
from tests.instances import llama_problem  # noqa: E402

dev = torch.device("cuda:0")
# decode cluster kernel, prefill 1-CTA SS kernel, prefill CTA-pair kernel (ragged M and N)
for m, k, n in [(16, 1024, 384), (300, 1024, 256), (600, 512, 384)]:
    x, w, s, xf, _ = llama_problem(m, k, n)
    pw = isb.PackedWeight.from_codes(torch.from_numpy(w.values).to(dev), 128,
                                     torch.from_numpy(w.scales).to(dev),
                                     torch.from_numpy(s.int_scales).to(dev), s.amplifier)
    xq, sa = isb.quantize_per_token(torch.from_numpy(xf).to(dev))
    out = isb.gemm_integer_scale(xq, sa, pw, out_dtype=torch.float32)
    assert np.array_equal(out.cpu().numpy().view(np.int32), O.gemm_integer_scale(x, w, s).output.view(np.int32))
    isb.gemm_float_scale(xq, sa, pw)
# grouped decode launch (K1 fused) and grouped prefill launch (pair kernel)
from bench import llama_like_weight  # noqa: E402
gen = torch.Generator(device=dev)
gen.manual_seed(3)
ws = []
for k, n in [(512, 384), (1024, 256)]:
    c, sc = isb.quantize_weight(llama_like_weight(k, n, gen, dev), 128, 4)
    si = isb.integerize_scales(sc.cpu().numpy(), 1024)
    ws.append(isb.PackedWeight.from_codes(c, 128, sc, si.int_scales, 1024))
for mm in (16, 32, 48, 520):  # MT = 16 / 32 / 64 decode tiles, pair-kernel prefill
    g = isb.GroupedGemm([{"weight": w, "x": torch.randn((mm, w.k), device=dev)} for w in ws])
    g.run()
# per-group prefill kernel on the general integer path (alpha = 8192, k_g > 16)
x, w, _, xf, _ = llama_problem(600, 512, 384)
s8192 = O.integerize_scales(w.scales, 8192)
pw = isb.PackedWeight.from_codes(torch.from_numpy(w.values).to(dev), 128,
                                 torch.from_numpy(w.scales).to(dev),
                                 torch.from_numpy(s8192.int_scales).to(dev), s8192.amplifier)
xq, sa = isb.quantize_per_token(torch.from_numpy(xf).to(dev))
out = isb.gemm_integer_scale(xq, sa, pw, out_dtype=torch.float32)
assert np.array_equal(out.cpu().numpy().view(np.int32), O.gemm_integer_scale(x, w, s8192).output.view(np.int32))
xh = torch.randn((64, 512), device=dev).half()
wh = (torch.randn((384, 512), device=dev) * 0.02).half()
isb.gemm_dense(xh, wh)
isb.gemm_dense(torch.randn((300, 512), device=dev).half(), wh)
w8 = O.quantize(O.generate_llama_like(256, 64, 3), 8, O.SYMMETRIC, O.PER_CHANNEL, 0)
inner = isb.dual_inner_quantize(torch.from_numpy(w8.values).to(dev), 128)
x8, s8 = isb.quantize_per_token(torch.randn((4, 256), device=dev))
isb.gemm_dual_quant(x8, s8, inner, w8.scales)
torch.cuda.synchronize()
print("sanitize run ok")
