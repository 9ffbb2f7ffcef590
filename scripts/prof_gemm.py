"""Tiny driver for ncu captures of one kernel: K3/K4 on a single shape, weights
rotated over 3 replicas. Usage: python scripts/prof_gemm.py M K N [int|float] [iters]
(ISB_ALPHA=8192 for the general per-group integer path, k_g up to ~124)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402

m, k, n = (int(a) for a in sys.argv[1:4])
path = sys.argv[4] if len(sys.argv) > 4 else "int"
iters = int(sys.argv[5]) if len(sys.argv) > 5 else 6
dev = torch.device("cuda:0")
if os.environ.get('ISB_AB_FLAG'):
    from paper_2405_14597_b200 import _lib
    _lib.load().isb_debug_set_flags(int(os.environ['ISB_AB_FLAG']))
gen = torch.Generator(device=dev)
gen.manual_seed(0)
ws = []
for _ in range(3):
    wf = bench.llama_like_weight(k, n, gen, dev)
    codes, scales = isb.quantize_weight(wf, 128, 4)
    alpha = int(os.environ.get("ISB_ALPHA", "1024"))
    s = isb.integerize_scales(scales.cpu().numpy(), alpha)
    ws.append(isb.PackedWeight.from_codes(codes, 128, scales, s.int_scales, alpha))
q, sa = isb.quantize_per_token(torch.randn((m, k), device=dev))
gemm = isb.gemm_integer_scale if path == "int" else isb.gemm_float_scale
out = torch.empty((m, n), dtype=torch.bfloat16, device=dev)
wsp = isb.Workspace()
for i in range(iters):
    gemm(q, sa, ws[i % 3], out=out, workspace=wsp)
torch.cuda.synchronize()
print("done")
