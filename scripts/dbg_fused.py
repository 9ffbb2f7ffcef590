"""Debug: fused act-quant GEMM vs quantize + GEMM on a few shapes."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2405_14597_b200 as isb
from oracle import oracle as O
from tests.instances import llama_problem
dev = torch.device("cuda:0")
for (m, k, n) in [(1, 4096, 4096), (5, 4096, 4096), (1, 4096, 12288), (5, 4096, 12288), (16, 4096, 8192), (16, 4096, 1024), (16, 4096, 256)]:
    x, w, s, xf, _ = llama_problem(m, k, n, seed_w=23 + n, seed_x=29 + m)
    pw = isb.PackedWeight.from_codes(torch.from_numpy(w.values).to(dev), 128, torch.from_numpy(w.scales).to(dev), torch.from_numpy(s.int_scales).to(dev), s.amplifier)
    xd = torch.from_numpy(xf).to(dev)
    q, sa = isb.quantize_per_token(xd)
    a = isb.gemm_integer_scale(q, sa, pw, out_dtype=torch.float32)
    b = isb.gemm_act_fused(xd, pw, out_dtype=torch.float32)
    torch.cuda.synchronize()
    bad = (a != b)
    print(m, k, n, "mismatch", int(bad.sum()), "of", a.numel(), "rows", sorted(set(torch.nonzero(bad)[:, 0].tolist()))[:8],
          "cols", torch.nonzero(bad)[:4, 1].tolist())
