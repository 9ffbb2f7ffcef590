"""Repeat the prefill GEMM on one shape and report where results differ from the first run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2405_14597_b200 as isb  # noqa: E402
from tests.instances import llama_problem  # noqa: E402

m, k, n = (int(a) for a in sys.argv[1:4])
x, w, s, _, _ = llama_problem(m, k, n, seed_w=5, seed_x=9)
dev = torch.device("cuda:0")
pw = isb.PackedWeight.from_codes(torch.from_numpy(w.values).to(dev), w.group,
                                 torch.from_numpy(w.scales).to(dev),
                                 torch.from_numpy(s.int_scales).to(dev), s.amplifier)
xq = torch.from_numpy(x.values.astype(np.int8)).to(dev)
sa = torch.from_numpy(x.scales).to(dev)
acc0 = isb.gemm_integer_scale(xq, sa, pw, out_dtype=torch.int32)
torch.cuda.synchronize()
bad = 0
for it in range(60):
    a = isb.gemm_integer_scale(xq, sa, pw, out_dtype=torch.int32)
    torch.cuda.synchronize()
    d = (a != acc0)
    if d.any():
        bad += 1
        idx = torch.nonzero(d)
        rows = idx[:, 0].unique().tolist()
        cols = idx[:, 1].unique().tolist()
        diff = (a.long() - acc0.long())[d]
        print(f"iter {it}: {int(d.sum())} diffs rows {rows[:10]}..({len(rows)}) cols {cols[:8]}..({len(cols)})"
              f" diff sample {diff[:6].tolist()}")
print("bad runs", bad, "of 60")
