import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from tests.instances import random_instance
import paper_2405_14597_b200 as isb
DEV = torch.device("cuda:0")
def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return (t.to(dtype) if dtype is not None else t).to(DEV)
rng = O.Rng(2718)
for it in range(20):
    m = 1 + rng.below(40); n = 1 + rng.below(300); k = 128 * (1 + rng.below(6)); g = [128, k][rng.below(2)]
    x, w, _, _ = random_instance(rng, m, k, n, g)
    amp = O.search_amplifier(w.scales); s = O.integerize_scales(w.scales, amp)
    if not O.overflow_analyzer(k, g, 8, 4, s)["safe"]:
        print(it, "unsafe skip"); continue
    ref = O.gemm_integer_scale(x, w, s)
    pw = isb.PackedWeight.from_codes(dev(w.values), g, dev(w.scales), dev(s.int_scales), s.amplifier)
    out = isb.gemm_integer_scale(dev(x.values, torch.int8), dev(x.scales), pw, out_dtype=torch.float32).cpu().numpy()
    bad = np.argwhere(out.view(np.int32) != ref.output.view(np.int32))
    print(it, f"m={m} n={n} k={k} g={g} amp={amp} maxk={s.int_scales.max()} bad={len(bad)}/{m*n}", bad[:5].tolist(),
          [(float(out[i, j]), float(ref.output[i, j])) for i, j in bad[:3]])
