"""Debug timeline of the decode kernel (globaltimer ns per role event).
Usage: python scripts/trace_decode.py M K N [cta]"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402
from paper_2405_14597_b200 import _lib  # noqa: E402

m, k, n = (int(a) for a in sys.argv[1:4])
cta = int(sys.argv[4]) if len(sys.argv) > 4 else 0
dev = torch.device("cuda:0")
gen = torch.Generator(device=dev)
gen.manual_seed(0)
ws = []
for _ in range(3):
    wf = bench.llama_like_weight(k, n, gen, dev)
    codes, scales = isb.quantize_weight(wf, 128, 4)
    s = isb.integerize_scales(scales.cpu().numpy(), 1024)
    ws.append(isb.PackedWeight.from_codes(codes, 128, scales, s.int_scales, 1024))
q, sa = isb.quantize_per_token(torch.randn((m, k), device=dev))
out = torch.empty((m, n), dtype=torch.bfloat16, device=dev)
for i in range(4):
    isb.gemm_integer_scale(q, sa, ws[i % 3], out=out)
torch.cuda.synchronize()
tr = torch.zeros((32, 512), dtype=torch.int64, device=dev)
lib = _lib.load()
lib.isb_debug_set_trace.argtypes = [C.c_void_p, C.c_int]
lib.isb_debug_set_trace(C.c_void_p(tr.data_ptr()), cta)
isb.gemm_integer_scale(q, sa, ws[1], out=out)
torch.cuda.synchronize()
lib.isb_debug_set_trace(None, 0)
t = tr.cpu()
c0 = int(t[10][0])
def row(r):
    return [int(x) - c0 if int(x) else None for x in t[r].tolist()]
print("cycles: entry", row(10)[1], "setup done", row(10)[0] and 0, "pre issued", row(10)[2], "pdl done", row(10)[3], "end", row(10)[4])
prod = row(0)
st0, ae, ld, xf, mma, epi = row(11), row(12), row(7), row(1), row(2), row(3)
for j in range(0, 512):
    if st0[j] is None:
        break
    print(f"step {j:3d} issue(b{2*j}) {prod[2*j] if 2*j < 512 else None} xf: start {st0[j]} a_empty {ae[j]} "
          f"loaded+stored {ld[j]} a_full {xf[j]} | mma {mma[j]} | epi {epi[j]}")
for sgi in range(8):
    a, b = row(4)[sgi], row(5)[sgi]
    if a is not None or b is not None:
        print(f"seg {sgi}: epilogue done {a}   fixup #{sgi} got {row(6)[sgi]} reduced {row(8)[sgi]} counted {row(9)[sgi]} finalised {b}")
