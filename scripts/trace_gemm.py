"""Debug timeline of the tcgen05 GEMM (globaltimer per role event, ns).
Usage: python scripts/trace_gemm.py M K N [cta]"""
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
xfl0 = torch.randn((m, k), device=dev)
for i in range(3):
    isb.gemm_act_fused(xfl0, ws[i % 3], out=out)
torch.cuda.synchronize()
tr = torch.zeros((32, 512), dtype=torch.int64, device=dev)
lib = _lib.load()
lib.isb_debug_set_trace.argtypes = [C.c_void_p, C.c_int]
lib.isb_debug_set_trace(C.c_void_p(tr.data_ptr()), cta)
xfl = torch.randn((m, k), device=dev)
if os.environ.get("FUSED"):
    isb.gemm_act_fused(xfl, ws[1], out=out)
else:
    isb.gemm_integer_scale(q, sa, ws[1], out=out)
torch.cuda.synchronize()
lib.isb_debug_set_trace(None, 0)
t = tr.cpu()
st = [int(x) for x in t[14][:148].tolist()]
mn = min(x for x in st if x)
names = {0: "prod", 1: "xf_data", 3: "xf_done", 2: "mma", 4: "epi_d"}
cnt = int((t[0] != 0).sum())
print(f"M={m} K={k} N={n} cta={cta}: {cnt} steps; cta start {st[cta] - mn} end {int(t[15][cta]) - mn}")
for i in range(cnt):
    print(f"{i:3d} " + " ".join(f"{nm}={(int(t[r, i]) - mn) if int(t[r, i]) else -1:6d}"
                               for r, nm in names.items()))
en = [int(x) - mn for x in t[15][:148].tolist() if int(x)]
sv = [x - mn for x in st if x]
print("CTA start: min", min(sv), "max", max(sv), " CTA end: min", min(en), "med",
      int(statistics.median(en)), "max", max(en), " n", len(en))
for it in range(8):
    vals = [int(t[r, it]) - mn if int(t[r, it]) else -1 for r in (8, 6, 7, 7)]
    if vals[0] > 0:
        print(f"tile {it}: epi_done={vals[0]} red_start={vals[1]} red_done={vals[2]}")

print("fused prologue (ns): entry/pdl/pass1/exchange/pass2:", [int(t[9, i]) - mn if int(t[9, i]) else None for i in range(5)])
