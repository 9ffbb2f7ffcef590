"""Debug timeline of one CTA of the tcgen05 GEMM (clock64 per role event).
Usage: python scripts/trace_gemm.py M K N [cta]"""
import ctypes as C
import os
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
wsp = isb.Workspace()
for i in range(4):
    isb.gemm_integer_scale(q, sa, ws[i % 3], out=out, workspace=wsp)
torch.cuda.synchronize()
tr = torch.zeros((32, 512), dtype=torch.int64, device=dev)
lib = _lib.load()
lib.isb_debug_set_trace.argtypes = [C.c_void_p, C.c_int]
lib.isb_debug_set_trace(C.c_void_p(tr.data_ptr()), cta)
isb.gemm_integer_scale(q, sa, ws[1], out=out, workspace=wsp)
torch.cuda.synchronize()
lib.isb_debug_set_trace(None, 0)
t = tr.cpu()
t0 = int(t[7, 0])
names = ["prod_issue", "xform_data", "mma_commit", "xform_done", "epi_dready", "prod_start",
         "cta_end", "cta_start", "mma_dempty", "mma_full", "mma_afull", "xf_lds", "xf_aempty",
         "prod_empty"]
print(f"M={m} K={k} N={n} cta={cta}: end at {int(t[6,0]) - t0} ns, prod_start {int(t[5,0]) - t0}")
cnt = int((t[0] != 0).sum())
for i in range(cnt):
    cols = [13, 0, 1, 11, 12, 3, 8, 9, 10, 2, 4]
    row = {r: (int(t[r, i]) - t0 if int(t[r, i]) else -1) for r in cols}
    print(f"{i:3d} " + " ".join(f"{names[r]}={row[r]:6d}" for r in cols))
st = t[14][:148].tolist()
en = t[15][:148].tolist()
mn = min(x for x in st if x)
print("CTA start (ns rel. min): ", sorted([x - mn for x in st if x])[:5], "...", sorted([x - mn for x in st if x])[-5:])
print("CTA end   (ns rel. min): ", sorted([x - mn for x in en if x])[:5], "...", sorted([x - mn for x in en if x])[-5:])
import statistics
def rel(r):
    return [int(x) - mn if int(x) else None for x in t[r][:148].tolist()]
cols = {"start": rel(14), "prod_done": rel(18), "mma_done": rel(19), "epi_groups_done": rel(16),
        "fx_stored": rel(20), "fx_fenced": rel(21), "fx_counted": rel(22), "fx_reduced": rel(23),
        "epi_fixup_done": rel(17), "end": rel(15)}
for name, v in cols.items():
    vv = [x for x in v if x is not None]
    print(f"{name:16s} min {min(vv):6d} med {int(statistics.median(vv)):6d} max {max(vv):6d}")
slow = sorted(range(148), key=lambda i: -(cols['end'][i] or 0))[:6]
for i in slow:
    print("slow cta", i, {k: v[i] for k, v in cols.items()})
