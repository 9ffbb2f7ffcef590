"""Grouped layer launch anatomy (LLaMA-2-7B layer, M from argv[1]): time with the
measurement knobs (isb_debug_set_flags) and a per-CTA timeline (isb_debug_set_trace):
start, first activation ready, quantize-phase end, retire."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14597_b200 as isb  # noqa: E402
from paper_2405_14597_b200._lib import load  # noqa: E402
from bench import LAYER, REPLICAS, build_layers  # noqa: E402
from scripts.group_quick import graph_time  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
dev = torch.device("cuda:0")
lib = load()
lib.isb_debug_set_flags.argtypes = [C.c_int]
lib.isb_debug_set_trace.argtypes = [C.c_void_p, C.c_int]
layers, xs = build_layers(isb, m, dev, seed=1234)
for flags in ([0, 7] if len(sys.argv) < 3 else [int(a) for a in sys.argv[2:]]):
    lib.isb_debug_set_flags(flags)
    plans = [isb.GroupedGemm([{"weight": l[3], "x": x} for l, x in zip(layers[r], xs)])
             for r in range(REPLICAS)]
    t = graph_time(lambda i: plans[i % REPLICAS].run())
    print(f"flags={flags}: {t:.2f} us", flush=True)
lib.isb_debug_set_flags(0)
tr = torch.zeros((17, 512), dtype=torch.int64, device=dev)
lib.isb_debug_set_trace(tr.data_ptr(), 0)
plan = isb.GroupedGemm([{"weight": l[3], "x": x} for l, x in zip(layers[0], xs)])
lib.isb_debug_set_trace(None, 0)
plan.run()
torch.cuda.synchronize()
tr.zero_()
torch.cuda.synchronize()
plan.run()
torch.cuda.synchronize()
t = tr.cpu().numpy()[:, :plan.grid].astype(np.float64)
t0 = t[0].min()
rel = (t - t0) / 1e3
for name, row in zip(["start", "first X ready", "quantize end", "retire"], rel):
    v = row[row > -1e5]
    print(f"{name:14s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us")
print("retire percentiles", np.percentile(rel[3], [10, 25, 50, 75, 90, 100]).round(2))
dur = rel[3] - rel[0]
print("busy percentiles", np.percentile(dur, [0, 10, 25, 50, 75, 90, 100]).round(2))
order = np.argsort(rel[3])
print("earliest retire CTAs", order[:8], "latest", order[-8:])

# the same launch inside a back-to-back sequence (PDL): timeline relative to the
# traced grid's first CTA start
tr.zero_()
torch.cuda.synchronize()
for _ in range(3):
    plans[0].run()
    plans[1].run()
    plans[2].run()
plans[1].run()
plans[2].run()
plan.run()
plans[1].run()
torch.cuda.synchronize()
t = tr.cpu().numpy()[:, :plan.grid].astype(np.float64)
rel = (t - t[0].min()) / 1e3
print("in sequence:")
for name, row in zip(["start", "first X ready", "quantize end", "retire"], rel):
    v = row[row > -1e5]
    print(f"{name:14s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f} us")

# three consecutive traced grids (replicas 0, 1, 2), absolute timeline
lib.isb_debug_set_flags(int(os.environ.get("SEQ_FLAGS", "0")))
trs = [torch.zeros((17, 512), dtype=torch.int64, device=dev) for _ in range(3)]
tps = []
for r in range(3):
    lib.isb_debug_set_trace(trs[r].data_ptr(), 0)
    tps.append(isb.GroupedGemm([{"weight": l[3], "x": x} for l, x in zip(layers[r], xs)]))
lib.isb_debug_set_trace(None, 0)
lib.isb_debug_set_flags(0)
for _ in range(2):
    for r in range(3):
        tps[r].run()
for tt in trs:
    tt.zero_()
torch.cuda.synchronize()
for _ in range(2):
    for r in range(3):
        plans[r].run()
for r in range(3):
    tps[r].run()
torch.cuda.synchronize()
T = [tt.cpu().numpy()[:, :tps[0].grid].astype(np.float64) for tt in trs]
z = T[0][0].min()
print("consecutive grids (us from grid A's first CTA start):")
for r in range(3):
    a = (T[r] - z) / 1e3
    md = lambda i: f"{np.median(a[i]):6.2f}"
    print(f"  grid {r}: entry min {a[4].min():6.2f} med {md(4)} | setup done med {md(0)} | "
          f"\n           pdl released med {md(5)} max {a[5].max():6.2f} | 1st weights med {md(7)} | X ready med {md(1)} | "
          f"last handoff med {md(9)} | red: enter last {md(12)} pb_full {md(10)} reduced {md(11)} | exit med {md(6)} max {a[6].max():6.2f}")

a = (T[2] - z) / 1e3
ex = a[6]
order = np.argsort(ex)
print("exit spread: p10 %.2f p50 %.2f p90 %.2f max %.2f" % tuple(np.percentile(ex, [10, 50, 90, 100])))
print("latest CTAs:", [(int(c), round(float(ex[c] - np.median(ex)), 2), round(float(a[9][c] - np.median(a[9])), 2)) for c in order[-12:]])
print("earliest CTAs:", [(int(c), round(float(ex[c] - np.median(ex)), 2)) for c in order[:6]])
qt = int(np.sum([1 for _ in range(0)]))
print("median exit of CTAs < 64 (quantize rows): %.2f, >= 64: %.2f" % (np.median(ex[:64]), np.median(ex[64:])))
print("median last-handoff of CTAs < 64: %.2f, >= 64: %.2f" % (np.median(a[9][:64]), np.median(a[9][64:])))
print("median X-ready of CTAs < 64: %.2f, >= 64: %.2f" % (np.median(a[1][:64]), np.median(a[1][64:])))
med = np.median(ex)
for c in list(order[-6:]) + list(order[70:73]):
    print(f"CTA {int(c):3d}: handoff {a[9][c]-med:6.2f} red_pbfull {a[10][c]-med:6.2f} retire {a[3][c]-med:6.2f} exit {a[6][c]-med:6.2f} | Xready {a[1][c]-med:6.2f} 1stW {a[7][c]-med:6.2f}")
import ctypes
print("list lengths / items of late CTAs:")

cl = trs[2].cpu().numpy()[13:16, :tps[0].grid].astype(np.float64)
for c in list(order[-4:]) + list(order[70:72]):
    print(f"CTA {int(c):3d} clocks: retire-handoff {cl[1][c]-cl[0][c]:8.0f}  exit-retire {cl[2][c]-cl[1][c]:8.0f}")
