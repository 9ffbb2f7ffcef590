"""Timeline of the CTA-pair prefill kernel (cluster 0, clock64): per 128-K block the MMA
warp's a_full / xfull wait completion and issue end, the transform's wfull / a_empty
waits, the epilogue's d_full / release. Usage: python trace_pair.py [M K N] [flags]
Needs a library built with the timeline compiled in (the product build has none):
  scripts/build_sp_variant.sh 10 8 $PWD/scripts/_var/sp_trace.so -DISB_SP_TRACE=1
  ISB_LIB_PATH=$PWD/scripts/_var/sp_trace.so python scripts/trace_pair.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402
from paper_2405_14597_b200 import _lib  # noqa: E402

m, k, n = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (2048, 4096, 22016)
flags = int(sys.argv[4]) if len(sys.argv) > 4 else 0
dev = torch.device("cuda:0")
gen = torch.Generator(device=dev)
gen.manual_seed(0)
wf = bench.llama_like_weight(k, n, gen, dev)
codes, scales = isb.quantize_weight(wf, 128, 4)
s = isb.integerize_scales(scales.cpu().numpy(), 1024)
w = isb.PackedWeight.from_codes(codes, 128, scales, s.int_scales, 1024)
q, sa = isb.quantize_per_token(torch.randn((m, k), device=dev))
out = torch.empty((m, n), dtype=torch.bfloat16, device=dev)
lib = _lib.load()
lib.isb_debug_set_flags(flags | int(os.environ.get('ISB_AB_FLAG', 0)))
for _ in range(3):
    isb.gemm_integer_scale(q, sa, w, out=out)
torch.cuda.synchronize()
tr = torch.zeros((48, 512), dtype=torch.int64, device=dev)
lib.isb_debug_set_trace.argtypes = [C.c_void_p, C.c_int]
lib.isb_debug_set_trace(C.c_void_p(tr.data_ptr()), 0)
isb.gemm_integer_scale(q, sa, w, out=out)
torch.cuda.synchronize()
lib.isb_debug_set_trace(None, 0)
lib.isb_debug_set_flags(0)
t = tr.cpu().numpy()
kb = k // 128
nb = int((t[2] != 0).sum())
t0 = t[2][0] - 1
print(f"M={m} K={k} N={n} flags={flags:#x}: {nb} blocks traced on the leader MMA warp")
iss = t[2][:nb]
d = np.diff(iss)
print(f"MMA issue-to-issue per block: median {np.median(d):.0f} cyc, mean {d.mean():.0f} "
      f"(ideal 512 at 256 tokens, 384 at 192)")
print("issue-to-issue percentiles 10/25/50/75/90/99: " + " ".join(f"{np.percentile(d, q):.0f}" for q in (10, 25, 50, 75, 90, 99)))
big = np.nonzero(d > 800)[0] + 1
if len(big):
    wb = t[0][big] - t[2][big - 1]
    wxx = t[1][big] - t[0][big]
    wi = t[2][big] - t[1][big]
    print(f"{len(big)} of {len(d)} intervals > 800 cyc: bfull wait {np.median(wb):.0f}, xfull wait {np.median(wxx):.0f}, "
          f"issue {np.median(wi):.0f} (medians); at kb: {np.bincount(big % kb, minlength=kb)[:8].tolist()} ...")
wa = t[0][1:nb] - t[2][:nb - 1]
wx = t[1][1:nb] - t[0][1:nb]
print(f"MMA waiting a_full after prev issue: median {np.median(wa):.0f}, mean {wa.mean():.0f}; "
      f"then xfull: median {np.median(wx):.0f}, mean {wx.mean():.0f}")
for r, lab in ((5, "leader xform arrive"), (21, "peer xform arrive")):
    x = t[r][t[r] != 0]
    if len(x) > 2:
        dd = np.diff(x[:nb])
        print(f"{lab:26s}: per-block interval median {np.median(dd):.0f}, mean {dd.mean():.0f}")
ph = [t[r] for r in (8, 9, 10, 11, 12, 5)]
ok = np.all([x != 0 for x in ph], axis=0)
if ok.sum():
    names = ["wfull->lds+release", "->fold done", "->a_empty ok", "->stores+fence", "->arrived"]
    for i, nm in enumerate(names):
        d = (ph[i + 1] - ph[i])[ok]
        print(f"xform phase {nm:22s}: median {np.median(d):.0f} mean {d.mean():.0f}")
    gap = (t[8][1:] - t[5][:-1])
    w = np.nonzero(ok)[0]
    st = np.diff(t[8][w])
    print(f"xform iteration start-to-start (same warp): median {np.median(st):.0f}")
print("first 12 blocks (rel. cycles): j, mma_afull, mma_xfull, mma_issued")
for j in range(min(12, nb)):
    print(j, *(int(t[r][j] - t0) if t[r][j] else -1 for r in (0, 1, 2)))
e8, e9, e10, e11 = t[8], t[9], t[10], t[11]
okc = (e8 != 0) & (e9 != 0) & (e10 != 0) & (e11 != 0)
if okc.sum() > 4:
    print(f"epilogue chunk (warp 0): tmem ld {np.median((e9 - e8)[okc]):.0f}, convert {np.median((e10 - e9)[okc]):.0f}, "
          f"pack+stage+store {np.median((e11 - e10)[okc]):.0f}, next chunk start {np.median((e8[1:] - e11[:-1])[okc[:-1] & (e8[1:] != 0)]):.0f} (medians, cycles)")
# fast bf16 epilogue path (warp ew 0): rows 8/9/10/11 at index 4*it and 8/9 at 4*it+1
ii = [i for i in range(0, 120) if t[8][4 * i] and t[9][4 * i] and t[10][4 * i] and t[11][4 * i] and t[8][4 * i + 1] and t[9][4 * i + 1]]
if len(ii) > 2:
    e = lambda r, o: np.array([t[r][4 * i + o] for i in ii], dtype=np.int64)
    ld, ca, sa_, cb, sb = e(9, 0) - e(8, 0), e(10, 0) - e(9, 0), e(11, 0) - e(10, 0), e(8, 1) - e(11, 0), e(9, 1) - e(8, 1)
    print(f"fast epilogue per tile (warp 0, medians, cycles): ld+release {np.median(ld):.0f}, convert A {np.median(ca):.0f}, "
          f"store A {np.median(sa_):.0f}, convert B {np.median(cb):.0f}, store B {np.median(sb):.0f}; "
          f"tile starts {[int(t[8][4 * i] - t0) for i in ii[:6]]}")
    if t[3][ii[0]]:
        c1 = np.array([t[3][i] for i in ii]) - e(9, 0)
        print(f"  convert A twice: first pass {np.median(c1):.0f}, second {np.median(e(10, 0) - np.array([t[3][i] for i in ii])):.0f}")
for base, who in ((12, "leader"), (28, "peer")):
    x12, x13, x14, x15 = t[base], t[base + 1], t[base + 2], t[base + 3]
    okx = (x12 != 0) & (x15 != 0)
    if okx.sum() > 4:
        print(f"transform warp 4 ({who}): wait W {np.median((x13 - x12)[okx]):.0f}, wait B slot free "
              f"{np.median((x14 - x13)[okx]):.0f}, expand+store+arrive {np.median((x15 - x14)[okx]):.0f}, "
              f"iteration {np.median(np.diff(x12[okx])):.0f} (medians, cycles)")
# leader warp 4 handles blocks j = 6u; its B slot frees when block j - NB completes
NB = int(os.environ.get("ISB_SP_NB_TRACE", 8))
x14, x15 = t[14], t[15]
us = [u for u in range(1, 512) if x14[u] and 6 * u - NB >= 0 and 6 * u < nb]
if us:
    dd = [x14[u] - t[2][6 * u - NB] for u in us]
    da = [t[0][6 * u] - x15[u] for u in us if x15[u]]
    print(f"issue(j-NB) -> slot free seen by warp (j): median {np.median(dd):.0f}; "
          f"warp arrive(j) -> MMA bfull(j) passed: median {np.median(da):.0f} (cycles, NB={NB})")
# globaltimer rows (ns): 32 + 2*row + cta; row 0 MMA passed bfull(j) (leader), 1 B slot free
# seen by the transform warp of j, 2 transform arrive(j), 3 MMA issued j (leader)
g = lambda row, cta: t[32 + 2 * row + cta]
jj = np.arange(8, min(nb, 500))
ok = (g(0, 0)[jj] != 0) & (g(2, 0)[jj] != 0) & (g(2, 1)[jj] != 0) & (g(1, 1)[jj] != 0)
jj = jj[ok]
if len(jj) > 4:
    med = lambda a: float(np.median(a))
    print(f"globaltimer ns (medians over {len(jj)} blocks): leader arrive -> MMA pass {med(g(0,0)[jj]-g(2,0)[jj]):.0f}, "
          f"peer arrive -> MMA pass {med(g(0,0)[jj]-g(2,1)[jj]):.0f}; "
          f"issue(j-NB) -> slot free at leader {med(g(1,0)[jj]-g(3,0)[jj-NB]):.0f} / peer {med(g(1,1)[jj]-g(3,0)[jj-NB]):.0f}; "
          f"slot free -> arrive leader {med(g(2,0)[jj]-g(1,0)[jj]):.0f} / peer {med(g(2,1)[jj]-g(1,1)[jj]):.0f}; "
          f"MMA pass -> issued {med(g(3,0)[jj]-g(0,0)[jj]):.0f}; issue-to-issue {med(np.diff(g(3,0)[jj])):.0f}")
ne = int((t[6] != 0).sum())
for it in range(min(ne, 6)):
    tile_end = t[2][(it + 1) * kb - 1] if (it + 1) * kb - 1 < nb else 0
    print(f"tile {it}: last issue {tile_end - t0}, d_full seen {t[6][it] - t0}, released {t[7][it] - t0}, "
          f"next first issue {t[2][(it + 1) * kb] - t0 if (it + 1) * kb < nb else -1}")
