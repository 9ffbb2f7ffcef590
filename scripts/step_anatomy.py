"""Where the decode layer step's time goes: graphs of (K1+K3) x 4, K3 x 4, K1 x 4,
on the bench's rotated layer replicas (weights stream from HBM)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402

dev = torch.device("cuda:0")
torch.cuda.set_device(dev)
m = int(os.environ.get("M", "16"))
layers, xs = bench.build_layers(isb, m, dev, seed=1234)
q = [torch.empty((m, k), dtype=torch.int8, device=dev) for _, k, _ in bench.LAYER]
sa = [torch.empty((m,), dtype=torch.float64, device=dev) for _ in bench.LAYER]
out = [torch.empty((m, n), dtype=torch.bfloat16, device=dev) for _, _, n in bench.LAYER]
wsp = isb.Workspace()


def k1(i):
    isb.quantize_per_token(xs[i], codes=q[i], scales=sa[i])


def k3(r, i):
    isb.gemm_integer_scale(q[i], sa[i], layers[r][i][3], out=out[i], workspace=wsp)


def timed(body, reps=30):
    body()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                body()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1000 / reps)
    return best


def fz(r, i):
    isb.gemm_act_fused(xs[i], layers[r][i][3], out=out[i], sa_out=sa[i], workspace=wsp)


def fused():
    for r in range(3):
        for i in range(4):
            fz(r, i)


def full():
    for r in range(3):
        for i in range(4):
            k1(i)
            k3(r, i)


def k3only():
    for r in range(3):
        for i in range(4):
            k3(r, i)


def k1only():
    for r in range(3):
        for i in range(4):
            k1(i)


for i in range(4):
    k1(i)
res = {}
if not os.environ.get("NO_FUSED"):
    res["fused"] = timed(fused, 10) / 3
res = {**res, "full": timed(full, 10) / 3, "k3only": timed(k3only, 10) / 3, "k1only": timed(k1only, 10) / 3}
for i, (name, k, n) in enumerate(bench.LAYER):
    res[f"k3_{name}"] = timed(lambda: [k3(r, i) for r in range(3)], 10) / 3
    res[f"k1_{name}"] = timed(lambda: k1(i), 30)
    res[f"k1k3_{name}"] = timed(lambda: [(k1(i), k3(r, i)) for r in range(3)], 10) / 3
    if not os.environ.get("NO_FUSED"):
        res[f"fused_{name}"] = timed(lambda: [fz(r, i) for r in range(3)], 10) / 3
print({k: round(v, 2) for k, v in res.items()})
