"""Where the e2e step goes: graphs of (H2D + K1/K3 + D2H) variants for the bench layer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2405_14597_b200 as isb  # noqa: E402
from paper_2405_14597_b200.runtime import GraphedLinears  # noqa: E402

dev = torch.device("cuda:0")
m = 16
layers, xs = bench.build_layers(isb, m, dev, seed=1234)


def run(variant):
    gs = []
    for r in range(3):
        g = GraphedLinears([l[3] for l in layers[r]], m, device=dev)
        for j, x in enumerate(xs):
            g.host_inputs[j].copy_(x.cpu())
        if variant == "no_h2d":   # inputs from device buffers (D2D copies) instead of host
            g.host_inputs = [t.to(dev) for t in g.host_inputs]
        elif variant == "no_d2h":  # outputs to device buffers instead of host
            g.host_outputs = [torch.empty_like(t, device=dev) for t in g.host_outputs]
        gs.append(g.capture())
    ms = bench.time_steps(lambda i: gs[i % 3].run(), 500, 20, 1) / 500
    return ms * 1e3


for v in ["full", "no_h2d", "no_d2h"]:
    print(v, round(run(v), 2), "us/step", flush=True)
