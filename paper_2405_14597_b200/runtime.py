"""Graph-captured execution of a set of integer-scale W4A8 linears.

The reference runs each GEMM as a blocking host call (gemm.cpp:205-262 inside
run_layer, gemm.cpp:489-516). On B200 the per-call host cost (argument checks,
ctypes, tensor-map encode, launch) is ~15-20 us — several times the device time
of a decode-sized GEMM — so serving code records the whole sequence once and
replays it: GraphedLinears captures, for every linear,

    host pinned input  --H2D-->  device activations
    K1 per-token quantize  ->  K3 integer-scale GEMM (or K4 float-scale)
    device output      --D2H-->  host pinned output

into one CUDA graph (kernels chained with programmatic dependent launch; the
copies on their own streams so transfers overlap the GEMMs).
`run()` replays it; the caller writes new activations into `host_inputs[i]`
before a step and reads `host_outputs[i]` after `synchronize()`.
"""
from __future__ import annotations

import torch

from . import ops


class GraphedLinears:
    def __init__(self, weights, m: int, in_dtype=torch.float32, out_dtype=torch.bfloat16,
                 path: str = "integer-scale", device=None, fused: bool = False):
        """weights: list of PackedWeight (one per linear); m: tokens per step."""
        self.weights = list(weights)
        self.m = m
        self.device = torch.device(device if device is not None else self.weights[0].device)
        self.path = path
        self.fused = fused
        dev = self.device
        self.host_inputs = [torch.zeros((m, w.k), dtype=in_dtype).pin_memory() for w in weights]
        self.host_outputs = [torch.empty((m, w.n), dtype=out_dtype).pin_memory()
                             for w in weights]
        self.x = [torch.empty((m, w.k), dtype=in_dtype, device=dev) for w in weights]
        self.q = [torch.empty((m, w.k), dtype=torch.int8, device=dev) for w in weights]
        self.sa = [torch.empty((m,), dtype=torch.float64, device=dev) for _ in weights]
        self.out = [torch.empty((m, w.n), dtype=out_dtype, device=dev) for w in weights]
        self.ws = ops.Workspace()
        self.stream = torch.cuda.Stream(device=dev)
        self.h2d_stream = torch.cuda.Stream(device=dev)
        self.d2h_stream = torch.cuda.Stream(device=dev)
        self.graph = None
        self.kernels_per_run = (1 if fused else 2) * len(self.weights)
        self.h2d_bytes = sum(t.numel() * t.element_size() for t in self.host_inputs)
        self.d2h_bytes = sum(t.numel() * t.element_size() for t in self.host_outputs)

    def _record(self):
        """Fork/join over three streams so the graph overlaps transfers with compute:
        all input copies start at once (copy stream), linear i's kernels start when
        its input has landed (compute stream), and its output copy runs while
        linear i+1 computes (copy-back stream)."""
        gemm = ops.gemm_integer_scale if self.path == "integer-scale" else ops.gemm_float_scale
        main, h2d, d2h = self.stream, self.h2d_stream, self.d2h_stream
        h2d.wait_stream(main)
        d2h.wait_stream(main)
        landed = []
        with torch.cuda.stream(h2d):
            for i in range(len(self.weights)):
                self.x[i].copy_(self.host_inputs[i], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d)
                landed.append(ev)
        for i, w in enumerate(self.weights):
            main.wait_event(landed[i])
            if self.fused:
                ops.gemm_act_fused(self.x[i], w, path=self.path, out=self.out[i],
                                   sa_out=self.sa[i], workspace=self.ws, stream=main)
            else:
                ops.quantize_per_token(self.x[i], codes=self.q[i], scales=self.sa[i],
                                       stream=main)
                gemm(self.q[i], self.sa[i], w, out=self.out[i], workspace=self.ws, stream=main)
            done = torch.cuda.Event()
            done.record(main)
            d2h.wait_event(done)
            with torch.cuda.stream(d2h):
                self.host_outputs[i].copy_(self.out[i], non_blocking=True)
        main.wait_stream(h2d)
        main.wait_stream(d2h)

    def capture(self):
        torch.cuda.synchronize(self.device)
        with torch.cuda.stream(self.stream):
            self._record()  # warm-up: sizes the workspace, loads kernels
        torch.cuda.synchronize(self.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(self.stream):
            with torch.cuda.graph(self.graph, stream=self.stream):
                self._record()
        self.stream.synchronize()
        return self

    def run(self):
        """Enqueue one step (inputs from host_inputs, results to host_outputs)."""
        if self.graph is None:
            self.capture()
        self.graph.replay()

    def synchronize(self):
        torch.cuda.synchronize(self.device)
