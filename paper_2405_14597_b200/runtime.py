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
mode="grouped" (the default when every weight qualifies) replaces the 2 x L kernels by ONE grouped layer launch
(ops.GroupedGemm: K1 folded in, all linears' tiles spread over the SMs): H2D of
every input -> grouped launch -> D2H of every output. mode="pipelined" launches one single-problem grouped kernel
per linear (K1 folded in) in the fork/join pattern above, so the PCIe transfers
— 2.85 MB per LLaMA-2-7B decode step, more than the kernels' time — overlap the
GEMMs: linear i computes while input i+1 lands and output i-1 leaves (measured
slower than "grouped" at the LLaMA-2-7B decode shapes: each copy node and launch
carries its own fixed cost; kept for layers whose transfers dwarf the kernels).
`run()` replays it; the caller writes new activations into `host_inputs[i]`
before a step and reads `host_outputs[i]` after `synchronize()`.
"""
from __future__ import annotations

import torch

from . import ops


class GraphedLinears:
    def __init__(self, weights, m: int, in_dtype=torch.float32, out_dtype=torch.bfloat16,
                 path: str = "integer-scale", device=None, fused: bool = False,
                 mode: str = "auto"):
        """weights: list of PackedWeight (one per linear); m: tokens per step.
        mode: "grouped" (one launch per step), "pipelined" (one grouped launch per
        linear, transfers overlapped), "per-linear" (K1 + K3 per linear, or the
        single-GEMM fused kernel with fused=True) or "auto" (grouped when there are
        at most 8 linears, all with group 128)."""
        self.weights = list(weights)
        if mode == "auto":
            mode = "grouped" if (not fused and len(self.weights) <= 8 and
                                 all(w.group == 128 and w.k % 128 == 0 for w in self.weights)) \
                else "per-linear"
        self.mode = mode
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
        self.grouped = None
        self.singles = None
        if mode == "pipelined":
            self.singles = [ops.GroupedGemm([{"weight": w, "x": x, "xq": q, "sa": sa, "out": o}],
                                            path=path, out_dtype=out_dtype)
                            for w, x, q, sa, o in zip(self.weights, self.x, self.q, self.sa,
                                                      self.out)]
            self.kernels_per_run = len(self.weights)
        elif mode == "grouped":
            self.grouped = ops.GroupedGemm(
                [{"weight": w, "x": x, "xq": q, "sa": sa, "out": o}
                 for w, x, q, sa, o in zip(self.weights, self.x, self.q, self.sa, self.out)],
                path=path, out_dtype=out_dtype)
            self.kernels_per_run = 1
        else:
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
        if self.grouped is not None:
            # every input on its own copy (copy engine), then the one layer launch,
            # then the outputs back
            h2d.wait_stream(main)
            with torch.cuda.stream(h2d):
                for i in range(len(self.weights)):
                    self.x[i].copy_(self.host_inputs[i], non_blocking=True)
            main.wait_stream(h2d)
            self.grouped.run(stream=main)
            d2h.wait_stream(main)
            with torch.cuda.stream(d2h):
                for i in range(len(self.weights)):
                    self.host_outputs[i].copy_(self.out[i], non_blocking=True)
            main.wait_stream(d2h)
            return
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
            if self.singles is not None:
                self.singles[i].run(stream=main)
            elif self.fused:
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
