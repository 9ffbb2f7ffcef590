#!/usr/bin/env python3
"""Benchmark: integer-scale W4A8 fine-grained GEMM on B200 (BASELINE.json metric
"W4A8 IntScale GEMM TOPS & µs/layer vs roofline; speedup vs float-scale").

Workload (BASELINE.json configs[1]): the LLaMA-2-7B linear layers of one decoder
layer at decode M=16 tokens (q/k/v fused 4096->12288, o 4096->4096, gate/up fused
4096->22016, down 11008->4096), group 128, alpha 1024. One step = the hot path
over one layer: per-token int8 quantize of each linear's float32 input + the
integer-scale GEMM of every linear, as ONE grouped layer launch
(csrc/gemm_group.cu; K1 folded in, the 4 linears' tiles spread over all SMs).
The per-linear form (K1 + K3 per linear, 8 launches) is timed beside it.
Weights are rotated over 3 layer replicas (3 x 107.5 MB > 2 x 126 MB L2) so each
step streams its weights from HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import numpy as np
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "W4A8 IntScale GEMM TOPS & µs/layer vs roofline; speedup vs float-scale"
GROUP = 128
ALPHA = 1024
# LLaMA-2-7B decoder-layer linears (K, N), q/k/v and gate/up fused.
LAYER = [("qkv_proj", 4096, 12288), ("o_proj", 4096, 4096), ("gate_up_proj", 4096, 22016),
         ("down_proj", 11008, 4096)]
REPLICAS = 3


def alg_bytes(m, k, n, x_b=1, o_b=2):
    """SURVEY §8d / BASELINE.md: N*K/2 + 4*N*K/g + M*K*x_b + 8*M + M*N*o_b."""
    return n * k // 2 + 4 * n * k // GROUP + m * k * x_b + 8 * m + m * n * o_b


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], "measured"
    except Exception:
        return 6650.0, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock + throttle reasons via NVML while the timed region runs."""

    def __init__(self, index=0, period=0.005):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.max_mhz = None
        self._t = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            names = {
                "sw_power_cap": N.nvmlClocksThrottleReasonSwPowerCap,
                "hw_slowdown": N.nvmlClocksThrottleReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksThrottleReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksThrottleReasonSwThermalSlowdown,
                "hw_power_brake_slowdown": N.nvmlClocksThrottleReasonHwPowerBrakeSlowdown,
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
                        r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        for k, bit in names.items():
                            if r & bit:
                                self.reasons.add(k)
                    except Exception:
                        pass
                    time.sleep(self.period)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------- dist
def init_dist():
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, ws):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------------- data
def llama_like_weight(k, n, gen, dev):
    """Device synthetic weight with the reference llama_like structure
    (tensor_io.cpp:101-122): per (column, group of 128) a scale 2^u with
    u ~ U(-9.99, -6.05), values uniform in +-0.97*7*2^u and one anchor at +-7*2^u,
    so 4-bit group scales land in [2^-10, 2^-6] and alpha=1024 gives k_g in [1, 15]."""
    import torch
    g = k // GROUP
    u = -9.99 + (-6.05 + 9.99) * torch.rand((g, n), generator=gen, device=dev, dtype=torch.float64)
    vmax = (7.0 * torch.exp2(u)).float()                                    # [g, n]
    w = (2.0 * torch.rand((g, GROUP, n), generator=gen, device=dev) - 1.0) * 0.97 * vmax[:, None]
    anchor = torch.randint(0, GROUP, (g, n), generator=gen, device=dev)
    sign = torch.where(torch.rand((g, n), generator=gen, device=dev) < 0.5, -1.0, 1.0)
    w.scatter_(1, anchor[:, None, :], (sign * vmax)[:, None, :])
    return w.reshape(k, n).contiguous()


LAYER_L3_8B = [("qkv_proj", 4096, 6144), ("o_proj", 4096, 4096), ("gate_up_proj", 4096, 28672),
               ("down_proj", 14336, 4096)]   # BASELINE configs[2] (C3): LLaMA-3-8B


def build_layers(isb, m, dev, seed, shapes=None):
    import torch
    shapes = shapes or LAYER
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    layers = []
    for _ in range(REPLICAS):
        lin = []
        for name, k, n in shapes:
            wf = llama_like_weight(k, n, gen, dev)
            codes, scales = isb.quantize_weight(wf, GROUP, 4)          # device group quantizer
            del wf
            s = isb.integerize_scales(scales.cpu().numpy(), ALPHA)      # offline, host
            w = isb.PackedWeight.from_codes(codes, GROUP, scales, s.int_scales, ALPHA)
            w.group_scales = scales  # kept for re-integerizing at another amplifier
            del codes
            lin.append((name, k, n, w, int(s.int_scales.max())))
        layers.append(lin)
    xs = [torch.randn((m, k), generator=gen, device=dev, dtype=torch.float32) for _, k, _ in shapes]
    return layers, xs


# ----------------------------------------------------------------------------- ours
class LayerStep:
    """One step: per-token quantization + integer-scale (or float-scale) GEMM for
    every linear of one layer replica, captured into a CUDA graph per replica.
    fused=True: one launch per linear (K1 fused into K3/K4, config C3);
    fused=False: K1 then K3/K4 (two launches per linear)."""

    def __init__(self, isb, layers, xs, m, path, dev, fused=False):
        import torch
        self.isb, self.layers, self.xs, self.m, self.path = isb, layers, xs, m, path
        self.fused = fused
        self.q = [torch.empty((m, k), dtype=torch.int8, device=dev) for _, k, _ in LAYER]
        self.sa = [torch.empty((m,), dtype=torch.float64, device=dev) for _ in LAYER]
        self.out = [torch.empty((m, n), dtype=torch.bfloat16, device=dev) for _, _, n in LAYER]
        self.ws = [isb.Workspace() for _ in range(REPLICAS)]
        self.graphs = []
        self.kernels_per_step = (1 if fused else 2) * len(LAYER)

    def run_eager(self, r):
        isb = self.isb
        if self.fused:
            path = "integer-scale" if self.path == "int" else "float-scale"
            for i, (_, k, n, w, _) in enumerate(self.layers[r]):
                isb.gemm_act_fused(self.xs[i], w, path=path, out=self.out[i],
                                   sa_out=self.sa[i], workspace=self.ws[r])
            return
        gemm = isb.gemm_integer_scale if self.path == "int" else isb.gemm_float_scale
        for i, (_, k, n, w, _) in enumerate(self.layers[r]):
            q, sa = self.q[i], self.sa[i]
            isb.quantize_per_token(self.xs[i], codes=q, scales=sa)
            gemm(q, sa, w, out=self.out[i], workspace=self.ws[r])

    def capture(self):
        import torch
        for r in range(REPLICAS):
            self.run_eager(r)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for r in range(REPLICAS):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    self.run_eager(r)
                self.graphs.append(g)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()

    def replay(self, step):
        self.graphs[step % REPLICAS].replay()


def time_steps(fn, steps, warmup, ws):
    import torch
    for i in range(warmup):
        fn(i)
    torch.cuda.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for i in range(steps):
        fn(warmup + i)
    end.record()
    torch.cuda.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    return start.elapsed_time(end)  # ms


def gemm_kernel_timing(isb, layers, xq_sa, m, path, iters=30):
    """Average device duration of each K3 (or K4) launch: `iters` back-to-back launches
    rotating the weight replicas (weights stream from HBM), captured in a CUDA graph so
    host launch overhead is excluded, timed with CUDA events on the launching stream."""
    import torch
    gemm = isb.gemm_integer_scale if path == "int" else isb.gemm_float_scale
    res = []
    wsp = isb.Workspace()
    for i, (name, k, n) in enumerate(LAYER):
        q, sa = xq_sa[i]
        out = torch.empty((m, n), dtype=torch.bfloat16, device=q.device)
        for r in range(REPLICAS):
            gemm(q, sa, layers[r][i][3], out=out, workspace=wsp)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for it in range(iters):
                    gemm(q, sa, layers[it % REPLICAS][i][3], out=out, workspace=wsp)
        torch.cuda.current_stream().wait_stream(s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1000.0 / iters
        res.append({"linear": name, "M": m, "K": k, "N": n, "us": round(us, 3),
                    "alg_bytes": alg_bytes(m, k, n), "gbps": round(alg_bytes(m, k, n) / us / 1e3, 1),
                    "tops": round(2.0 * m * n * k / us / 1e6, 2)})
    return res


def dense_layer_timing(isb, m, dev, wd, iters=10):
    """Per-linear device time of the dense fp16 baseline (isb_gemm_dense, tcgen05
    kind::f16, no cuBLAS) on the same shapes: fp16 x [M][K], fp16 w [N][K] rotated over
    the replicas `wd`, CUDA graph, CUDA events."""
    import torch
    res = []
    for i, (name, k, n) in enumerate(LAYER):
        x = torch.randn((m, k), device=dev).half()
        out = torch.empty((m, n), dtype=torch.float16, device=dev)
        for r in range(len(wd)):
            isb.gemm_dense(x, wd[r][i], out=out)
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                for it in range(iters):
                    isb.gemm_dense(x, wd[it % len(wd)][i], out=out)
        torch.cuda.current_stream().wait_stream(s)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) * 1000.0 / iters)
    return res


_A8192 = {}


def alpha8192_layers(isb, layers, dev):
    """The bench layers re-integerized at alpha = 8192 (the paper's LLaMA-3 recipe):
    same codes and float scales, k_g = round(s * 8192)."""
    if "l" not in _A8192:
        out = []
        for lin in layers[:1]:
            row = []
            for name, k, n, w, _ in lin:
                codes = w.unpack_codes()
                scales = w.group_scales
                si = isb.integerize_scales(scales.cpu().numpy(), 8192)
                row.append((name, k, n, isb.PackedWeight.from_codes(codes, GROUP, scales,
                                                                   si.int_scales, 8192),
                            int(si.int_scales.max())))
            out.append(row)
        # prefill is tensor-bound: one replica, referenced REPLICAS times
        _A8192["l"] = out * REPLICAS
    return _A8192["l"]


def grouped_plans(isb, layers, xs, path, out_dtype=None):
    import torch
    out_dtype = out_dtype or torch.bfloat16
    return [isb.GroupedGemm([{"weight": l[3], "x": x} for l, x in zip(layers[r], xs)],
                            path=path, out_dtype=out_dtype) for r in range(REPLICAS)]


def graph_of(fns):
    """One CUDA graph per replica callable (captured on a side stream)."""
    import torch
    for f in fns:
        f()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graphs = []
    with torch.cuda.stream(s):
        for f in fns:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                f()
            graphs.append(g)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    return graphs


def replica_stepper(runs, steps, warmup):
    """Step i runs replica i % R. Steps are replayed from CUDA graphs holding 4R
    consecutive steps (programmatic dependent launch between them) — as a serving
    loop replays one graph per decode iteration holding every layer — so the timed
    region is K launches back to back; steps that do not fill a group replay
    one-step graphs. Returns fn(i) enqueuing step i."""
    R = len(runs)
    singles = graph_of(runs)
    G = 4  # rounds of the R replicas per group graph
    group = graph_of([lambda: [f() for _ in range(G) for f in runs]])[0]
    first_timed = warmup
    total = warmup + steps

    def fn(i):
        # full R-step groups inside the timed region start at multiples of R after warmup
        j = i - first_timed
        if i >= first_timed and j % (G * R) == 0 and i + G * R <= total:
            group.replay()
        elif i >= first_timed and j % (G * R) != 0 and (i - j % (G * R)) + G * R <= total:
            pass  # covered by the group replay issued at the group's first step
        else:
            singles[(i - first_timed) % R].replay()
    return fn


def grouped_layer_us(isb, layers, xs, path, iters=100):
    """Device time of one grouped layer launch (graph of `iters` launches rotating the
    weight replicas, CUDA events on the replay stream)."""
    import torch
    plans = grouped_plans(isb, layers, xs, path)
    g = graph_of([lambda: [plans[i % REPLICAS].run() for i in range(iters)]])[0]
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters, plans[0]


def grouped_prefill_us(isb, layers, xq_sa, iters=8):
    """Device time of the layer's four integer-scale GEMMs at prefill M as ONE grouped
    launch (isb_group_plan with pre-quantized codes: the CTA-pair fold kernel, tiles of
    all four linears dealt longest-first over the SM pairs), graph of `iters` launches
    rotating the weight replicas."""
    import torch
    plans = [isb.GroupedGemm([{"weight": l[3], "xq": q, "sa": sa}
                              for l, (q, sa) in zip(layers[r], xq_sa)])
             for r in range(REPLICAS)]
    g = graph_of([lambda: [plans[i % REPLICAS].run() for i in range(iters)]])[0]
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / iters, plans[0]


def run_ours(args, ws, rank, local):
    import numpy as np
    import torch

    import paper_2405_14597_b200 as isb
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    m = args.m
    layers, xs = build_layers(isb, m, dev, seed=1234 + rank)
    max_k = max(l[4] for lin in layers for l in lin)
    ops_per_step = sum(2 * m * k * n for _, k, n in LAYER)
    # algorithmic bytes of the grouped step: float32 activations read in-kernel (x_b=4)
    layer_bytes = sum(alg_bytes(m, k, n, x_b=4) for _, k, n in LAYER)

    # ---- headline: one grouped layer launch per step (K1 folded in), CUDA graph per replica
    plans = grouped_plans(isb, layers, xs, "integer-scale")
    step_fn = replica_stepper([p.run for p in plans], args.steps, args.warmup)
    with ClockSampler(local) as clk:
        ms = time_steps(step_fn, args.steps, args.warmup, ws)
    ms = max_over_ranks(ms, ws)
    ms_per_step = ms / args.steps
    us_step = ms_per_step * 1e3
    value = ws * ops_per_step / (ms_per_step * 1e-3) / 1e12  # TOPS, whole job

    # ---- float-scale denominator, identical structure (grouped K4)
    fplans = grouped_plans(isb, layers, xs, "float-scale")
    fms = max_over_ranks(time_steps(replica_stepper([p.run for p in fplans], args.steps,
                                                    args.warmup), args.steps, args.warmup, ws),
                         ws) / args.steps
    # ---- per-linear form: K1 + K3 per linear (8 launches), the round-1 step
    step = LayerStep(isb, layers, xs, m, "int", dev)
    step.capture()
    ums = max_over_ranks(time_steps(step.replay, args.steps, args.warmup, ws), ws) / args.steps

    # ---- e2e: host pinned X in, host bf16 out, every step, through the public runtime
    # API (paper_2405_14597_b200.runtime.GraphedLinears, grouped mode: H2D copies, one
    # grouped layer launch, D2H copies recorded into one CUDA graph, replayed per step).
    from paper_2405_14597_b200.runtime import GraphedLinears
    runners = []
    for r in range(REPLICAS):
        g = GraphedLinears([l[3] for l in layers[r]], m, device=dev, mode="grouped")
        for j, x in enumerate(xs):
            g.host_inputs[j].copy_(x.cpu())
        runners.append(g.capture())
    e2e_ms = max_over_ranks(time_steps(lambda i: runners[i % REPLICAS].run(), args.steps,
                                       args.warmup, ws), ws) / args.steps
    h2d, d2h = runners[0].h2d_bytes, runners[0].d2h_bytes
    # alternative runtime mode: one single-problem grouped launch per linear, the PCIe
    # transfers overlapping the GEMMs
    prunners = []
    for r in range(REPLICAS):
        g = GraphedLinears([l[3] for l in layers[r]], m, device=dev, mode="pipelined")
        for j, x in enumerate(xs):
            g.host_inputs[j].copy_(x.cpu())
        prunners.append(g.capture())
    e2e_pipe_ms = max_over_ranks(time_steps(lambda i: prunners[i % REPLICAS].run(), args.steps,
                                            args.warmup, ws), ws) / args.steps
    # the same through per-call eager API calls (host launch overhead included)
    xh = [x.cpu().pin_memory() for x in xs]
    oh = [torch.empty((m, n), dtype=torch.bfloat16).pin_memory() for _, _, n in LAYER]
    xd = [torch.empty_like(x) for x in xs]
    eplans = [isb.GroupedGemm([{"weight": l[3], "x": x} for l, x in zip(layers[r], xd)])
              for r in range(REPLICAS)]

    def e2e_eager(i):
        p = eplans[i % REPLICAS]
        for j in range(len(LAYER)):
            xd[j].copy_(xh[j], non_blocking=True)
        p.run()
        for j in range(len(LAYER)):
            oh[j].copy_(p.outs[j], non_blocking=True)

    e2e_eager_ms = max_over_ranks(time_steps(e2e_eager, min(args.steps, 200), args.warmup, ws),
                                  ws) / min(args.steps, 200)

    # ---- per-linear kernel table (single-GEMM kernels, events on the launching stream)
    xq_sa = [isb.quantize_per_token(x) for x in xs]
    kt = gemm_kernel_timing(isb, layers, xq_sa, m, "int")
    kf = gemm_kernel_timing(isb, layers, xq_sa, m, "float")
    peak, peak_kind = load_peaks()
    # Dominant kernel: the grouped layer launch (the whole step is this one kernel).
    achieved = layer_bytes / us_step / 1e3  # GB/s
    traffic = None
    # the latest committed ncu capture of this kernel (dram read + write per launch)
    tpath = next((os.path.join(ROOT, "profiles", f"{t}_traffic.json")
                  for t in ("r02d", "r02b", "r02")
                  if os.path.exists(os.path.join(ROOT, "profiles", f"{t}_traffic.json"))), "")
    if os.path.exists(tpath) and m == 16:
        try:
            with open(tpath) as f:
                traffic = json.load(f).get("grouped_layer_m16_bytes_per_launch")
        except Exception:
            traffic = None

    # ---- dense fp16 baseline (hand-written tcgen05 kind::f16, no cuBLAS), same shapes
    wd = [[(torch.randn((n, k), device=dev) * 0.02).half() for _, k, n in LAYER]
          for _ in range(REPLICAS)]
    dense_m = dense_layer_timing(isb, m, dev, wd, iters=30)

    # ---- decode / prefill sweep of the whole layer: int vs float vs fp16 dense
    sweep, tensor_roof = [], None
    if not args.no_sweep:
        for mm in args.sweep:
            ops = sum(2 * mm * k * n for _, k, n in LAYER)
            us_d = sum(dense_layer_timing(isb, mm, dev, wd, iters=10 if mm <= 256 else 4))
            row = {"M": mm}
            if mm <= 64:
                xm = [torch.randn((mm, k), device=dev) for _, k, _ in LAYER]
                us_i, pl = grouped_layer_us(isb, layers, xm, "integer-scale")
                us_f, _ = grouped_layer_us(isb, layers, xm, "float-scale")
                byts = sum(alg_bytes(mm, k, n, x_b=4) for _, k, n in LAYER)
                row["kernel"] = f"grouped layer launch (K1 fused), MT={pl.tile_tokens}"
            else:
                xq = [isb.quantize_per_token(torch.randn((mm, k), device=dev)) for _, k, _ in LAYER]
                ti = gemm_kernel_timing(isb, layers, xq, mm, "int", iters=10)
                tf = gemm_kernel_timing(isb, layers, xq, mm, "float", iters=10)
                us_pl = sum(r["us"] for r in ti)
                us_f = sum(r["us"] for r in tf)
                byts = sum(r["alg_bytes"] for r in ti)
                row["per_linear_int"] = ti
                row["us_per_layer_int_per_linear_launches"] = round(us_pl, 2)
                if mm >= 512:
                    us_i, gpl = grouped_prefill_us(isb, layers, xq)
                    row["kernel"] = ("int: grouped prefill launch of the 4 linears (k_g-folded "
                                     "CTA-pair kernel gemm_w4a8_sp, 512-token x 128-channel pair "
                                     "tiles, LPT); float: per-linear per-group-epilogue kernel")
                else:
                    us_i = us_pl
                    row["kernel"] = "per-linear prefill kernels (int: k_g-folded SS-256, float: per-group)"
            row.update({"us_per_layer_int": round(us_i, 2), "us_per_layer_float": round(us_f, 2),
                        "speedup_vs_float": round(us_f / us_i, 3),
                        "us_per_layer_fp16_dense": round(us_d, 2),
                        "speedup_vs_fp16_dense": round(us_d / us_i, 3),
                        "tops_int": round(ops / us_i / 1e6, 1),
                        "hbm_frac_int": round(byts / us_i / 1e3 / peak, 3),
                        # int8 tensor roofline: nominal 4.5 POPS; measured 4.79 POPS
                        # (tcgen05 kind::i8 128x256, profiles/r01_mma_peak.txt)
                        "tensor_frac_int_nominal": round(ops / us_i / 1e6 / 4500.0, 3),
                        "tensor_frac_int_measured": round(ops / us_i / 1e6 / 4786.0, 3)})
            if mm >= 256:
                # the general integer path (alpha = 8192: k_g up to ~124, no fold) on the
                # per-group skeleton K4 runs on — integer vs float scale with identical tiling
                lay8 = alpha8192_layers(isb, layers, dev)
                t8 = gemm_kernel_timing(isb, lay8, xq, mm, "int", iters=10)
                us_8 = sum(r["us"] for r in t8)
                row.update({"us_per_layer_int_alpha8192": round(us_8, 2),
                            "alpha8192_max_int_scale": max(l[4] for l in lay8[0]),
                            "speedup_int_alpha8192_vs_float_same_tiling": round(us_f / us_8, 3),
                            "tops_int_alpha8192": round(ops / us_8 / 1e6, 1)})
            sweep.append(row)
            if mm == 2048:
                tensor_roof = {"bound": "tensor", "achieved": round(ops / us_i / 1e6, 1),
                               "peak": 4786.0, "peak_kind": "measured tcgen05 kind::i8 (r01_mma_peak)",
                               "unit": "TOPS", "frac": round(ops / us_i / 1e6 / 4786.0, 4),
                               "frac_nominal_4500": round(ops / us_i / 1e6 / 4500.0, 4),
                               "kernel": "gemm_w4a8_sp (CTA pair, k_g folded), grouped launch of "
                                         "the LLaMA-2-7B layer's 4 linears, M=2048",
                               "per_linear_launches_us": round(us_pl, 2)}

    moe_res = None
    if not args.no_moe:
        moe_res = moe_bench(isb, dev, args)

    # ---- C3: LLaMA-3-8B decoder-layer linears, per-token act quant fused (grouped launch
    # with K1 inside) at decode, and the grouped prefill launch at M = 2048
    c3 = None
    if not args.no_sweep:
        l3, x3 = build_layers(isb, m, dev, seed=99, shapes=LAYER_L3_8B)
        us3, _ = grouped_layer_us(isb, l3, x3, "integer-scale")
        us3f, _ = grouped_layer_us(isb, l3, x3, "float-scale")
        b3 = sum(alg_bytes(m, k, n, x_b=4) for _, k, n in LAYER_L3_8B)
        xq3 = [isb.quantize_per_token(torch.randn((2048, k), device=dev)) for _, k, _ in LAYER_L3_8B]
        us3p, _ = grouped_prefill_us(isb, l3, xq3)
        ops3 = sum(2 * 2048 * k * n for _, k, n in LAYER_L3_8B)
        c3 = {"workload": "llama3-8b decoder-layer linears (BASELINE configs[2]), 1 GPU",
              "linears": [{"name": a, "K": k, "N": n} for a, k, n in LAYER_L3_8B],
              "decode_M": m, "decode_us_per_layer": round(us3, 2),
              "decode_float_scale_us_per_layer": round(us3f, 2),
              "decode_hbm_frac": round(b3 / us3 / 1e3 / peak, 3),
              "prefill_M": 2048, "prefill_us_per_layer": round(us3p, 2),
              "prefill_tops": round(ops3 / us3p / 1e6, 1),
              "prefill_tensor_frac_measured": round(ops3 / us3p / 1e6 / 4786.0, 3),
              "note": "decode: one grouped launch with the per-token quantizer fused (float32 "
                      "activations in); prefill: pre-quantized, one grouped CTA-pair launch"}
        del l3

    result = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "TOPS",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 5),
        "us_per_layer": round(us_step, 2),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int8 (s8 x s4->s8 MMA, s32 accumulate)",
        "data": "synthetic (llama_like-structured int4 weights, gaussian activations; device-generated)",
        "config": {
            "workload": f"llama2-7b decoder-layer linears, decode M={m}",
            "M": m, "linears": [{"name": a, "K": k, "N": n} for a, k, n in LAYER],
            "group": GROUP, "alpha": ALPHA, "max_int_scale": max_k,
            "step": "one grouped layer launch: per-token quantize of the 4 float32 inputs + "
                    "integer-scale GEMM of the 4 linears (gemm_w4a8_group, CUDA graph)",
            "l2": f"weights rotated over {REPLICAS} layer replicas ({REPLICAS}x107.5MB > 2x126MB L2)",
            "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
        },
        "speedup_vs_float_scale": round(fms * 1e3 / us_step, 3),
        "float_scale_us_per_layer": round(fms * 1e3, 2),
        "per_linear_us_per_layer": round(ums * 1e3, 2),
        "per_linear_step": "K1 + K3 per linear (8 launches, CUDA graph)",
        "grouped_plan": {"grid": plans[0].grid, "tile_tokens": plans[0].tile_tokens,
                         "budget_steps_per_cta": plans[0].makespan_steps},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic,
                     "kernel": f"gemm_w4a8_group<{plans[0].tile_tokens}, integer-scale> "
                               f"LLaMA-2-7B layer M={m} (4 linears, K1 fused)",
                     "alg_bytes_per_launch": layer_bytes, "us_per_launch": round(us_step, 3),
                     "per_linear_single_gemm": kt},
        "roofline_tensor_prefill": tensor_roof,
        "c3_llama3_8b": c3,
        "float_scale_kernel": kf,
        "fp16_dense": {"kernel": "gemm_f16_tc (tcgen05 kind::f16, fp32 acc, no cuBLAS)",
                       "us_per_linear": [round(v, 2) for v in dense_m],
                       "us_per_layer": round(sum(dense_m), 2),
                       "speedup_w4a8_step_vs_fp16": round(sum(dense_m) / us_step, 3)},
        "e2e": {"value": round(ws * ops_per_step / (e2e_ms * 1e-3) / 1e12, 3), "unit": "TOPS",
                "us_per_layer": round(e2e_ms * 1e3, 2),
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "runtime.GraphedLinears (mode=grouped): H2D of the 4 float32 inputs -> "
                       "one grouped launch (K1 fused) -> D2H of the 4 bf16 outputs, one CUDA graph",
                "pipelined_mode_us_per_layer": round(e2e_pipe_ms * 1e3, 2),
                "eager_api_us_per_layer": round(e2e_eager_ms * 1e3, 2)},
        "gpu_launches": args.steps * 1,
        "clocks": clk.summary(),
        "sweep": sweep,
        "mixtral_moe": moe_res,
    }
    return result


def moe_bench(isb, dev, args, n_experts=8, tokens=16, k=4096, f=14336):
    """Config C5 on one GPU: Mixtral-8x7B expert FFN, T=16 decode tokens top-2 routed
    (32 expert rows, 4 per expert). Per step: ONE grouped launch for the 8 experts'
    w1|w3 GEMMs (4096 -> 2 x 14336, K1 fused), SiLU(gate) * up (torch elementwise),
    ONE grouped launch for the 8 experts' w2 GEMMs (14336 -> 4096, K1 fused); CUDA graph."""
    import torch
    gen = torch.Generator(device=dev)
    gen.manual_seed(77)
    rows = 2 * tokens // n_experts
    experts, byts = [], 0
    for _ in range(n_experts):
        packs = []
        for kk, nn in ((k, 2 * f), (f, k)):
            wf = llama_like_weight(kk, nn, gen, dev)
            codes, scales = isb.quantize_weight(wf, GROUP, 4)
            del wf
            si = isb.integerize_scales(scales.cpu().numpy(), ALPHA)
            packs.append(isb.PackedWeight.from_codes(codes, GROUP, scales, si.int_scales, ALPHA))
            byts += alg_bytes(rows, kk, nn, x_b=4)
        experts.append(packs)
    x = torch.randn((n_experts, rows, k), generator=gen, device=dev)
    gu = torch.empty((n_experts, rows, 2 * f), dtype=torch.float32, device=dev)
    h = torch.empty((n_experts, rows, f), dtype=torch.float32, device=dev)
    y = torch.empty((n_experts, rows, k), dtype=torch.bfloat16, device=dev)
    g13 = isb.GroupedGemm([{"weight": experts[e][0], "x": x[e], "out": gu[e]}
                           for e in range(n_experts)], out_dtype=torch.float32)
    g2 = isb.GroupedGemm([{"weight": experts[e][1], "x": h[e], "out": y[e]}
                          for e in range(n_experts)], out_dtype=torch.bfloat16)

    def step():
        g13.run()
        torch.mul(torch.nn.functional.silu(gu[..., :f]), gu[..., f:], out=h)
        g2.run()

    g = graph_of([step])[0]
    n = max(20, min(args.steps, 200))
    ms = time_steps(lambda i: g.replay(), n, args.warmup, 1) / n
    ops_ = n_experts * 2 * rows * (k * 2 * f + f * k)
    peak, _ = load_peaks()
    return {"config": f"Mixtral-8x7B expert FFN, {n_experts} experts on 1 GPU, {tokens} tokens "
                      f"top-2 ({rows} rows/expert): grouped w1|w3 launch (K1 fused) + SiLU*up "
                      f"(torch) + grouped w2 launch (K1 fused), CUDA graph",
            "us_per_moe_layer": round(ms * 1e3, 2), "tops": round(ops_ / (ms * 1e-3) / 1e12, 2),
            "alg_bytes": byts, "hbm_frac": round(byts / (ms * 1e-3) / 1e9 / peak, 3)}


# ----------------------------------------------------------------------------- CPU legs
def cpu_layer_sample(m, threads, repeats=1, seed=42):
    """The oracle (CPU restatement of gemm_integer_scale, gemm.cpp:205-262) on one
    LLaMA-2-7B layer at M rows, reference-style row-partitioned std::threads.
    Returns (TOPS, seconds per layer)."""
    from oracle import oracle as O
    probs = []
    for i, (_, k, n) in enumerate(LAYER):
        w = O.quantize_weight(O.generate_llama_like(k, n, seed + i), GROUP)
        x = O.quantize_per_token(O.generate_gaussian(m, k, 1.0, seed + 100 + i))
        s = O.integerize_scales(w.scales, ALPHA)
        probs.append((x, w, s))
    times = []
    for _ in range(repeats):
        t = 0.0
        for x, w, s in probs:
            r = O.gemm_integer_scale(x, w, s, workers=threads, record=False)
            t += r.stats["wall_ms"] / 1e3
        times.append(t)
    if not times:
        return None, None, probs
    sec = statistics.median(times)
    ops = sum(2 * m * k * n for _, k, n in LAYER)
    return ops / sec / 1e12, sec, probs


def _slice_cols(O, w, s, c0, c1):
    """Columns [c0, c1) of a quantized weight and its scales (unit n*G + g)."""
    g = w.values.shape[0] // w.group
    ws = O.QuantizedTensor(np.ascontiguousarray(w.values[:, c0:c1]), w.bit_width, w.scheme,
                           w.kind, w.group, w.scales[c0 * g:c1 * g], w.zero_points)
    ss = O.IntegerScaleSet(s.int_scales[c0 * g:c1 * g], s.amplifier, s.exponent)
    return ws, ss


def run_reference(args, ws, rank):
    """--impl reference: the reference path's CPU implementation (the oracle port of
    gemm_integer_scale — the reference itself cannot be built here) on this box's
    host cores, on the same workload. Each step is a bounded column slice of the
    layer's linears (round robin) so the whole run stays within a few minutes."""
    if rank != 0:
        return None
    import numpy as np  # noqa: F401
    from oracle import oracle as O
    threads = min(os.cpu_count() or 1, args.m)  # the reference parallelises over rows only
    _, _, probs = cpu_layer_sample(args.m, threads, repeats=0)
    # calibrate seconds per MAC on a 512-column slice
    x, w, s = probs[0]
    wsl, ssl = _slice_cols(O, w, s, 0, 512)
    t = O.gemm_integer_scale(x, wsl, ssl, workers=threads, record=False).stats["wall_ms"] / 1e3
    sec_per_mac = t / (args.m * 512 * w.values.shape[0])
    budget = 150.0 / (args.steps + args.warmup)
    ops = 0
    sec = 0.0
    cursor = [0] * len(probs)
    for i in range(args.warmup + args.steps):
        li = i % len(probs)
        x, w, s = probs[li]
        k, n = w.values.shape
        cols = int(max(128, min(n, budget / (sec_per_mac * args.m * k))))
        c0 = cursor[li] % n
        c1 = min(n, c0 + cols)
        cursor[li] = c1
        wsl, ssl = _slice_cols(O, w, s, c0, c1)
        r = O.gemm_integer_scale(x, wsl, ssl, workers=threads, record=False)
        if i >= args.warmup:
            sec += r.stats["wall_ms"] / 1e3
            ops += 2 * args.m * k * (c1 - c0)
    v = ops / sec / 1e12
    sample = (f"per step a column slice (~{budget:.2f} s of CPU work) of one LLaMA-2-7B layer "
              f"linear at M={args.m}, round robin over the 4 linears; oracle port of "
              f"gemm_integer_scale with {threads} row-partitioned threads")
    return {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TOPS", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int64 (CPU int16 codes, int64 accumulate)",
        "data": "synthetic (reference generators: llama_like W seed 42+i, gaussian X)",
        "config": {"workload": f"llama2-7b decoder-layer linears, decode M={args.m}", "M": args.m,
                   "linears": [{"name": a, "K": k, "N": n} for a, k, n in LAYER],
                   "group": GROUP, "alpha": ALPHA},
        "cpu_baseline": {"value": v, "unit": "TOPS", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "TOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def cpu_baseline(args):
    """The oracle port of gemm_integer_scale on this box's host cores, one LLaMA-2-7B
    layer's 4 linears at M rows, median of 3 like run_bench (analysis.cpp:195-215),
    at workers = nproc (the reported value) and workers = 1."""
    nproc = os.cpu_count() or 1
    threads = min(nproc, args.m)  # the reference parallelises over rows only (gemm.cpp:63-68)
    tops, sec, _ = cpu_layer_sample(args.m, threads, repeats=3)
    tops1, sec1, _ = cpu_layer_sample(args.m, 1, repeats=3)
    try:
        model = next(l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo")
                     if l.startswith("model name"))
    except Exception:
        model = "unknown"
    return {"value": tops, "unit": "TOPS", "cores": threads, "kind": "port",
            "sample": (f"one LLaMA-2-7B layer's 4 linears at M={args.m}, median of 3 "
                       f"({sec * 1e3:.0f} ms/layer); oracle port of gemm_integer_scale, "
                       f"{threads} row-partitioned threads of {nproc} on {model}; "
                       f"-O3 -DNDEBUG -ffp-contract=off"),
            "workers_1": {"value": tops1, "ms_per_layer": round(sec1 * 1e3, 1), "cores": 1},
            "workers_nproc": {"value": tops, "ms_per_layer": round(sec * 1e3, 1),
                              "cores": threads, "nproc": nproc, "cpu": model}}



# ----------------------------------------------------------------------------- tensor parallel
# BASELINE configs[3] (C4): LLaMA-2-70B decoder-layer linears across N GPUs, Megatron
# layout — qkv / gate_up column-parallel (N-split; their outputs stay sharded for the
# head-parallel attention / the sharded SwiGLU), o / down row-parallel (K-split on group
# boundaries: per-token scale from an all-reduce MAX of partial row maxima, raw int32
# accumulator, exact all-reduce SUM in int32, one Eq. 2 epilogue; parallel.py).
LAYER_70B = [("qkv_proj", 8192, 10240, "col"), ("o_proj", 8192, 8192, "row"),
             ("gate_up_proj", 8192, 57344, "col"), ("down_proj", 28672, 8192, "row")]


def run_tp(args, ws, rank, local):
    import torch
    import paper_2405_14597_b200 as isb
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    m = args.m
    gen = torch.Generator(device=dev)
    gen.manual_seed(4321 + rank)
    lin = []
    for name, k, n, kind in LAYER_70B:
        ks, ns = (k, n // ws) if kind == "col" else (k // ws, n)
        assert ks % GROUP == 0 and ns % 128 == 0, (name, ks, ns)
        wf = llama_like_weight(ks, ns, gen, dev)
        codes, scales = isb.quantize_weight(wf, GROUP, 4)
        del wf
        si = isb.integerize_scales(scales.cpu().numpy(), ALPHA)
        w = isb.PackedWeight.from_codes(codes, GROUP, scales, si.int_scales, ALPHA)
        x = torch.randn((m, ks), generator=gen, device=dev)   # replicated (col) / K-slice (row)
        lin.append((name, k, n, kind, ks, ns, w, x))
    wsp = isb.Workspace()
    rows = [l for l in lin if l[3] == "row"]
    # both row-parallel linears' partial maxima / int32 accumulators live in ONE buffer each,
    # so a step needs one all-reduce MAX and one all-reduce SUM
    amax_all = torch.empty((len(rows), m), dtype=torch.float32, device=dev)
    acc_all = torch.empty((sum(m * l[5] for l in rows),), dtype=torch.int32, device=dev)
    bufs, off = {}, 0
    for name, k, n, kind, ks, ns, w, x in lin:
        b = {"xq": torch.empty((m, ks), dtype=torch.int8, device=dev),
             "sa": torch.empty((m,), dtype=torch.float64, device=dev),
             "out": torch.empty((m, ns), dtype=torch.bfloat16, device=dev)}
        if kind == "row":
            b["acc"] = acc_all[off:off + m * ns].view(m, ns)
            off += m * ns
        bufs[name] = b
    for i, l in enumerate(rows):
        bufs[l[0]]["amax"] = amax_all[i]

    cols = [l for l in lin if l[3] == "col"]
    # the column linears (K1 fused) and the row linears (pre-quantized, raw int32
    # accumulators) each run as ONE grouped launch (isb_group_plan)
    col_plan = isb.GroupedGemm([{"weight": l[6], "x": l[7], "xq": bufs[l[0]]["xq"],
                                 "sa": bufs[l[0]]["sa"], "out": bufs[l[0]]["out"]} for l in cols])
    row_plan = isb.GroupedGemm([{"weight": l[6], "xq": bufs[l[0]]["xq"], "sa": bufs[l[0]]["sa"],
                                 "out": bufs[l[0]]["acc"]} for l in rows], out_dtype=torch.int32)

    def seg_local():      # column linears (K1 + K3), partial row maxima of the row linears
        col_plan.run()
        for name, k, n, kind, ks, ns, w, x in rows:
            b = bufs[name]
            isb.row_absmax(x, out=b["amax"])

    def seg_row_gemm():   # quantize with the global maxima, raw int32 accumulators
        for name, k, n, kind, ks, ns, w, x in rows:
            b = bufs[name]
            isb.quantize_per_token_amax(x, b["amax"], codes=b["xq"], scales=b["sa"])
        row_plan.run()

    def seg_finalize():   # one Eq. 2 epilogue per reduced accumulator
        for name, k, n, kind, ks, ns, w, x in rows:
            b = bufs[name]
            isb.finalize_acc(b["acc"], b["sa"], ALPHA, out=b["out"])

    graphs = graph_of([seg_local, seg_row_gemm, seg_finalize])

    def step(collectives):
        graphs[0].replay()
        if collectives and ws > 1:
            import torch.distributed as dist
            dist.all_reduce(amax_all, op=dist.ReduceOp.MAX)
        graphs[1].replay()
        if collectives and ws > 1:
            import torch.distributed as dist
            dist.all_reduce(acc_all, op=dist.ReduceOp.SUM)
        graphs[2].replay()

    ops = sum(2 * m * k * n for _, k, n, _ in LAYER_70B)   # the whole layer, all ranks
    res = {}
    for mode in ("with_collectives", "compute_only"):
        fn = (lambda i, c=(mode == "with_collectives"): step(c))
        ms = max_over_ranks(time_steps(fn, args.steps, args.warmup, ws), ws) / args.steps
        res[mode] = ms
    us = res["with_collectives"] * 1e3
    return {
        "metric": METRIC, "value": round(ops / us / 1e6, 3), "unit": "TOPS", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["with_collectives"], 5),
        "us_per_layer": round(us, 2), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int8 (s8 x s4->s8 MMA, s32 accumulate)",
        "data": "synthetic (llama_like-structured int4 weights per shard, gaussian activations)",
        "config": {"workload": f"llama2-70b decoder-layer linears, tensor-parallel tp{ws}, M={m}",
                   "M": m, "parallelism": f"tp{ws} (Megatron: qkv/gate_up column-parallel, "
                                          "o/down row-parallel, exact int32 all-reduce)",
                   "linears": [{"name": a, "K": k, "N": n, "split": kind,
                                "shard_K": (k if kind == "col" else k // ws),
                                "shard_N": (n // ws if kind == "col" else n)}
                               for a, k, n, kind in LAYER_70B],
                   "group": GROUP, "alpha": ALPHA},
        "compute_only_us_per_layer": round(res["compute_only"] * 1e3, 2),
        "collective_us_per_layer": round((res["with_collectives"] - res["compute_only"]) * 1e3, 2),
        "launches": "per step: 3 CUDA graphs (one grouped launch of the column linears with K1 "
                    "fused + the row linears' partial maxima | amax-quantize + one grouped "
                    "int32 launch of the row linears | Eq. 2 finalize) with, when N > 1, one "
                    "NCCL all-reduce MAX (both row linears' maxima) and one all-reduce SUM "
                    "(both int32 accumulators) between",
        "gpu_launches": args.steps * 10,
    }

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--m", type=int, default=16)
    ap.add_argument("--sweep", type=int, nargs="*", default=[1, 2, 4, 8, 16, 32, 64, 2048])
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-moe", action="store_true")
    ap.add_argument("--mode", default="layer", choices=["layer", "tp"],
                    help="layer: the headline (one grouped LLaMA-2-7B layer launch per step, "
                         "replicated per GPU); tp: LLaMA-2-70B layer linears tensor-parallel")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched directly with --gpus N: re-exec as N ranks (one process per GPU)
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))

    if args.impl == "reference":
        ws = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        res = run_reference(args, ws, rank)
        if res is not None:
            print(json.dumps(res))
        return

    ws, rank, local = init_dist()
    if args.mode == "tp":
        res = run_tp(args, ws, rank, local)
        if rank == 0:
            print(json.dumps(res))
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    res = run_ours(args, ws, rank, local)
    if rank == 0:
        if ws == 1 and not args.no_cpu:
            res["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(res))
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
