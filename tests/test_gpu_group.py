"""Grouped layer launch (isb_group_plan_*, csrc/gemm_group.cu) parity.

Per problem the grouped launch must equal quantize(x, 8, symmetric, per_token)
(quantize.cpp:93-145) followed by gemm_integer_scale (gemm.cpp:205-262) bit for
bit — checked against the oracle on small shapes and, at the LLaMA / Mixtral
sizes, against K1 + the single-GEMM kernel (itself oracle-checked in
test_gpu_parity.py / test_gpu_scale.py). Float scale (gemm.cpp:156-203): within
the fp32-accumulation bound. Replays (CUDA graph, >= 50) must be identical: the
in-kernel readiness counters re-arm themselves at the end of every launch.
"""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU, skipped there
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2405_14597_b200 as isb  # noqa: E402

DEV = torch.device("cuda:0")
LLAMA2_7B = [(4096, 12288), (4096, 4096), (4096, 22016), (11008, 4096)]


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(DEV)


def device_weight(k, n, seed, amp=1024):
    """llama_like weight quantized on the device (bit-exact group quantizer)."""
    from bench import llama_like_weight
    gen = torch.Generator(device=DEV)
    gen.manual_seed(seed)
    wf = llama_like_weight(k, n, gen, DEV)
    codes, scales = isb.quantize_weight(wf, 128, 4)
    si = isb.integerize_scales(scales.cpu().numpy(), amp)
    return isb.PackedWeight.from_codes(codes, 128, scales, si.int_scales, amp)


_W = {}


def layer_weights(shapes, tag=0):
    key = (tuple(shapes), tag)
    if key not in _W:
        _W[key] = [device_weight(k, n, seed=11 * k + n + tag) for k, n in shapes]
    return _W[key]


def single_reference(x, w, path, out_dtype):
    q, sa = isb.quantize_per_token(x)
    f = isb.gemm_integer_scale if path == "integer-scale" else isb.gemm_float_scale
    return q, sa, f(q, sa, w, out_dtype=out_dtype)


@pytest.mark.parametrize("m", [1, 3, 16, 17, 32, 40, 64])
def test_group_layer_matches_k1_plus_k3(m):
    ws = layer_weights(LLAMA2_7B)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(100 + m)
    xs = [torch.randn((m, k), generator=gen, device=DEV) * (1 + i) for i, (k, _) in
          enumerate(LLAMA2_7B)]
    codes = [torch.empty((m, k), dtype=torch.int8, device=DEV) for k, _ in LLAMA2_7B]
    scales = [torch.empty((m,), dtype=torch.float64, device=DEV) for _ in LLAMA2_7B]
    g = isb.GroupedGemm([{"weight": w, "x": x, "xq": c, "sa": s}
                         for w, x, c, s in zip(ws, xs, codes, scales)])
    outs = g.run()
    torch.cuda.synchronize()
    for i, (x, w) in enumerate(zip(xs, ws)):
        q, sa, ref = single_reference(x, w, "integer-scale", torch.bfloat16)
        assert torch.equal(codes[i], q), f"codes differ (problem {i})"
        assert torch.equal(scales[i], sa), f"scales differ (problem {i})"
        assert torch.equal(outs[i], ref), f"output differs (problem {i}, m={m})"
    assert not g.nonfinite()


def test_group_small_vs_oracle_all_dtypes():
    """Oracle directly: two problems of different K/N/M, float32 activations."""
    shapes = [(3, 512, 384), (5, 1024, 256)]
    probs, refs = [], []
    for i, (m, k, n) in enumerate(shapes):
        wf = O.generate_llama_like(k, n, 40 + i)
        xf = O.generate_gaussian(m, k, 1.0, 50 + i)
        wo = O.quantize_weight(wf, 128)
        so = O.integerize_scales(wo.scales, 1024)
        xo = O.quantize_per_token(xf)
        refs.append((xo, O.gemm_integer_scale(xo, wo, so), O.gemm_float_scale(xo, wo)))
        w = isb.PackedWeight.from_codes(dev(wo.values), 128, dev(wo.scales), dev(so.int_scales),
                                        so.amplifier)
        probs.append((w, dev(xf)))
    for dt in (torch.float32, torch.bfloat16, torch.int32):
        g = isb.GroupedGemm([{"weight": w, "x": x} for w, x in probs], out_dtype=dt)
        outs = [o.clone() for o in g.run()]
        torch.cuda.synchronize()
        for (xo, ri, _), o in zip(refs, outs):
            if dt == torch.int32:
                assert np.array_equal(o.cpu().numpy().astype(np.int64), ri.acc)
            elif dt == torch.float32:
                assert np.array_equal(o.cpu().numpy().view(np.int32), ri.output.view(np.int32))
            else:
                assert torch.equal(o.cpu(), torch.from_numpy(ri.output).to(torch.bfloat16))
    g = isb.GroupedGemm([{"weight": w, "x": x} for w, x in probs], path="float-scale",
                        out_dtype=torch.float32)
    outs = g.run()
    torch.cuda.synchronize()
    for (xo, _, rf), o in zip(refs, outs):
        err = np.abs(o.cpu().numpy().astype(np.float64) - rf.output_f64).max()
        assert err <= 1e-5 * np.abs(rf.output_f64).max()


def test_group_prequantized_inputs():
    m = 16
    ws = layer_weights(LLAMA2_7B)
    xq = [isb.quantize_per_token(torch.randn((m, k), device=DEV)) for k, _ in LLAMA2_7B]
    g = isb.GroupedGemm([{"weight": w, "xq": q, "sa": s} for w, (q, s) in zip(ws, xq)])
    outs = g.run()
    for (q, s), w, o in zip(xq, ws, outs):
        assert torch.equal(o, isb.gemm_integer_scale(q, s, w))


def test_group_graph_replay_is_stable_and_tracks_inputs():
    """50 graph replays of the quantizing launch give identical results (the
    readiness counters re-arm); changing the activations in place between replays
    changes the result exactly as K1 + K3 does."""
    m = 16
    ws = layer_weights(LLAMA2_7B)
    xs = [torch.randn((m, k), device=DEV) for k, _ in LLAMA2_7B]
    g = isb.GroupedGemm([{"weight": w, "x": x} for w, x in zip(ws, xs)])
    g.run()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(graph, stream=s):
            g.run()
    torch.cuda.current_stream().wait_stream(s)
    graph.replay()
    torch.cuda.synchronize()
    first = [o.clone() for o in g.outs]
    bad = torch.zeros((), dtype=torch.int64, device=DEV)
    for _ in range(50):
        graph.replay()
        for o, f in zip(g.outs, first):
            bad += (o != f).sum()
    torch.cuda.synchronize()
    assert int(bad) == 0
    for i, (x, w) in enumerate(zip(xs, ws)):
        assert torch.equal(first[i], single_reference(x, w, "integer-scale", torch.bfloat16)[2])
    for x in xs:
        x.mul_(-0.5).add_(0.25)
    graph.replay()
    torch.cuda.synchronize()
    for i, (x, w) in enumerate(zip(xs, ws)):
        assert torch.equal(g.outs[i], single_reference(x, w, "integer-scale", torch.bfloat16)[2])


def test_group_moe_experts_ragged_rows():
    """Mixtral-8x7B w1|w3 experts (4096 -> 2 x 14336) with ragged routed rows,
    including an expert with no tokens; bf16 activations."""
    counts = [5, 0, 3, 1, 9, 2, 4, 8]
    w = layer_weights([(4096, 28672)], tag=7)[0]
    xs = [torch.randn((c, 4096), device=DEV).to(torch.bfloat16) for c in counts]
    g = isb.GroupedGemm([{"weight": w, "x": x} for x in xs], out_dtype=torch.float32)
    outs = g.run()
    torch.cuda.synchronize()
    for x, o in zip(xs, outs):
        if x.shape[0] == 0:
            assert o.shape == (0, 28672)
            continue
        assert torch.equal(o, single_reference(x, w, "integer-scale", torch.float32)[2])


def test_group_float_scale_within_bound():
    m = 16
    ws = layer_weights(LLAMA2_7B)
    xs = [torch.randn((m, k), device=DEV) for k, _ in LLAMA2_7B]
    g = isb.GroupedGemm([{"weight": w, "x": x} for w, x in zip(ws, xs)], path="float-scale",
                        out_dtype=torch.float32)
    outs = g.run()
    for x, w, o in zip(xs, ws, outs):
        ref = single_reference(x, w, "float-scale", torch.float32)[2].double()
        tol = 1e-5 * ref.abs().max()
        assert float((o.double() - ref).abs().max()) <= float(tol)


def test_group_schedules_with_split_tiles():
    """Different CTA counts pour the tiles into different budgets (tiles split into
    pieces reduced through global memory in piece order): the integer result never
    changes; 20 launches each."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = r"""
import sys, torch
sys.path.insert(0, %r)
import paper_2405_14597_b200 as isb
from tests.test_gpu_group import layer_weights, single_reference, LLAMA2_7B, DEV
for m in (1, 16, 40):
    ws = layer_weights(LLAMA2_7B)
    xs = [torch.randn((m, k), device=DEV) for k, _ in LLAMA2_7B]
    g = isb.GroupedGemm([{"weight": w, "x": x} for w, x in zip(ws, xs)])
    for _ in range(20):
        g.run()
    torch.cuda.synchronize()
    for x, w, o in zip(xs, ws, g.outs):
        assert torch.equal(o, single_reference(x, w, "integer-scale", torch.bfloat16)[2]), (m, g.grid)
print("ok", g.grid)
""" % root
    for n in ("148", "131", "37", "5"):
        r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                           env=dict(os.environ, ISB_GROUP_CTAS=n), timeout=600)
        assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-1500:] + r.stderr[-3000:]
        assert int(r.stdout.split()[-1]) <= int(n)


def test_group_single_small_problem_many_pieces():
    """One N=K=4096 GEMM at M=16 (32 tiles over ~148 CTAs): every tile is split into
    several pieces; integer output bit-exact, float within the fp32 bound."""
    w = layer_weights([(4096, 4096)])[0]
    x = torch.randn((16, 4096), device=DEV)
    g = isb.GroupedGemm([{"weight": w, "x": x}], out_dtype=torch.float32)
    for _ in range(10):
        g.run()
    assert torch.equal(g.outs[0], single_reference(x, w, "integer-scale", torch.float32)[2])
    gf = isb.GroupedGemm([{"weight": w, "x": x}], path="float-scale", out_dtype=torch.float32)
    o = gf.run()[0].double()
    ref = single_reference(x, w, "float-scale", torch.float32)[2].double()
    assert float((o - ref).abs().max()) <= 1e-5 * float(ref.abs().max())


def test_group_refuses_unsafe_layer_and_flags_nonfinite():
    from tests.instances import overflow_rig
    x, w, s = overflow_rig(16)
    pw = isb.PackedWeight.from_codes(dev(w.values), w.group, dev(w.scales), dev(s.int_scales),
                                     s.amplifier)
    with pytest.raises(isb.OverflowError_):
        isb.GroupedGemm([{"weight": pw, "x": torch.ones((1, 4096), device=DEV)}])
    ws = layer_weights(LLAMA2_7B)
    xs = [torch.randn((4, k), device=DEV) for k, _ in LLAMA2_7B]
    xs[2][1, 7] = float("nan")
    g = isb.GroupedGemm([{"weight": w, "x": x} for w, x in zip(ws, xs)])
    g.run()
    assert g.nonfinite()
    assert not g.nonfinite()  # cleared


# ------------------------------------------------------------------ grouped prefill
# Every problem M >= 512 on the integer path with k_g <= 16: the plan routes to K1 per
# problem + ONE grouped CTA-pair fold launch (gemm_sp.cu, LPT over the layer's tiles).
@pytest.mark.parametrize("m", [512, 1000, 2048])
def test_group_prefill_layer_matches_single_gemms(m):
    ws = layer_weights(LLAMA2_7B)
    gen = torch.Generator(device=DEV)
    gen.manual_seed(300 + m)
    xs = [torch.randn((m, k), generator=gen, device=DEV) for k, _ in LLAMA2_7B]
    g = isb.GroupedGemm([{"weight": w, "x": x} for w, x in zip(ws, xs)])
    assert g.tile_tokens == 512
    outs = g.run()
    torch.cuda.synchronize()
    for i, (x, w) in enumerate(zip(xs, ws)):
        _, _, ref = single_reference(x, w, "integer-scale", torch.bfloat16)
        assert torch.equal(outs[i], ref), f"output differs (problem {i}, m={m})"
    first = [o.clone() for o in outs]
    for _ in range(20):  # replays identical (races would show here)
        g.run()
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(first, outs))
    assert not g.nonfinite()


def test_group_prefill_prequantized_vs_oracle():
    """Small pre-quantized problems (oracle-generated) through the prefill route: int32
    accumulator and float32 output bit-exact against gemm_integer_scale (gemm.cpp:205-262)."""
    shapes = [(600, 256, 384), (520, 512, 256)]
    probs, refs = [], []
    for i, (m, k, n) in enumerate(shapes):
        w = O.quantize_weight(O.generate_llama_like(k, n, 70 + i), 128)
        s = O.integerize_scales(w.scales, 1024)
        x = O.quantize_per_token(O.generate_gaussian(m, k, 1.0, 80 + i))
        pw = isb.PackedWeight.from_codes(dev(w.values), 128, dev(w.scales), dev(s.int_scales), 1024)
        refs.append(O.gemm_integer_scale(x, w, s))
        probs.append({"weight": pw, "xq": dev(x.values, torch.int8), "sa": dev(x.scales)})
    for dt in (torch.int32, torch.float32):
        g = isb.GroupedGemm(probs, out_dtype=dt)
        assert g.tile_tokens == 512
        outs = g.run()
        torch.cuda.synchronize()
        for o, ref in zip(outs, refs):
            got = o.cpu().numpy()
            if dt == torch.int32:
                assert np.array_equal(got.astype(np.int64), ref.acc)
            else:
                assert np.array_equal(got.view(np.int32), ref.output.view(np.int32))


def test_group_prefill_float_and_general_integer_route_sequentially():
    """Prefill-sized problems the pair kernel does not cover (float scale; k_g > 16 at
    alpha = 8192) run K1 per problem + the single-GEMM prefill kernels in turn: equal to
    the per-problem calls."""
    from bench import llama_like_weight
    gw = torch.Generator(device=DEV)
    gw.manual_seed(5)
    ws7, w8192 = [], []
    for k, n in LLAMA2_7B[:2]:
        codes, scales = isb.quantize_weight(llama_like_weight(k, n, gw, DEV), 128, 4)
        for amp, dst in ((1024, ws7), (8192, w8192)):
            si = isb.integerize_scales(scales.cpu().numpy(), amp)
            dst.append(isb.PackedWeight.from_codes(codes, 128, scales, si.int_scales, amp))
    assert max(w.info["max_int_scale"] for w in w8192) > 16
    gen = torch.Generator(device=DEV)
    gen.manual_seed(77)
    xs = [torch.randn((600, k), generator=gen, device=DEV) for k, _ in LLAMA2_7B[:2]]
    for path, ws in (("float-scale", ws7), ("integer-scale", w8192)):
        g = isb.GroupedGemm([{"weight": w, "x": x} for w, x in zip(ws, xs)], path=path)
        assert g.tile_tokens == 0  # sequential route
        outs = g.run()
        torch.cuda.synchronize()
        for x, w, o in zip(xs, ws, outs):
            _, _, ref = single_reference(x, w, path, torch.bfloat16)
            assert torch.equal(o, ref), path
