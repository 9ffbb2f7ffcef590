"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle on
identical inputs. Integer/byte work must be bit-exact; the integer-scale float32
output is bit-exact (0 ULP); bf16/fp16 outputs equal the host-rounded oracle
float32; the float-scale (fp32 Atom-style) variant is within a stated tolerance.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.instances import llama_problem, make_w, make_x, overflow_rig, random_instance

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU, skipped there
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2405_14597_b200 as isb  # noqa: E402

DEV = torch.device("cuda:0")


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(DEV)


def pack(w: O.QuantizedTensor, s: O.IntegerScaleSet | None):
    return isb.PackedWeight.from_codes(
        dev(w.values), w.group if w.kind == O.GROUP else w.rows, dev(w.scales),
        None if s is None else dev(s.int_scales), 1 if s is None else s.amplifier)


def to_bf16_np(f32: np.ndarray) -> np.ndarray:
    return torch.from_numpy(f32).to(torch.bfloat16).float().numpy()


# ------------------------------------------------------------------------- K1
@pytest.mark.parametrize("m,k", [(1, 4096), (16, 4096), (3, 256), (64, 11008), (5, 14336),
                                 (2, 28672), (7, 100), (4, 4)])
def test_quantize_per_token_bit_exact(m, k):
    xf = O.generate_gaussian(m, k, 1.0, 43 + m + k)
    xf[0, :] = 0.0 if m > 2 else xf[0, :]          # an all-zero row => s = 1
    ref = O.quantize_per_token(xf)
    codes, scales = isb.quantize_per_token(dev(xf), check_finite=True)
    torch.cuda.synchronize()
    assert np.array_equal(codes.cpu().numpy().astype(np.int16), ref.values)
    assert np.array_equal(scales.cpu().numpy(), ref.scales)          # doubles, bitwise


def test_quantize_ties_and_extremes():
    # exact ties: amax = 127 makes s = 1 and x/s = x, so +-0.5, 2.5, -3.5 are ties
    x = np.array([[127.0, 0.5, -0.5, 2.5, -3.5, 126.5, -126.5, 0.0]], np.float32)
    ref = O.quantize_per_token(x)
    codes, scales = isb.quantize_per_token(dev(x))
    assert codes.cpu().numpy().astype(np.int16).tolist() == ref.values.tolist()
    assert ref.values.tolist() == [[127, 1, -1, 3, -4, 127, -127, 0]]
    # per-token pins, test_quantize.cpp:330-339
    x = np.array([[1.0, -2.0], [0.5, 0.25], [0.0, 0.0]], np.float32)
    codes, scales = isb.quantize_per_token(dev(x))
    assert scales.cpu().numpy().tolist() == [2.0 / 127.0, 0.5 / 127.0, 1.0]
    assert codes.cpu().numpy()[0, 1] == -127


def test_quantize_bf16_input_matches_float_of_bf16():
    xf = O.generate_gaussian(8, 4096, 1.0, 5)
    xb = torch.from_numpy(xf).to(torch.bfloat16)
    ref = O.quantize_per_token(xb.float().numpy())
    codes, scales = isb.quantize_per_token(xb.to(DEV))
    assert np.array_equal(codes.cpu().numpy().astype(np.int16), ref.values)
    assert np.array_equal(scales.cpu().numpy(), ref.scales)


def test_quantize_rejects_non_finite():
    x = np.ones((2, 64), np.float32)
    x[1, 3] = np.nan
    with pytest.raises(isb.ValueError_):
        isb.quantize_per_token(dev(x), check_finite=True)


def test_weight_group_quantizer_bit_exact():
    wf = O.generate_llama_like(512, 300, 7)
    ref = O.quantize_weight(wf, 128)
    codes, scales = isb.quantize_weight(dev(wf), 128, 4)
    assert np.array_equal(codes.cpu().numpy(), ref.values)
    assert np.array_equal(scales.cpu().numpy(), ref.scales)


# ------------------------------------------------------------------------- K2
@pytest.mark.parametrize("k,n", [(256, 128), (4096, 300), (384, 1), (130, 7), (8, 2)])
def test_pack_roundtrip_and_reference_bytes(k, n):
    rng = O.Rng(k * 1000 + n)
    codes = (rng.below(16, k * n) - 8).astype(np.int16).reshape(k, n)
    g = 2 if k % 128 else 128
    scales = np.full(n * (k // g), 0.01)
    w = isb.PackedWeight.from_codes(dev(codes), g, dev(scales))
    assert np.array_equal(w.unpack_codes().cpu().numpy(), codes)
    assert np.array_equal(w.repack_signed4().cpu().numpy(), O.pack_signed4(codes))
    # and from the reference byte stream
    w2 = isb.PackedWeight.from_signed4(dev(O.pack_signed4(codes)), k, n, g, dev(scales))
    assert np.array_equal(w2.unpack_codes().cpu().numpy(), codes)


def test_pack_rejects_out_of_range_and_bad_length():
    codes = np.zeros((128, 4), np.int16)
    codes[3, 1] = 8
    with pytest.raises(isb.ValueError_):
        isb.PackedWeight.from_codes(dev(codes), 128, dev(np.ones(4)))
    with pytest.raises(isb.LengthError):
        isb.PackedWeight.from_signed4(dev(np.zeros(3, np.uint8)), 2, 4, 2, dev(np.ones(4)))


# ------------------------------------------------------------------------- K3 / K4
SHAPES = [(1, 4096, 4096), (2, 256, 4), (8, 256, 300), (16, 4096, 4096), (16, 11008, 512),
          (33, 1024, 640), (64, 2048, 1024), (100, 512, 256), (128, 4096, 512),
          (300, 1024, 384)]


@pytest.mark.parametrize("m,k,n", SHAPES)
def test_integer_scale_bit_exact(m, k, n):
    x, w, s, _, _ = llama_problem(m, k, n, seed_w=42 + n, seed_x=43 + m)
    ref = O.gemm_integer_scale(x, w, s)
    pw = pack(w, s)
    xq, sa = dev(x.values, torch.int8), dev(x.scales)
    out32 = isb.gemm_integer_scale(xq, sa, pw, out_dtype=torch.float32)
    outbf = isb.gemm_integer_scale(xq, sa, pw, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    got = out32.cpu().numpy()
    assert np.array_equal(got.view(np.int32), ref.output.view(np.int32)), \
        f"max ulp {O.ulp_distance(got, ref.output).max()}"
    assert np.array_equal(outbf.float().cpu().numpy(), to_bf16_np(ref.output))


@pytest.mark.parametrize("m,k,n", SHAPES)
def test_float_scale_within_tolerance(m, k, n):
    x, w, s, _, _ = llama_problem(m, k, n, seed_w=42 + n, seed_x=43 + m)
    ref = O.gemm_float_scale(x, w)
    pw = pack(w, s)
    out = isb.gemm_float_scale(dev(x.values, torch.int8), dev(x.scales), pw,
                               out_dtype=torch.float32).cpu().numpy().astype(np.float64)
    # fp32 accumulation of K/g terms vs the reference's double: |err| <= G * 2^-23 * sum|terms|
    groups = k // 128
    scale_abs = np.abs(ref.partials).reshape(m, n, groups) * w.scales.reshape(n, groups)[None]
    bound = 2.0 * groups * 2.0 ** -23 * scale_abs.sum(axis=2) * x.scales[:, None] + 1e-30
    assert (np.abs(out - ref.output_f64) <= bound).all()


def test_integer_scale_alpha_8192_general_epilogue():
    # alpha = 8192 puts k_g up to ~124 (outside the k<=16 fold band)
    x, w, _, _, _ = llama_problem(16, 4096, 1024, amp=1024)
    s = O.integerize_scales(w.scales, 8192)
    assert s.int_scales.max() > 16
    assert O.overflow_analyzer(4096, 128, 8, 4, s)["safe"]
    ref = O.gemm_integer_scale(x, w, s)
    out = isb.gemm_integer_scale(dev(x.values, torch.int8), dev(x.scales), pack(w, s),
                                 out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(out.view(np.int32), ref.output.view(np.int32))


def test_random_instances_vs_oracle_tensor_core():
    rng = O.Rng(2718)
    for _ in range(20):
        m = 1 + rng.below(40)
        n = 1 + rng.below(300)
        k = 128 * (1 + rng.below(6))
        g = [128, k][rng.below(2)]
        x, w, _, _ = random_instance(rng, m, k, n, g)
        amp = O.search_amplifier(w.scales)
        s = O.integerize_scales(w.scales, amp)
        if not O.overflow_analyzer(k, g, 8, 4, s)["safe"]:
            continue
        ref = O.gemm_integer_scale(x, w, s)
        out = isb.gemm_integer_scale(dev(x.values, torch.int8), dev(x.scales), pack(w, s),
                                     out_dtype=torch.float32).cpu().numpy()
        assert np.array_equal(out.view(np.int32), ref.output.view(np.int32))


def test_workspace_is_left_clean_and_results_repeat():
    x, w, s, _, _ = llama_problem(16, 4096, 4096)
    pw = pack(w, s)
    xq, sa = dev(x.values, torch.int8), dev(x.scales)
    ws = isb.Workspace()
    a = isb.gemm_integer_scale(xq, sa, pw, torch.float32, workspace=ws)
    for _ in range(5):
        b = isb.gemm_integer_scale(xq, sa, pw, torch.float32, workspace=ws)
        assert torch.equal(a, b)
    torch.cuda.synchronize()
    assert int(ws.buf.view(torch.int32).abs().sum()) == 0  # split-K workspace left clean


@pytest.mark.parametrize("m", [1, 5, 16, 17, 32])
@pytest.mark.parametrize("k,n,g", [(4096, 12288, 128), (11008, 4096, 128), (4096, 22016, 128),
                                   (11008, 1000, 256), (2048, 640, 512), (256, 4, 128)])
def test_decode_stream_k_bit_exact(m, k, n, g):
    """Decode shapes on every LLaMA-2-7B linear plus ragged N / g > 128: int32 acc
    and float32 output bit-exact for every split pattern of the cluster split-K kernel."""
    x, w, s, _, _ = llama_problem(m, k, n, seed_w=7 + n + g, seed_x=11 + m, g=g)
    ref = O.gemm_integer_scale(x, w, s)
    pw = pack(w, s)
    xq, sa = dev(x.values, torch.int8), dev(x.scales)
    ws = isb.Workspace()
    for _ in range(2):  # second call reuses the workspace the first left clean
        out = isb.gemm_integer_scale(xq, sa, pw, out_dtype=torch.float32, workspace=ws)
        got = out.cpu().numpy()
        assert np.array_equal(got.view(np.int32), ref.output.view(np.int32))
    outf = isb.gemm_float_scale(xq, sa, pw, out_dtype=torch.float32, workspace=ws)
    rf = O.gemm_float_scale(x, w)
    err = np.abs(outf.cpu().numpy().astype(np.float64) - rf.output_f64)
    assert err.max() <= 1e-5 * np.abs(rf.output_f64).max() + 1e-30


# ------------------------------------------------------------------------- checked kernel
def test_checked_matches_oracle_stats_small_groups():
    rng = O.Rng(1007)
    for _ in range(30):
        m = 1 + rng.below(8)
        n = 1 + rng.below(8)
        k = 4 * (1 + rng.below(8))
        g = [1, 2, 4, k][rng.below(4)]
        x, w, _, _ = random_instance(rng, m, k, n, g)
        amp = O.search_amplifier(w.scales)
        s = O.integerize_scales(w.scales, amp)
        pw = pack(w, s)
        xq, sa = dev(x.values, torch.int8), dev(x.scales)
        ri = O.gemm_integer_scale(x, w, s)
        out, of, acc, part, st = isb.gemm_checked("integer-scale", xq, sa, pw, want_partials=True)
        assert np.array_equal(out.cpu().numpy().view(np.int32), ri.output.view(np.int32))
        assert np.array_equal(acc.cpu().numpy(), ri.acc)
        assert np.array_equal(part.cpu().numpy(), ri.partials)
        assert st["max_abs_accumulator"] == ri.stats["max_abs_accumulator"]
        rf = O.gemm_float_scale(x, w)
        out, of, _, _, st = isb.gemm_checked("float-scale", xq, sa, pw)
        assert np.array_equal(out.cpu().numpy().view(np.int32), rf.output.view(np.int32))
        assert np.array_equal(of.cpu().numpy(), rf.output_f64)
        assert st["max_abs_accumulator"] == rf.stats["max_abs_accumulator"]


def test_checked_overflow_rig():
    x, w, s = overflow_rig(2)
    pw = pack(w, s)
    xq, sa = dev(x.values, torch.int8), dev(x.scales)
    out, of, acc, _, st = isb.gemm_checked("integer-scale", xq, sa, pw)
    assert st["overflow_detected"] and st["max_abs_accumulator"] == 4260372480
    assert (st["overflow_i"], st["overflow_j"]) == (0, 0)
    assert acc.cpu().numpy()[0, 0] == -4260372480        # permissive: non-wrapped int64
    ref = O.gemm_integer_scale(x, w, s)
    assert np.array_equal(out.cpu().numpy().view(np.int32), ref.output.view(np.int32))
    with pytest.raises(isb.OverflowError_, match=r"\(0, 0\)"):
        isb.gemm_checked("integer-scale", xq, sa, pw, strict=True)


# ------------------------------------------------------------------------- K3 prefill (k_g folded)
FOLD_SHAPES = [(256, 1024, 256), (300, 1024, 384), (512, 2048, 640), (448, 11008, 128),
               (1000, 512, 1000), (777, 4096, 130)]


@pytest.mark.parametrize("m,k,n", FOLD_SHAPES)
def test_fold_prefill_bit_exact(m, k, n):
    """M >= 256 with k_g <= 16 runs the folded kernel (k_g * w expanded into the int8
    operand, whole-K accumulation in TMEM): float32 output 0 ULP, bf16 = RN(f32)."""
    x, w, s, _, _ = llama_problem(m, k, n, seed_w=100 + n, seed_x=200 + m)
    assert s.int_scales.max() <= 16
    ref = O.gemm_integer_scale(x, w, s)
    pw = pack(w, s)
    xq, sa = dev(x.values, torch.int8), dev(x.scales)
    out32 = isb.gemm_integer_scale(xq, sa, pw, out_dtype=torch.float32)
    outbf = isb.gemm_integer_scale(xq, sa, pw, out_dtype=torch.bfloat16)
    out16 = isb.gemm_integer_scale(xq, sa, pw, out_dtype=torch.float16)
    torch.cuda.synchronize()
    got = out32.cpu().numpy()
    assert np.array_equal(got.view(np.int32), ref.output.view(np.int32)), \
        f"max ulp {O.ulp_distance(got, ref.output).max()}"
    assert np.array_equal(outbf.float().cpu().numpy(), to_bf16_np(ref.output))
    assert np.array_equal(out16.float().cpu().numpy(),
                          torch.from_numpy(ref.output).half().float().numpy())


def test_fold_extreme_codes_and_k16():
    """The fold's edge: k_g = 16 with codes -8 and 7 (k*w = -128 / 112) and extreme
    activations (+-127), all in one tile, against the oracle."""
    m, k, n, g = 300, 512, 256, 128
    rng = np.random.default_rng(11)
    codes = rng.integers(-8, 8, size=(k, n)).astype(np.int16)
    codes[:64, :] = -8
    codes[64:128, :] = 7
    groups = k // g
    amp = 1024
    ks = rng.integers(1, 17, size=(n, groups))
    ks[:, 0] = 16
    scales = (ks / amp).astype(np.float64).reshape(-1)
    w = O.QuantizedTensor(codes, 4, O.SYMMETRIC, O.GROUP, g, scales, np.zeros(0, np.int32))
    s = O.integerize_scales(scales, amp)
    assert s.int_scales.max() == 16
    xv = rng.integers(-127, 128, size=(m, k)).astype(np.int16)
    xv[0, :] = 127
    xv[1, :] = -127
    x = O.QuantizedTensor(xv, 8, O.SYMMETRIC, O.PER_TOKEN, 0,
                          rng.uniform(1e-3, 1e-1, size=m).astype(np.float64), np.zeros(0, np.int32))
    assert O.overflow_analyzer(k, g, 8, 4, s)["safe"]
    ref = O.gemm_integer_scale(x, w, s)
    out = isb.gemm_integer_scale(dev(x.values, torch.int8), dev(x.scales), pack(w, s),
                                 out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(out.view(np.int32), ref.output.view(np.int32))


# ------------------------------------------------------------------------- K1 (+) K3 fused
@pytest.mark.parametrize("m,k,n", [(1, 4096, 4096), (5, 4096, 12288), (16, 11008, 4096),
                                   (16, 4096, 22016), (33, 2048, 640), (64, 4096, 1024),
                                   (100, 1024, 256)])
def test_act_fused_matches_quantize_then_gemm(m, k, n):
    """Config C3: per-token quantization fused into the GEMM (one launch) gives the
    reference codes/scales and the bit-exact integer-scale output; M = 100 takes the
    unfused fallback."""
    x, w, s, xf, _ = llama_problem(m, k, n, seed_w=23 + n, seed_x=29 + m)
    ref = O.gemm_integer_scale(x, w, s)
    pw = pack(w, s)
    xd = dev(xf)
    sa = torch.empty((m,), dtype=torch.float64, device=DEV)
    out = isb.gemm_act_fused(xd, pw, out_dtype=torch.float32, sa_out=sa)
    torch.cuda.synchronize()
    assert np.array_equal(sa.cpu().numpy(), x.scales)
    got = out.cpu().numpy()
    assert np.array_equal(got.view(np.int32), ref.output.view(np.int32))
    outf = isb.gemm_act_fused(xd, pw, path="float-scale", out_dtype=torch.float32)
    rf = O.gemm_float_scale(x, w)
    err = np.abs(outf.cpu().numpy().astype(np.float64) - rf.output_f64)
    assert err.max() <= 1e-5 * np.abs(rf.output_f64).max() + 1e-30


def test_act_fused_bf16_input_and_zero_rows():
    m, k, n = 7, 4096, 512
    x, w, s, xf, _ = llama_problem(m, k, n, seed_w=3, seed_x=4)
    xf[2, :] = 0.0  # an all-zero token: scale 1.0, codes 0 (quantize.cpp:123)
    xb = torch.from_numpy(xf).to(torch.bfloat16)
    xo = O.quantize_per_token(xb.float().numpy())
    ref = O.gemm_integer_scale(xo, w, s)
    pw = pack(w, s)
    sa = torch.empty((m,), dtype=torch.float64, device=DEV)
    out = isb.gemm_act_fused(xb.to(DEV), pw, out_dtype=torch.float32, sa_out=sa)
    torch.cuda.synchronize()
    assert np.array_equal(sa.cpu().numpy(), xo.scales)
    assert xo.scales[2] == 1.0
    assert np.array_equal(out.cpu().numpy().view(np.int32), ref.output.view(np.int32))


# ------------------------------------------------------------------------- runtime
@pytest.mark.parametrize("fused", [False, True])
def test_graphed_linears_match_direct_calls(fused):
    from paper_2405_14597_b200.runtime import GraphedLinears
    shapes = [(4096, 1024), (2048, 640)]
    m = 16
    ws, xs, refs = [], [], []
    for i, (k, n) in enumerate(shapes):
        x, w, s, xf, _ = llama_problem(m, k, n, seed_w=31 + i, seed_x=37 + i)
        ws.append(pack(w, s))
        xs.append(xf)
        refs.append(O.gemm_integer_scale(x, w, s).output)
    g = GraphedLinears(ws, m, out_dtype=torch.float32, fused=fused).capture()
    for step in range(3):
        for j, xf in enumerate(xs):
            g.host_inputs[j].copy_(torch.from_numpy(xf * (1.0 + step)))
        g.run()
        g.synchronize()
        for j, xf in enumerate(xs):
            k, n = shapes[j]
            x2 = O.quantize_per_token((xf * (1.0 + step)).astype(np.float32))
            w2 = O.QuantizedTensor  # noqa: F841 (weights unchanged)
            got = g.host_outputs[j].numpy()
            if step == 0:
                assert np.array_equal(got.view(np.int32), refs[j].view(np.int32))
            else:
                _, w, s, _, _ = llama_problem(m, k, n, seed_w=31 + j, seed_x=37 + j)
                ref = O.gemm_integer_scale(x2, w, s).output
                assert np.array_equal(got.view(np.int32), ref.view(np.int32))


# ------------------------------------------------------------------------- coarse (per-channel)
@pytest.mark.parametrize("m,k,n", [(1, 4096, 4096), (16, 4096, 1024), (5, 11008, 256),
                                   (100, 1024, 256), (300, 2048, 640)])
def test_coarse_per_channel_bit_exact(m, k, n):
    """gemm_coarse (gemm.cpp:264-309) on tcgen05: exact int32 sum over K, the
    reference's double epilogue (double(acc) * s_w) * s_a -> float32 0 ULP."""
    wf = O.generate_llama_like(k, n, 61 + n)
    xf = O.generate_gaussian(m, k, 1.0, 67 + m)
    w = O.quantize(wf, 4, O.SYMMETRIC, O.PER_CHANNEL, k)
    x = O.quantize_per_token(xf)
    ref = O.gemm_coarse(x, w)
    pw = isb.PackedWeight.from_codes(dev(w.values), k, dev(w.scales))
    xq, sa = dev(x.values, torch.int8), dev(x.scales)
    out = isb.gemm_coarse(xq, sa, pw, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(out.view(np.int32), ref.output.view(np.int32))
    outb = isb.gemm_coarse(xq, sa, pw, out_dtype=torch.bfloat16).float().cpu().numpy()
    assert np.array_equal(outb, to_bf16_np(ref.output))


def test_coarse_rejects_grouped_weights():
    x, w, s, _, _ = llama_problem(4, 1024, 256)
    with pytest.raises(isb.ParamError):
        isb.gemm_coarse(dev(x.values, torch.int8), dev(x.scales), pack(w, s))
