"""QServe-style dual quantization on the device (dual_inner_quantize, gemm.cpp:311-345;
gemm_dual_quant, gemm.cpp:347-412) against the oracle restatement: inner codes, scales
and zero points identical; float32 output and its double value bit-exact (the device
keeps the reference's sequential double accumulation)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from tests.instances import random_instance

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

import paper_2405_14597_b200 as isb  # noqa: E402

DEV = torch.device("cuda:0")


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    return (t.to(dtype) if dtype is not None else t).to(DEV)


def run_both(x, w8, g):
    inner_o = O.dual_inner_quantize(w8, g)
    inner_d = isb.dual_inner_quantize(dev(w8.values), g)
    assert np.array_equal(inner_d.codes.cpu().numpy(), inner_o.values)
    assert np.array_equal(inner_d.scales.cpu().numpy().view(np.int64), inner_o.scales.view(np.int64))
    assert np.array_equal(inner_d.zero_points.cpu().numpy(), inner_o.zero_points)
    ref = O.gemm_dual_quant(x, w8, inner_o)
    out, of = isb.gemm_dual_quant(dev(x.values, torch.int8), dev(x.scales), inner_d, w8.scales,
                                  want_f64=True)
    assert np.array_equal(out.cpu().numpy().view(np.int32), ref.output.view(np.int32))
    assert np.array_equal(of.cpu().numpy().view(np.int64), ref.output_f64.view(np.int64))


def test_dual_quant_random_instances_bit_exact():
    """test_gemm.cpp:253-292 ("all four paths agree with the oracle"), dual leg:
    mt19937_64 seed 2718 instance shapes, 8-bit per-channel outer weight."""
    rng = O.Rng(2718)
    for _ in range(20):
        m = 1 + rng.below(6)
        n = 1 + rng.below(6)
        kbase = 1 + rng.below(8)
        g = [1, 2, 4, 4 * kbase][rng.below(4)]
        k = 4 * kbase
        x, _, _, wf = random_instance(rng, m, k, n, g)
        w8 = O.quantize(wf, 8, O.SYMMETRIC, O.PER_CHANNEL, 0)
        run_both(x, w8, g)


@pytest.mark.parametrize("m,k,n,g", [(16, 4096, 4096, 128), (3, 11008, 256, 128), (64, 1024, 300, 64)])
def test_dual_quant_llama_shapes_bit_exact(m, k, n, g):
    wf = O.generate_llama_like(k, n, 42)
    xf = O.generate_gaussian(m, k, 1.0, 43)
    x = O.quantize_per_token(xf)
    w8 = O.quantize(wf, 8, O.SYMMETRIC, O.PER_CHANNEL, 0)
    run_both(x, w8, g)


def test_dual_quant_scalar_example_and_validation():
    """test_gemm.cpp:183-199 ((5 - 3) * 0.5 * 1 = 1.0f) and the value checks of
    gemm.cpp:366-372 / validate_activation (gemm.cpp:114)."""
    inner = isb.DualInner(dev(np.array([[5]], np.int16)), dev(np.array([0.5])),
                          dev(np.array([3], np.int32)), 1)
    xq, sa = dev(np.array([[1]], np.int8)), dev(np.array([1.0]))
    assert float(isb.gemm_dual_quant(xq, sa, inner, [1.0])[0, 0]) == 1.0
    bad = isb.DualInner(dev(np.array([[16]], np.int16)), inner.scales, inner.zero_points, 1)
    with pytest.raises(isb.ValueError_):
        isb.gemm_dual_quant(xq, sa, bad, [1.0])
    badz = isb.DualInner(inner.codes, inner.scales, dev(np.array([16], np.int32)), 1)
    with pytest.raises(isb.ValueError_):
        isb.gemm_dual_quant(xq, sa, badz, [1.0])
    bads = isb.DualInner(inner.codes, dev(np.array([0.0])), inner.zero_points, 1)
    with pytest.raises(isb.ValueError_):
        isb.gemm_dual_quant(xq, sa, bads, [1.0])
    with pytest.raises(isb.ValueError_):
        isb.gemm_dual_quant(dev(np.array([[-128]], np.int8)), sa, inner, [1.0])
    with pytest.raises(isb.ParamError):
        isb.dual_inner_quantize(dev(np.zeros((6, 2), np.int16)), 4)


def test_dual_identity_inner_equals_coarse():
    """acceptance.cpp:397-415: identity inner stage (s = 1, z = 0, g = K) over codes in
    [0, 15] equals the coarse path bit for bit — on the device, dual vs coarse kernels."""
    rng = O.Rng(23)
    m, k, n = 5, 256, 130
    xq = (rng.below(255, m * k) - 127).astype(np.int16).reshape(m, k)
    wq = rng.below(16, k * n).astype(np.int16).reshape(k, n)
    sw = np.exp2(-6.0 + 6.0 * rng.u01(n))
    x = O.QuantizedTensor(xq, 8, O.SYMMETRIC, O.PER_TOKEN, 0, 0.01 + rng.u01(m), np.zeros(0, np.int32))
    outer = O.QuantizedTensor(wq, 8, O.SYMMETRIC, O.PER_CHANNEL, k, sw, np.zeros(0, np.int32))
    ident = isb.DualInner(dev(wq), dev(np.ones(n)), dev(np.zeros(n, np.int32)), k)
    out = isb.gemm_dual_quant(dev(xq, torch.int8), dev(x.scales), ident, sw).cpu().numpy()
    rc = O.gemm_coarse(x, outer).output
    assert np.array_equal(out.view(np.int32), rc.view(np.int32))
