"""Pins the CPU oracle (oracle/oracle.cpp) against every golden vector and
known-answer test the reference's own suite holds for the hot path
(SURVEY.md §8c). Each test cites the reference test it transcribes.

The reference cannot be compiled in this image (Eigen3 absent), so these
transcriptions ARE the oracle's parity pin.
"""
import numpy as np
import pytest

from oracle import oracle as O
from tests.instances import random_instance, make_x, make_w, overflow_rig


def q_act(rows, scales):
    """make_activation, test_gemm.cpp:31-48."""
    v = np.array(rows, np.int16)
    return O.QuantizedTensor(v, 8, O.SYMMETRIC, O.PER_TOKEN, 0, np.array(scales, np.float64),
                             np.zeros(0, np.int32))


def q_w(rows, scales, bits, kind, group=0):
    """make_weight, test_gemm.cpp:50-67."""
    v = np.array(rows, np.int16)
    return O.QuantizedTensor(v, bits, O.SYMMETRIC, kind, group, np.array(scales, np.float64),
                             np.zeros(0, np.int32))


# --------------------------------------------------------------------------- generators
def test_generator_determinism():  # test_tensor_io.cpp:226-240
    a = O.generate_gaussian(16, 16, 1.0, 42)
    assert np.array_equal(a, O.generate_gaussian(16, 16, 1.0, 42))
    assert not np.array_equal(a, O.generate_gaussian(16, 16, 1.0, 43))
    u = O.generate_uniform(8, 8, -2.0, 3.0, 7)
    assert np.array_equal(u, O.generate_uniform(8, 8, -2.0, 3.0, 7))
    assert (u >= -2.0).all() and (u < 3.0).all()
    l = O.generate_llama_like(256, 8, 11)
    assert np.array_equal(l, O.generate_llama_like(256, 8, 11))


def test_degenerate_uniform():  # test_tensor_io.cpp:243-248
    assert (O.generate_uniform(4, 4, 0.0, 0.0, 1) == 0.0).all()
    assert (O.generate_uniform(4, 4, 2.5, 2.5, 1) == 2.5).all()


def test_generator_validation():  # test_tensor_io.cpp:250-256
    for args in [(0, 4), (4, 0)]:
        with pytest.raises(O.OracleError) as e:
            O.generate_gaussian(*args, 1.0, 0)
        assert e.value.code == O.PARAM
    for sigma in (0.0, -1.0):
        with pytest.raises(O.OracleError):
            O.generate_gaussian(4, 4, sigma, 0)
    with pytest.raises(O.OracleError):
        O.generate_uniform(4, 4, 1.0, 0.0, 0)
    with pytest.raises(O.OracleError) as e:
        O.generate_llama_like(100, 4, 0)
    assert e.value.code == O.PARAM


def test_llama_like_min_scale_window():  # test_tensor_io.cpp:258-270
    for seed in (1, 2, 3, 4, 5):
        w = O.generate_llama_like(256, 16, seed)
        q = O.quantize_weight(w, 128)
        assert 2.0 ** -10 < q.scales.min() < 2.0 ** -9
        assert q.scales.max() <= 2.0 ** -6 * (1.0 + 1e-6)


def test_readme_search_amplifier_example():  # proj/README.md:115-122
    w = O.generate_llama_like(4096, 8, 1)
    q = O.quantize_weight(w, 128)
    assert q.scales.size == 256
    assert q.scales.min() == 0.0010120436948324954
    assert O.search_amplifier(q.scales) == 1024
    assert O.search_amplifier_exponent(q.scales) == 10


def test_readme_gemm_example():  # proj/README.md:124-135, CLI synthesis intscale_cli.cpp:123-135,185-196
    seed = 3
    w = O.quantize_weight(O.generate_llama_like(256, 4, seed), 128)
    x = O.quantize_per_token(O.generate_gaussian(2, 256, 1.0, seed + 1))
    s = O.integerize_scales(w.scales, O.search_amplifier(w.scales))
    r = O.gemm_integer_scale(x, w, s)
    assert r.stats["int_to_float_conversions"] == 8
    assert r.stats["integer_multiply_adds"] == 2064
    assert r.stats["max_abs_accumulator"] == 10106
    assert not r.stats["overflow_detected"]


# --------------------------------------------------------------------------- quantizer
def test_symmetric_pins():  # test_quantize.cpp:75-97
    q = O.quantize(np.array([[0.0, 7.0, -7.0]], np.float32), 4, O.SYMMETRIC, O.PER_TENSOR, 0)
    assert q.scales.tolist() == [1.0]
    assert q.values.tolist() == [[0, 7, -7]]
    q8 = O.quantize(np.array([[1.0]], np.float32), 8, O.SYMMETRIC, O.PER_TENSOR, 0)
    assert q8.scales[0] == 1.0 / 127.0
    assert q8.values[0, 0] == 127


def test_asymmetric_pins():  # test_quantize.cpp:99-120
    q = O.quantize(np.array([[0.0, 3.0]], np.float32), 4, O.ASYMMETRIC, O.PER_TENSOR, 0)
    assert q.scales[0] == 0.2 and q.zero_points[0] == 0
    assert q.values.tolist() == [[0, 15]]
    qn = O.quantize(np.array([[-3.0, 1.0]], np.float32), 4, O.ASYMMETRIC, O.PER_TENSOR, 0)
    assert abs(qn.scales[0] - 4.0 / 15.0) <= 1e-15 * 4.0 / 15.0
    assert qn.zero_points[0] == 11
    assert qn.values.tolist() == [[0, 15]]


def test_zero_range_units():  # test_quantize.cpp:122-136
    qs = O.quantize(np.zeros((4, 4), np.float32), 4, O.SYMMETRIC, O.PER_TOKEN, 0)
    assert (qs.scales == 1.0).all() and (qs.values == 0).all()


def test_unit_bookkeeping():  # test_quantize.cpp:43-62
    assert O.unit_count(O.PER_TENSOR, 0, 8, 6) == 1
    assert O.unit_count(O.PER_TOKEN, 0, 8, 6) == 8
    assert O.unit_count(O.PER_CHANNEL, 0, 8, 6) == 6
    assert O.unit_count(O.GROUP, 4, 8, 6) == 12
    assert O.unit_count(O.GROUP, 128, 4096, 4096) == 131072
    for g in (3, 0):
        with pytest.raises(O.OracleError) as e:
            O.unit_count(O.GROUP, g, 8, 2)
        assert e.value.code == O.PARAM


def test_per_token_scales():  # test_quantize.cpp:330-339
    x = np.array([[1.0, -2.0], [0.5, 0.25], [0.0, 0.0]], np.float32)
    q = O.quantize_per_token(x)
    assert q.scales[0] == 2.0 / 127.0
    assert q.scales[1] == 0.5 / 127.0
    assert q.scales[2] == 1.0
    assert q.values[0, 1] == -127


def test_ties_away_from_zero():  # test_integer_scale.cpp:127-132 (codes col0 [7, -4])
    w1 = np.array([[0.875, 3.5], [-0.4375, -1.75]], np.float32)
    q = O.quantize(w1, 4, O.SYMMETRIC, O.GROUP, 2)
    assert q.scales.tolist() == [0.125, 0.5]
    assert q.values[:, 0].tolist() == [7, -4]
    assert q.values[:, 1].tolist() == [7, -4]


def test_half_step_bound():  # test_quantize.cpp:148-189 (property)
    rng = O.Rng(5)
    x = (4.0 * rng.u01(64 * 256) - 2.0).astype(np.float32).reshape(64, 256)
    q = O.quantize_per_token(x)
    recon = q.values.astype(np.float64) * q.scales[:, None]
    assert (np.abs(recon - x.astype(np.float64)) <= q.scales[:, None] / 2 * (1 + 1e-12)).all()


# --------------------------------------------------------------------------- integer scale
def test_amplifier_search_pins():  # test_integer_scale.cpp:26-34
    assert O.search_amplifier([0.3, 0.9, 5.0]) == 4
    assert O.search_amplifier([0.5]) == 2
    assert O.search_amplifier([1.5, 2.0]) == 1
    assert O.search_amplifier([1.0]) == 1
    assert O.search_amplifier([2.0 ** -10]) == 1024
    assert O.search_amplifier_exponent([2.0 ** -10, 0.25]) == 10


def test_amplifier_search_validation():  # test_integer_scale.cpp:36-42
    for bad in ([], [0.0], [-0.5], [float("nan")], [1e-300]):
        with pytest.raises(O.OracleError) as e:
            O.search_amplifier(bad)
        assert e.value.code == O.PARAM


def test_integerize_pins():  # test_integer_scale.cpp:44-57
    s = O.integerize_scales([0.25, 0.125], 8)
    assert s.amplifier == 8 and s.exponent == 3 and s.int_scales.tolist() == [2, 1]
    assert O.integerize_scales([0.3], 4).int_scales[0] == 1
    assert O.integerize_scales([1.0], 1024).int_scales[0] == 1024
    assert O.integerize_scales([0.0001], 1024).int_scales[0] == 1
    assert O.integerize_scales([2.5 / 1024], 1024).int_scales[0] == 3
    assert O.integerize_scales([1.5 / 1024], 1024).int_scales[0] == 2


def test_integerize_validation():  # test_integer_scale.cpp:59-66
    for amp in (0, 3, -4):
        with pytest.raises(O.OracleError) as e:
            O.integerize_scales([0.5], amp)
        assert e.value.code == O.PARAM
    for s in ([], [-1.0]):
        with pytest.raises(O.OracleError) as e:
            O.integerize_scales(s, 8)
        assert e.value.code == O.PARAM
    with pytest.raises(O.OracleError) as e:
        O.integerize_scales([3.0e6], 1024)
    assert e.value.code == O.OVERFLOW


def test_integerize_half_unit():  # test_integer_scale.cpp:109-119
    rng = O.Rng(99)
    for _ in range(200):
        s = O.exp2(-11.0 + 13.0 * rng.u01())
        k = O.integerize_scales([s], 1024).int_scales[0]
        assert abs(k / 1024 - s) <= 1.0 / 2048


# --------------------------------------------------------------------------- packing
def test_nibble_pins():  # test_tensor_io.cpp:65-86
    assert O.pack_signed4([[-8, 7]]).tolist() == [0x78]
    assert O.unpack_signed4(bytes([0x78]), 1, 2).tolist() == [[-8, 7]]
    assert O.pack_signed4([[3]]).tolist() == [0x03]
    assert O.pack_signed4([[-1]]).tolist() == [0x0F]
    assert O.unpack_signed4(bytes([0x0F]), 1, 1).tolist() == [[-1]]
    v8 = [[-8, -1, 0, 1, 2, -2, 7, -7]]
    assert O.pack_signed4(v8).tolist() == [0xF8, 0x10, 0xE2, 0x97]
    assert O.unpack_signed4(bytes([0xF8, 0x10, 0xE2, 0x97]), 1, 8).tolist() == v8
    for bad in ([[8]], [[-9]]):
        with pytest.raises(O.OracleError) as e:
            O.pack_signed4(bad)
        assert e.value.code == O.VALUE
    with pytest.raises(O.OracleError) as e:
        O.unpack_signed4(bytes([0xF8]), 1, 3)
    assert e.value.code == O.LENGTH


# --------------------------------------------------------------------------- overflow bound
def test_overflow_bound_pins():  # test_analysis.cpp:33-62
    r = O.overflow_analyzer(128, 128, 8, 4, O.IntegerScaleSet(np.array([1], np.int32), 1, 0))
    assert r["static_bound"] == 130048 and r["safe"]
    assert abs(r["headroom_bits"] - 14.0113) <= 14.0113 * 1e-3
    s = O.IntegerScaleSet(np.full(32, 1024, np.int32), 1024, 10)
    r = O.overflow_analyzer(4096, 128, 8, 4, s)
    assert r["static_bound"] == 4261412864 and not r["safe"] and r["headroom_bits"] < 0
    r = O.overflow_analyzer(4, 2, 4, 4, O.IntegerScaleSet(np.array([1, 2, 3, 4], np.int32), 1, 0))
    assert r["static_bound"] == 784 and r["safe"]


def test_overflow_analyzer_validation():  # test_analysis.cpp:64-70
    one = O.IntegerScaleSet(np.array([1], np.int32), 1, 0)
    zero = O.IntegerScaleSet(np.array([0], np.int32), 1, 0)
    for args in [(128, 100, 8, 4, one), (128, 128, 6, 4, one), (128, 128, 8, 5, one),
                 (128, 128, 8, 4, zero), (256, 128, 8, 4, one)]:
        with pytest.raises(O.OracleError) as e:
            O.overflow_analyzer(*args)
        assert e.value.code == O.PARAM


def test_expected_counters():  # test_analysis.cpp:106-124
    assert O.expected_counters("float-scale", 2, 3, 8, 4) == (12, 48)
    assert O.expected_counters("integer-scale", 2, 3, 8, 4) == (6, 60)
    assert O.expected_counters("coarse", 2, 3, 8, 8) == (6, 48)
    assert O.expected_counters("dual-quant", 2, 3, 8, 4) == (48, 0)


# --------------------------------------------------------------------------- GEMM
def test_scalar_hand_example():  # test_gemm.cpp:94-118
    x = q_act([[2, 3]], [0.5])
    w = q_w([[4], [5]], [0.25, 0.125], 4, O.GROUP, 1)
    rf = O.gemm_float_scale(x, w)
    assert rf.output[0, 0] == np.float32(1.9375)
    assert rf.stats["int_to_float_conversions"] == 2
    assert rf.stats["integer_multiply_adds"] == 2
    assert rf.stats["max_abs_accumulator"] == 15
    assert not rf.stats["overflow_detected"]
    s = O.integerize_scales(w.scales, 8)
    assert s.int_scales.tolist() == [2, 1]
    ri = O.gemm_integer_scale(x, w, s)
    assert ri.output[0, 0] == np.float32(1.9375)
    assert ri.stats["int_to_float_conversions"] == 1
    assert ri.stats["integer_multiply_adds"] == 4
    assert ri.stats["max_abs_accumulator"] == 31
    assert ri.acc[0, 0] == 31


def test_unit_scales_plain_matmul():  # test_gemm.cpp:120-135
    x = q_act([[1, 2, 3, 4], [-1, 0, 1, 0]], [1.0, 1.0])
    w = q_w([[1, -1], [2, 0], [0, 3], [-2, 1]], [1.0, 1.0], 4, O.PER_CHANNEL)
    rf = O.gemm_float_scale(x, w)
    assert rf.output.tolist() == [[-3.0, 12.0], [-1.0, 4.0]]


def test_int_scales_equal_amplifier_is_coarse():  # test_gemm.cpp:137-166
    rng = O.Rng(17)
    m, k, n, g = 3, 8, 4, 2
    xq = np.empty((m, k), np.int16)
    for i in range(m):
        for j in range(k):
            xq[i, j] = int(rng.next(1)[0] % np.uint64(255)) - 127
    wq = np.empty((k, n), np.int16)
    for i in range(k):
        for j in range(n):
            wq[i, j] = int(rng.next(1)[0] % np.uint64(16)) - 8
    xs = np.array([0.25 + rng.u01() for _ in range(m)])
    x = O.QuantizedTensor(xq, 8, O.SYMMETRIC, O.PER_TOKEN, 0, xs, np.zeros(0, np.int32))
    wg = O.QuantizedTensor(wq, 4, O.SYMMETRIC, O.GROUP, g, np.ones((k // g) * n),
                           np.zeros(0, np.int32))
    wc = O.QuantizedTensor(wq, 4, O.SYMMETRIC, O.PER_CHANNEL, 0, np.ones(n), np.zeros(0, np.int32))
    coarse = O.gemm_float_scale(x, wc).output   # per-channel float == coarse (test_gemm.cpp:168-181)
    for amp in (1, 8, 1024):
        s = O.integerize_scales(wg.scales, amp)
        assert np.array_equal(O.gemm_integer_scale(x, wg, s).output, coarse)


def test_forty_random_instances_vs_oracle():  # test_gemm.cpp:253-292
    rng = O.Rng(2718)
    for _ in range(40):
        m = 1 + rng.below(6)
        n = 1 + rng.below(6)
        kbase = 1 + rng.below(8)
        g = [1, 2, 4, 4 * kbase][rng.below(4)]
        k = 4 * kbase
        x, w, _, _ = random_instance(rng, m, k, n, g)
        rf = O.gemm_float_scale(x, w)
        assert (O.ulp_distance(rf.output, O.gemm_oracle("float-scale", x, w)) <= 1).all()
        amp = O.search_amplifier(w.scales)
        s = O.integerize_scales(w.scales, amp)
        ri = O.gemm_integer_scale(x, w, s)
        assert (O.ulp_distance(ri.output, O.gemm_oracle("integer-scale", x, w, amp)) <= 1).all()


def test_zero_activation():  # test_gemm.cpp:294-301
    x = q_act([[0, 0]], [1.0])
    w = q_w([[3, -2], [5, 1]], [0.25, 0.5], 4, O.PER_CHANNEL)
    assert (O.gemm_float_scale(x, w).output == 0).all()
    s = O.integerize_scales(w.scales, 1024)
    assert (O.gemm_integer_scale(x, w, s).output == 0).all()


def test_operand_validation():  # test_gemm.cpp:303-339
    x = q_act([[1, 2]], [1.0])
    w = q_w([[1], [1]], [1.0], 4, O.GROUP, 1)

    def code(fn):
        with pytest.raises(O.OracleError) as e:
            fn()
        return e.value.code

    assert code(lambda: O.gemm_float_scale(x, w)) == O.PARAM
    w3 = q_w([[1], [1], [1]], [1.0, 1.0, 1.0], 4, O.GROUP, 1)
    assert code(lambda: O.gemm_float_scale(x, w3)) == O.DIMENSION
    wok = q_w([[1], [1]], [1.0, 1.0], 4, O.GROUP, 1)
    O.gemm_float_scale(x, wok)
    xs = O.QuantizedTensor(x.values, 8, O.SYMMETRIC, O.PER_TENSOR, 0, x.scales, x.zero_points)
    assert code(lambda: O.gemm_float_scale(xs, wok)) == O.PARAM
    x4 = O.QuantizedTensor(x.values, 4, O.SYMMETRIC, O.PER_TOKEN, 0, x.scales, x.zero_points)
    assert code(lambda: O.gemm_float_scale(x4, wok)) == O.PARAM
    xneg = q_act([[-128, 0]], [1.0])
    assert code(lambda: O.gemm_float_scale(xneg, wok)) == O.VALUE
    wbig = q_w([[9], [1]], [1.0, 1.0], 4, O.GROUP, 1)
    assert code(lambda: O.gemm_float_scale(x, wbig)) == O.VALUE
    s = O.integerize_scales(wok.scales, 8)
    tampered = O.IntegerScaleSet(s.int_scales.copy(), s.amplifier, s.exponent)
    tampered.int_scales[0] += 1
    assert code(lambda: O.gemm_integer_scale(x, wok, tampered)) == O.PARAM


def test_overflow_rig_permissive_and_strict():  # test_gemm.cpp:345-383
    x, w, s = overflow_rig(2)
    assert x.scales[0] == 1.0
    assert (w.values == -7).all()
    assert (s.int_scales == 1170).all()
    r = O.gemm_integer_scale(x, w, s)
    assert r.stats["overflow_detected"]
    assert r.stats["max_abs_accumulator"] == 113792 * 1170 * 32 == 4260372480
    rep = O.overflow_analyzer(4096, 128, 8, 4, s)
    assert not rep["safe"]
    assert r.stats["max_abs_accumulator"] <= rep["static_bound"]
    with pytest.raises(O.OracleError) as e:
        O.gemm_integer_scale(x, w, s, strict=True)
    assert e.value.code == O.OVERFLOW and "(0, 0)" in e.value.msg
    # permissive still returns the non-wrapped int64 result (gemm.cpp:246-252)
    assert r.acc[0, 0] == -4260372480


def test_fallback_policy():  # test_gemm.cpp:385-407 and test_cli.cpp:236-243
    x, w, s = overflow_rig(2)
    r = O.run_layer(x, w, "integer-scale", s, fallback=True)
    assert r.stats["fallback_applied"]
    rf = O.gemm_float_scale(x, w)
    assert np.array_equal(r.output, rf.output)
    assert r.stats["int_to_float_conversions"] == rf.stats["int_to_float_conversions"] == 2 * 32
    assert not r.stats["overflow_detected"]
    rng = O.Rng(23)
    xi, wi, _, _ = random_instance(rng, 2, 8, 3, 4)
    si = O.integerize_scales(wi.scales, O.search_amplifier(wi.scales))
    rs = O.run_layer(xi, wi, "integer-scale", si, fallback=True)
    assert not rs.stats["fallback_applied"]
    assert rs.stats["int_to_float_conversions"] == 6
    rn = O.run_layer(x, w, "integer-scale", s, fallback=False)
    assert not rn.stats["fallback_applied"] and rn.stats["overflow_detected"]


def test_recorded_partials():  # test_gemm.cpp:409-425
    rng = O.Rng(29)
    x, w, _, _ = random_instance(rng, 3, 16, 4, 4)
    r = O.gemm_float_scale(x, w)
    groups = 4
    xv, wv = x.values.astype(np.int64), w.values.astype(np.int64)
    for i in range(3):
        for j in range(4):
            for gi in range(groups):
                p = int((xv[i, gi * 4:(gi + 1) * 4] * wv[gi * 4:(gi + 1) * 4, j]).sum())
                assert r.partials[i, j * groups + gi] == p
    assert np.array_equal(r.output, r.output_f64.astype(np.float32))


def test_amplifier_error_bound():  # test_gemm.cpp:427-450
    rng = O.Rng(31)
    for _ in range(30):
        x, w, _, _ = random_instance(rng, 2, 32, 4, 8)
        amp = O.search_amplifier(w.scales)
        s = O.integerize_scales(w.scales, amp)
        ri = O.gemm_integer_scale(x, w, s)
        rf = O.gemm_float_scale(x, w)
        sum_abs = np.abs(ri.partials).reshape(2, 4, 4).sum(axis=2)
        bound = x.scales[:, None] * sum_abs / (2.0 * amp)
        diff = np.abs(ri.output_f64 - rf.output_f64)
        assert (diff <= bound * (1 + 1e-9) + 1e-300).all()


def test_worker_invariance():  # test_gemm.cpp:452-484
    rng = O.Rng(37)
    x, w, _, _ = random_instance(rng, 16, 32, 8, 8)
    s = O.integerize_scales(w.scales, O.search_amplifier(w.scales))
    f1 = O.gemm_float_scale(x, w)
    i1 = O.gemm_integer_scale(x, w, s)
    for workers in (2, 3, 8):
        f = O.gemm_float_scale(x, w, workers=workers)
        assert np.array_equal(f.output, f1.output)
        assert f.stats["max_abs_accumulator"] == f1.stats["max_abs_accumulator"]
        ii = O.gemm_integer_scale(x, w, s, workers=workers)
        assert np.array_equal(ii.output, i1.output)
        assert ii.stats["max_abs_accumulator"] == i1.stats["max_abs_accumulator"]
    xr, wr, sr = overflow_rig(4)
    with pytest.raises(O.OracleError) as e:
        O.gemm_integer_scale(xr, wr, sr, strict=True, workers=4)
    assert e.value.code == O.OVERFLOW


def test_counter_closed_forms():  # test_gemm.cpp:486-520
    rng = O.Rng(41)
    for _ in range(10):
        m = 1 + rng.below(5)
        n = 1 + rng.below(5)
        k = 8 * (1 + rng.below(4))
        g = 4
        x, w, _, _ = random_instance(rng, m, k, n, g)
        s = O.integerize_scales(w.scales, O.search_amplifier(w.scales))
        rf = O.gemm_float_scale(x, w)
        assert rf.stats["int_to_float_conversions"] == m * n * (k // g)
        assert rf.stats["integer_multiply_adds"] == m * n * k
        ri = O.gemm_integer_scale(x, w, s)
        assert ri.stats["int_to_float_conversions"] == m * n
        assert ri.stats["integer_multiply_adds"] == m * n * (k + k // g)


# --------------------------------------------------------------------------- acceptance
def test_acceptance_1_dyadic_agreement():  # acceptance.cpp:86-128
    rng = O.Rng(1001)
    amp = 1024
    worst = 0
    for _ in range(1000):
        m = 1 + rng.below(64)
        n = 1 + rng.below(64)
        k = 4 * (1 + rng.below(16))
        g = [1, 2, 4, k][rng.below(4)]
        units = (k // g) * n
        ws = (1 + rng.below(4096, units)).astype(np.float64) / amp
        xs = (1 + rng.below(1024, m)).astype(np.float64) / 256.0
        x = make_x(rng, m, k, xs)
        w = make_w(rng, k, n, g, ws)
        s = O.integerize_scales(ws, amp)
        rf = O.gemm_float_scale(x, w, record=False)
        ri = O.gemm_integer_scale(x, w, s, record=False)
        worst = max(worst, int(O.ulp_distance(rf.output, ri.output).max()))
    assert worst <= 1


def test_acceptance_2_bounded_agreement():  # acceptance.cpp:133-188
    rng = O.Rng(1002)
    amp = 1024
    for _ in range(1000):
        m = 1 + rng.below(8)
        n = 1 + rng.below(8)
        k = 4 * (1 + rng.below(8))
        g = [1, 2, 4, k][rng.below(4)]
        groups = k // g
        units = groups * n
        ws = np.array([O.exp2(-11.0 + 13.0 * rng.u01()) * (1.0 + rng.u01()) for _ in range(units)])
        xs = np.array([O.exp2(-8.0 + 12.0 * rng.u01()) for _ in range(m)])
        x = make_x(rng, m, k, xs)
        w = make_w(rng, k, n, g, ws)
        s = O.integerize_scales(ws, amp)
        rf = O.gemm_float_scale(x, w)
        ri = O.gemm_integer_scale(x, w, s)
        sum_abs = np.abs(ri.partials).reshape(m, n, groups).sum(axis=2)
        bound = xs[:, None] * sum_abs / (2.0 * amp)
        diff = np.abs(ri.output_f64 - rf.output_f64)
        assert (diff <= bound * (1 + 1e-9) + 1e-300).all()
        assert np.array_equal(rf.output, rf.output_f64.astype(np.float32))
        assert np.array_equal(ri.output, ri.output_f64.astype(np.float32))


@pytest.mark.slow
def test_acceptance_3_conversion_accounting():  # acceptance.cpp:193-221
    m, k, n, g = 1, 4096, 22016, 128
    wq = O.quantize_weight(O.generate_llama_like(k, n, 42), g)
    xq = O.quantize_per_token(O.generate_gaussian(m, k, 1.0, 43))
    rf = O.gemm_float_scale(xq, wq, record=False)
    s = O.integerize_scales(wq.scales, 1024)
    ri = O.gemm_integer_scale(xq, wq, s, record=False)
    assert rf.stats["int_to_float_conversions"] == 704512
    assert ri.stats["int_to_float_conversions"] == 22016
    sq = O.quantize_weight(O.generate_llama_like(4096, 4096, 44), 128)
    assert sq.scales.size == 131072
    # llama_like at alpha=1024 keeps every k in [1, 15] (the fold-safe band).
    assert s.int_scales.min() >= 1 and s.int_scales.max() <= 15


def test_acceptance_7_oracle_and_partials():  # acceptance.cpp:334-427 (fine-grained paths)
    rng = O.Rng(1007)
    for _ in range(500):
        m = 1 + rng.below(8)
        n = 1 + rng.below(8)
        k = 4 * (1 + rng.below(8))
        g = [1, 2, 4, k][rng.below(4)]
        groups = k // g
        mag = O.exp2(-8.0 + 8.0 * rng.u01())
        xf = (4.0 * rng.u01(m * k) - 2.0).astype(np.float32).reshape(m, k)
        wf = ((2.0 * rng.u01(k * n) - 1.0) * mag).astype(np.float32).reshape(k, n)
        x = O.quantize_per_token(xf)
        w = O.quantize(wf, 4, O.SYMMETRIC, O.GROUP, g)
        amp = O.search_amplifier(w.scales)
        s = O.integerize_scales(w.scales, amp)
        rf = O.gemm_float_scale(x, w)
        ri = O.gemm_integer_scale(x, w, s)
        assert (O.ulp_distance(rf.output, O.gemm_oracle("float-scale", x, w)) <= 1).all()
        assert (O.ulp_distance(ri.output, O.gemm_oracle("integer-scale", x, w, amp)) <= 1).all()
        ref_p = np.einsum("mgk,gkn->mng", x.values.astype(np.int64).reshape(m, groups, g),
                          w.values.astype(np.int64).reshape(groups, g, n)).reshape(m, n * groups)
        assert np.array_equal(rf.partials, ref_p) and np.array_equal(ri.partials, ref_p)
        # skip the coarse/dual draws: acceptance.cpp:396-399 draws k*n + n more values
        rng.next(k * n + n)


def test_acceptance_8_overflow_soundness():  # acceptance.cpp:432-504
    rng = O.Rng(1008)
    for _ in range(300):
        m = 1 + rng.below(6)
        n = 1 + rng.below(6)
        k = 4 * (1 + rng.below(8))
        g = [1, 2, 4, k][rng.below(4)]
        units = (k // g) * n
        ws = np.array([O.exp2(-11.0 + 13.0 * rng.u01()) * (1.0 + rng.u01()) for _ in range(units)])
        xs = np.array([O.exp2(-4.0 + 8.0 * rng.u01()) for _ in range(m)])
        x = make_x(rng, m, k, xs)
        w = make_w(rng, k, n, g, ws)
        s = O.integerize_scales(ws, 1024)
        ones = O.IntegerScaleSet(np.ones(units, np.int32), 1, 0)
        ri = O.gemm_integer_scale(x, w, s, record=False)
        assert ri.stats["max_abs_accumulator"] <= O.overflow_analyzer(k, g, 8, 4, s)["static_bound"]
        rf = O.gemm_float_scale(x, w, record=False)
        assert rf.stats["max_abs_accumulator"] <= O.overflow_analyzer(k, g, 8, 4, ones)["static_bound"]
    x, w, s = overflow_rig(2)
    rep = O.overflow_analyzer(4096, 128, 8, 4, s)
    with pytest.raises(O.OracleError):
        O.gemm_integer_scale(x, w, s, strict=True)
    perm = O.gemm_integer_scale(x, w, s)
    assert perm.stats["overflow_detected"]
    assert perm.stats["max_abs_accumulator"] <= rep["static_bound"]
    fb = O.run_layer(x, w, "integer-scale", s, fallback=True)
    assert fb.stats["fallback_applied"] and not rep["safe"]
    assert np.array_equal(fb.output, O.gemm_float_scale(x, w).output)


def test_coarse_equals_integer_path_when_k_equals_alpha():
    """test_gemm.cpp:137-166 ("integer scales equal to the amplifier reproduce coarse
    exactly"): group-of-2 unit scales integerised at alpha in {1, 8, 1024} vs
    per-channel unit scales through gemm_coarse — identical outputs."""
    rng = O.Rng(17)
    m, k, n, g = 3, 8, 4, 2
    xq = (rng.below(255, m * k) - 127).astype(np.int16).reshape(m, k)
    wq = (rng.below(16, k * n) - 8).astype(np.int16).reshape(k, n)
    sa = 0.25 + rng.u01(m)
    x = O.QuantizedTensor(xq, 8, O.SYMMETRIC, O.PER_TOKEN, 0, np.asarray(sa, np.float64),
                          np.zeros(0, np.int32))
    wg = O.QuantizedTensor(wq, 4, O.SYMMETRIC, O.GROUP, g, np.ones((k // g) * n), np.zeros(0, np.int32))
    wc = O.QuantizedTensor(wq, 4, O.SYMMETRIC, O.PER_CHANNEL, k, np.ones(n), np.zeros(0, np.int32))
    for amp in (1, 8, 1024):
        s = O.integerize_scales(wg.scales, amp)
        ri = O.gemm_integer_scale(x, wg, s).output
        rc = O.gemm_coarse(x, wc).output
        assert np.array_equal(ri.view(np.int32), rc.view(np.int32))


def test_dual_quant_scalar_and_identity_inner():
    """test_gemm.cpp:183-226: (5 - 3) * 0.5 = 1 reconstructed weight times activation 1
    gives 1.0f; an identity inner stage (s = 1, z = 0, g = K) over codes in [0, 15]
    reproduces the coarse path bit for bit (mt19937_64 seed 19 draw order)."""
    x = q_act([[1]], [1.0])
    w8 = O.QuantizedTensor(np.array([[5]], np.int16), 8, O.SYMMETRIC, O.PER_CHANNEL, 1,
                           np.array([1.0]), np.zeros(0, np.int32))
    inner = O.DualInnerQuant(np.array([[5]], np.int16), np.array([0.5]), np.array([3], np.int32), 1)
    assert O.gemm_dual_quant(x, w8, inner).output[0, 0] == np.float32(1.0)
    rng = O.Rng(19)
    m, k, n = 3, 8, 3
    xq = (rng.next(m * k) % np.uint64(255)).astype(np.int64).reshape(m, k) - 127
    wq = (rng.next(k * n) % np.uint64(16)).astype(np.int64).reshape(k, n)
    x2 = O.QuantizedTensor(xq.astype(np.int16), 8, O.SYMMETRIC, O.PER_TOKEN, 0,
                           np.full(m, 0.125), np.zeros(0, np.int32))
    outer = O.QuantizedTensor(wq.astype(np.int16), 8, O.SYMMETRIC, O.PER_CHANNEL, k,
                              np.full(n, 0.25), np.zeros(0, np.int32))
    ident = O.DualInnerQuant(wq.astype(np.int16), np.ones(n), np.zeros(n, np.int32), k)
    rd = O.gemm_dual_quant(x2, outer, ident).output
    rc = O.gemm_coarse(x2, outer).output
    assert np.array_equal(rd.view(np.int32), rc.view(np.int32))


def test_dual_inner_quantize_reconstructs_within_half_step():
    """test_gemm.cpp:228-250: inner codes in [0, 15]; groups straddling zero reconstruct
    the outer codes within half an inner step (random_instance seed 20, g = 4)."""
    rng = O.Rng(20)
    _, _, _, wf = random_instance(rng, 1, 16, 6, 16)
    w8 = O.quantize(wf, 8, O.SYMMETRIC, O.PER_CHANNEL, 0)
    inner = O.dual_inner_quantize(w8, 4)
    assert inner.values.shape == (16, 6) and inner.scales.size == 24
    assert inner.values.min() >= 0 and inner.values.max() <= 15
    for j in range(6):
        for t in range(4):
            u = j * 4 + t
            col = w8.values[t * 4:(t + 1) * 4, j]
            if col.min() > 0 or col.max() < 0:
                continue
            for r in range(t * 4, (t + 1) * 4):
                recon = (float(inner.values[r, j]) - float(inner.zero_points[u])) * inner.scales[u]
                assert abs(recon - float(w8.values[r, j])) <= inner.scales[u] / 2
