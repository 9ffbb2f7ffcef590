"""Fixture builders shared by the oracle and GPU parity tests. They replay the
reference tests' own construction (draw order included) on the oracle's
std::mt19937_64 stream."""
import numpy as np

from oracle import oracle as O


def random_instance(rng: "O.Rng", m, k, n, g):
    """random_instance, test_gemm.cpp:76-90."""
    xf = (4.0 * rng.u01(m * k) - 2.0).astype(np.float32).reshape(m, k)
    mag = O.exp2(-8.0 + 8.0 * rng.u01())
    wf = ((2.0 * rng.u01(k * n) - 1.0) * mag).astype(np.float32).reshape(k, n)
    return O.quantize_per_token(xf), O.quantize(wf, 4, O.SYMMETRIC, O.GROUP, g), xf, wf


def make_x(rng: "O.Rng", m, k, scales):
    """make_x, acceptance.cpp:42-54: codes in [-127, 127]."""
    v = (rng.below(255, m * k) - 127).astype(np.int16).reshape(m, k)
    return O.QuantizedTensor(v, 8, O.SYMMETRIC, O.PER_TOKEN, 0, np.asarray(scales, np.float64),
                             np.zeros(0, np.int32))


def make_w(rng: "O.Rng", k, n, g, scales):
    """make_w, acceptance.cpp:56-67: codes in [-8, 7]."""
    v = (rng.below(16, k * n) - 8).astype(np.int16).reshape(k, n)
    return O.QuantizedTensor(v, 4, O.SYMMETRIC, O.GROUP, g, np.asarray(scales, np.float64),
                             np.zeros(0, np.int32))


def overflow_rig(n=2):
    """OverflowRig, test_gemm.cpp:345-355: K=4096 of 127 against -8.0 weights."""
    x = O.quantize_per_token(np.full((1, 4096), 127.0, np.float32))
    w = O.quantize_weight(np.full((4096, n), -8.0, np.float32), 128)
    s = O.integerize_scales(w.scales, 1024)
    return x, w, s


def llama_problem(m, k, n, seed_w=42, seed_x=43, g=128, amp=1024):
    """The measurement fixture of SURVEY §8d: W = llama_like(K, N, 42) group-4bit,
    X = gaussian(M, K, 43) per-token 8-bit, alpha = 1024."""
    wf = O.generate_llama_like(k, n, seed_w)
    xf = O.generate_gaussian(m, k, 1.0, seed_x)
    w = O.quantize_weight(wf, g)
    x = O.quantize_per_token(xf)
    s = O.integerize_scales(w.scales, amp)
    return x, w, s, xf, wf
