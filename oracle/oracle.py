"""ORACLE — TEST INFRASTRUCTURE ONLY.

numpy/ctypes front end of ``oracle/oracle.cpp``, the CPU restatement of the
reference integer-scale path (/root/reference/proj). Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline and ``--impl
reference``) may import this module; the product package never does.

Parity pin: golden vectors from the reference's own tests, transcribed in
``tests/test_oracle_golden.py`` (the reference itself cannot be built here —
it needs Eigen3, absent from the image).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")

# Status codes shared with include/intscale_b200.h (types.hpp:29-67 taxonomy).
OK, PARAM, DIMENSION, VALUE, OVERFLOW, LENGTH, FORMAT, ERROR = range(8)
STATUS_NAMES = {
    PARAM: "ParamError", DIMENSION: "DimensionError", VALUE: "ValueError",
    OVERFLOW: "OverflowError", LENGTH: "LengthError", FORMAT: "FormatError", ERROR: "Error",
}

PER_TENSOR, PER_TOKEN, PER_CHANNEL, GROUP = range(4)
SYMMETRIC, ASYMMETRIC = 0, 1


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


class OrStats(C.Structure):
    _fields_ = [
        ("int_to_float_conversions", C.c_int64),
        ("integer_multiply_adds", C.c_int64),
        ("max_abs_accumulator", C.c_int64),
        ("overflow_detected", C.c_int32),
        ("fallback_applied", C.c_int32),
        ("overflow_i", C.c_int64),
        ("overflow_j", C.c_int64),
        ("wall_ms", C.c_double),
    ]


class OrReport(C.Structure):
    _fields_ = [
        ("static_bound", C.c_int64),
        ("observed_max", C.c_int64),
        ("headroom_bits", C.c_double),
        ("safe", C.c_int32),
    ]


_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.or_last_error.restype = C.c_char_p
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(rc: int):
    if rc != OK:
        raise OracleError(rc, lib().or_last_error().decode())


# --------------------------------------------------------------------------- generators
def generate_gaussian(rows, cols, sigma=1.0, seed=0):
    out = np.empty((rows, cols) if rows > 0 and cols > 0 else (1, 1), np.float32)
    _check(lib().or_generate(0, C.c_int64(rows), C.c_int64(cols), C.c_double(sigma),
                             C.c_double(0.0), C.c_uint64(seed), _p(out)))
    return out


def generate_uniform(rows, cols, lo=-1.0, hi=1.0, seed=0):
    out = np.empty((max(rows, 1), max(cols, 1)), np.float32)
    _check(lib().or_generate(1, C.c_int64(rows), C.c_int64(cols), C.c_double(lo),
                             C.c_double(hi), C.c_uint64(seed), _p(out)))
    return out


def generate_llama_like(rows, cols, seed=0):
    out = np.empty((max(rows, 1), max(cols, 1)), np.float32)
    _check(lib().or_generate(2, C.c_int64(rows), C.c_int64(cols), C.c_double(0.0),
                             C.c_double(0.0), C.c_uint64(seed), _p(out)))
    return out


# --------------------------------------------------------------------------- quantizer
@dataclass
class QuantizedTensor:
    values: np.ndarray          # int16 codes, rows x cols (types.hpp:21)
    bit_width: int
    scheme: int
    kind: int
    group: int
    scales: np.ndarray          # float64 per unit (quantize.hpp:49-51)
    zero_points: np.ndarray     # int32 per unit (asymmetric) or empty

    @property
    def rows(self):
        return self.values.shape[0]

    @property
    def cols(self):
        return self.values.shape[1]


def unit_count(kind, group, rows, cols):
    out = C.c_int64()
    _check(lib().or_unit_count(kind, C.c_int64(group), C.c_int64(rows), C.c_int64(cols),
                               C.byref(out)))
    return out.value


def quantize(x, bit_width, scheme=SYMMETRIC, kind=GROUP, group=128) -> QuantizedTensor:
    x = np.ascontiguousarray(x, np.float32)
    rows, cols = x.shape
    units = unit_count(kind, group, rows, cols) if rows > 0 and cols > 0 else 1
    codes = np.empty((rows, cols), np.int16)
    scales = np.empty(units, np.float64)
    zps = np.zeros(units if scheme == ASYMMETRIC else 1, np.int32)
    _check(lib().or_quantize(_p(x), C.c_int64(rows), C.c_int64(cols), bit_width, scheme, kind,
                             C.c_int64(group), _p(codes), _p(scales), _p(zps)))
    return QuantizedTensor(codes, bit_width, scheme, kind, group if kind == GROUP else 0, scales,
                           zps if scheme == ASYMMETRIC else np.zeros(0, np.int32))


def quantize_per_token(x):
    return quantize(x, 8, SYMMETRIC, PER_TOKEN, 0)


def quantize_weight(w, group=128):
    return quantize(w, 4, SYMMETRIC, GROUP, group)


# --------------------------------------------------------------------------- integer scale
@dataclass
class IntegerScaleSet:
    int_scales: np.ndarray
    amplifier: int
    exponent: int


def search_amplifier_exponent(scales):
    s = np.ascontiguousarray(scales, np.float64)
    e = C.c_int()
    _check(lib().or_search_amplifier_exponent(_p(s), C.c_int64(s.size), C.byref(e)))
    return e.value


def search_amplifier(scales):
    return 1 << search_amplifier_exponent(scales)


def integerize_scales(scales, amplifier) -> IntegerScaleSet:
    s = np.ascontiguousarray(scales, np.float64)
    out = np.empty(max(s.size, 1), np.int32)
    e = C.c_int()
    _check(lib().or_integerize_scales(_p(s), C.c_int64(s.size), C.c_int64(amplifier), _p(out),
                                      C.byref(e)))
    return IntegerScaleSet(out[: s.size], int(amplifier), e.value)


# --------------------------------------------------------------------------- nibble packing
def pack_signed4(values):
    v = np.ascontiguousarray(values, np.int16).reshape(-1)
    out = np.empty((v.size + 1) // 2, np.uint8)
    _check(lib().or_pack_signed4(_p(v), C.c_int64(v.size), _p(out)))
    return out


def unpack_signed4(data, rows, cols):
    b = np.ascontiguousarray(np.frombuffer(bytes(data), np.uint8))
    out = np.empty((rows, cols), np.int16)
    _check(lib().or_unpack_signed4(_p(b), C.c_int64(b.size), C.c_int64(rows), C.c_int64(cols),
                                   _p(out)))
    return out


# --------------------------------------------------------------------------- GEMM paths
@dataclass
class GemmResult:
    output: np.ndarray                 # float32 M x N
    stats: dict
    output_f64: np.ndarray | None = None
    acc: np.ndarray | None = None      # int64 scaled accumulator (integer path)
    partials: np.ndarray | None = None  # int64 signed P_g, M x (N*G)


def _stats_dict(st: OrStats):
    return {f: getattr(st, f) for f, _ in OrStats._fields_}


def gemm_integer_scale(x: QuantizedTensor, w: QuantizedTensor, s: IntegerScaleSet, strict=False,
                       workers=1, record=True) -> GemmResult:
    m, k = x.values.shape
    kw, n = w.values.shape
    g = w.group if w.kind == GROUP else kw
    groups = kw // g if g and kw % g == 0 else 1
    out = np.empty((m, n), np.float32)
    of = np.empty((m, n), np.float64) if record else None
    acc = np.empty((m, n), np.int64) if record else None
    part = np.empty((m, n * groups), np.int64) if record else None
    st = OrStats()
    xv = np.ascontiguousarray(x.values, np.int16)
    wv = np.ascontiguousarray(w.values, np.int16)
    ks = np.ascontiguousarray(s.int_scales, np.int32)
    _check(lib().or_gemm_integer_scale(
        x.bit_width, x.scheme, x.kind, w.scheme, _p(xv), _p(np.ascontiguousarray(x.scales, np.float64)), C.c_int64(m), C.c_int64(k),
        C.c_int64(x.scales.size), _p(wv), C.c_int64(kw), C.c_int64(n), w.bit_width, w.kind,
        C.c_int64(w.group), _p(np.ascontiguousarray(w.scales, np.float64)),
        C.c_int64(w.scales.size), _p(ks), C.c_int64(ks.size), C.c_int64(s.amplifier),
        s.exponent, int(strict), workers, _p(out), _p(of), _p(acc), _p(part), C.byref(st)))
    return GemmResult(out, _stats_dict(st), of, acc, part)


def gemm_float_scale(x: QuantizedTensor, w: QuantizedTensor, strict=False, workers=1,
                     record=True) -> GemmResult:
    m, k = x.values.shape
    kw, n = w.values.shape
    g = w.group if w.kind == GROUP else kw
    groups = kw // g if g and kw % g == 0 else 1
    out = np.empty((m, n), np.float32)
    of = np.empty((m, n), np.float64) if record else None
    part = np.empty((m, n * groups), np.int64) if record else None
    st = OrStats()
    _check(lib().or_gemm_float_scale(
        x.bit_width, x.scheme, x.kind, w.scheme, _p(np.ascontiguousarray(x.values, np.int16)),
        _p(np.ascontiguousarray(x.scales, np.float64)), C.c_int64(m), C.c_int64(k),
        C.c_int64(x.scales.size), _p(np.ascontiguousarray(w.values, np.int16)), C.c_int64(kw),
        C.c_int64(n), w.bit_width, w.kind, C.c_int64(w.group),
        _p(np.ascontiguousarray(w.scales, np.float64)), C.c_int64(w.scales.size), int(strict),
        workers, _p(out), _p(of), _p(part), C.byref(st)))
    return GemmResult(out, _stats_dict(st), of, None, part)


def gemm_coarse(x: QuantizedTensor, w: QuantizedTensor, workers=1) -> "GemmResult":
    """gemm_coarse, gemm.cpp:264-309: per-channel weights only (:267-268);
    out = float(double(acc) * s_w[j] * s_a[i]) — the same double expression, in the
    same order, as the float-scale path with a single group per channel
    (gemm.cpp:190-194), which this restatement therefore shares."""
    if w.kind != PER_CHANNEL:
        raise OracleError(PARAM, "coarse path requires per-channel weights")
    return gemm_float_scale(x, w, workers=workers)


class DualInnerQuant:
    """DualInnerQuant, gemm.hpp:22-27: codes K x N in [0, 15], scales / zero points per
    unit j*G + t, group size."""

    def __init__(self, values, scales, zero_points, group):
        self.values, self.scales, self.zero_points, self.group = values, scales, zero_points, group


def dual_inner_quantize(w8: QuantizedTensor, group: int) -> DualInnerQuant:
    """dual_inner_quantize, gemm.cpp:311-345 (8-bit per-channel symmetric outer weight)."""
    if w8.bit_width != 8 or w8.scheme != SYMMETRIC or w8.kind != PER_CHANNEL:
        raise OracleError(PARAM, "dual quantization layers over an 8-bit per-channel symmetric weight")
    k, n = w8.values.shape
    g = int(group)
    units = (k // g) * n if g >= 1 else 1
    codes = np.empty((k, n), np.int16)
    scales = np.empty(max(units, 1), np.float64)
    zps = np.empty(max(units, 1), np.int32)
    _check(lib().or_dual_inner_quantize(_p(np.ascontiguousarray(w8.values, np.int16)), C.c_int64(k),
                                        C.c_int64(n), C.c_int64(g), _p(codes), _p(scales), _p(zps)))
    return DualInnerQuant(codes, scales[:units], zps[:units], g)


def gemm_dual_quant(x: QuantizedTensor, w8: QuantizedTensor, inner: DualInnerQuant) -> GemmResult:
    """gemm_dual_quant, gemm.cpp:347-412: output float32 and the double pre-rounding value."""
    m, k = x.values.shape
    n = w8.values.shape[1]
    out = np.empty((m, n), np.float32)
    of = np.empty((m, n), np.float64)
    _check(lib().or_gemm_dual_quant(
        _p(np.ascontiguousarray(x.values, np.int16)), _p(np.ascontiguousarray(x.scales, np.float64)),
        C.c_int64(m), C.c_int64(k), _p(np.ascontiguousarray(inner.values, np.int16)),
        _p(np.ascontiguousarray(inner.scales, np.float64)),
        _p(np.ascontiguousarray(inner.zero_points, np.int32)), C.c_int64(inner.group),
        _p(np.ascontiguousarray(w8.scales, np.float64)), C.c_int64(n), _p(out), _p(of)))
    return GemmResult(out, {}, of, None, None)


def gemm_oracle(path: str, x: QuantizedTensor, w: QuantizedTensor, amplifier=1):
    m, k = x.values.shape
    kw, n = w.values.shape
    out = np.empty((m, n), np.float32)
    _check(lib().or_gemm_oracle(
        1 if path == "integer-scale" else 0, x.bit_width, x.scheme, x.kind, w.scheme, _p(np.ascontiguousarray(x.values, np.int16)),
        _p(np.ascontiguousarray(x.scales, np.float64)), C.c_int64(m), C.c_int64(k),
        C.c_int64(x.scales.size), _p(np.ascontiguousarray(w.values, np.int16)), C.c_int64(kw),
        C.c_int64(n), w.bit_width, w.kind, C.c_int64(w.group),
        _p(np.ascontiguousarray(w.scales, np.float64)), C.c_int64(w.scales.size),
        C.c_int64(amplifier), _p(out)))
    return out


def overflow_analyzer(k, group, act_bits, w_bits, s: IntegerScaleSet):
    ks = np.ascontiguousarray(s.int_scales, np.int32)
    r = OrReport()
    _check(lib().or_overflow_analyzer(C.c_int64(k), C.c_int64(group), act_bits, w_bits, _p(ks),
                                      C.c_int64(ks.size), C.byref(r)))
    return {f: getattr(r, f) for f, _ in OrReport._fields_}


def run_layer(x, w, path: str, s: IntegerScaleSet | None = None, fallback=False, strict=False,
              workers=1) -> GemmResult:
    """gemm.cpp:489-516 (float/integer paths)."""
    if path == "float-scale":
        return gemm_float_scale(x, w, strict, workers)
    if s is None:
        raise OracleError(PARAM, "integer-scale path needs an IntegerScaleSet")
    if fallback:
        g = w.group if w.kind == GROUP else w.rows
        rep = overflow_analyzer(x.cols, g, x.bit_width, w.bit_width, s)
        if not rep["safe"]:
            r = gemm_float_scale(x, w, strict, workers)
            r.stats["fallback_applied"] = 1
            return r
    return gemm_integer_scale(x, w, s, strict, workers)


def expected_counters(path: str, m, n, k, g):
    p = {"float-scale": 0, "integer-scale": 1, "coarse": 2, "dual-quant": 3}[path]
    conv, imads = C.c_int64(), C.c_int64()
    lib().or_expected_counters(p, C.c_int64(m), C.c_int64(n), C.c_int64(k), C.c_int64(g),
                               C.byref(conv), C.byref(imads))
    return conv.value, imads.value


def ulp_distance(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Float32 ULP distance (test_gemm.cpp:22-29)."""
    def key(x):
        u = np.ascontiguousarray(x, np.float32).view(np.int32).astype(np.int64)
        return np.where(u < 0, np.int64(-(2 ** 31)) - u, u)
    d = np.abs(key(a) - key(b))
    return np.where(np.asarray(a, np.float32) == np.asarray(b, np.float32), 0, d)


class Rng:
    """std::mt19937_64 replay (acceptance.cpp:34-39 ``Rng``)."""

    def __init__(self, seed: int):
        L = lib()
        L.or_rng_new.restype = C.c_void_p
        self._h = C.c_void_p(L.or_rng_new(C.c_uint64(seed)))

    def __del__(self):
        try:
            lib().or_rng_free(self._h)
        except Exception:
            pass

    def next(self, n: int = 1) -> np.ndarray:
        out = np.empty(n, np.uint64)
        lib().or_rng_next(self._h, C.c_int64(n), _p(out))
        return out

    def u01(self, n: int | None = None):
        v = (self.next(1 if n is None else n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        return float(v[0]) if n is None else v

    def below(self, bound: int, n: int | None = None):
        v = self.next(1 if n is None else n) % np.uint64(bound)
        return int(v[0]) if n is None else v.astype(np.int64)


def exp2(x: float) -> float:
    """std::exp2 from the same libm the reference links (tensor_io.cpp:113)."""
    f = lib().or_exp2
    f.restype = C.c_double
    f.argtypes = [C.c_double]
    return f(x)
