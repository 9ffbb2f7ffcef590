"""Python host mirror of the reference operator API for the hot path, over the
C ABI (include/intscale_b200.h). Names and argument meaning follow the
reference (proj/include/intscale/*.hpp); tensors are torch CUDA tensors used
purely as device memory. Every compute call runs a CUDA kernel of
libintscale_b200.so — nothing here computes on the CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import (ISB_BF16, ISB_F16, ISB_F32, ISB_I32, ISB_PATH_FLOAT_SCALE,
                   ISB_PATH_INTEGER_SCALE, GemmStats, GroupInfo, GroupProblem, WeightInfo, check,
                   load)

_DT = {torch.float32: ISB_F32, torch.bfloat16: ISB_BF16, torch.float16: ISB_F16,
       torch.int32: ISB_I32}


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _cuda(t, dtype=None):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise _lib.ParamError("expected a CUDA tensor")
    if dtype is not None and t.dtype != dtype:
        raise _lib.ParamError(f"expected dtype {dtype}, got {t.dtype}")
    return t.contiguous()


# ---------------------------------------------------------------------------- K1
def quantize_per_token(x: torch.Tensor, check_finite: bool = False, stream=None, codes=None,
                       scales=None):
    """quantize(x, 8, symmetric, per_token) — quantize.cpp:93-145. Returns
    (codes int8 [M, K], scales float64 [M]); `codes`/`scales` may be preallocated."""
    x = _cuda(x)
    if x.dtype not in (torch.float32, torch.bfloat16):
        raise _lib.ParamError("activations must be float32 or bfloat16")
    if x.dim() != 2:
        raise _lib.ParamError("activations must be 2-d")
    m, k = x.shape
    if codes is None:
        codes = torch.empty((m, k), dtype=torch.int8, device=x.device)
    if scales is None:
        scales = torch.empty((m,), dtype=torch.float64, device=x.device)
    check(load().isb_quantize_per_token(_ptr(x), _DT[x.dtype], m, k, _ptr(codes), _ptr(scales),
                                        int(check_finite), _stream(stream)))
    return codes, scales


def row_absmax(x: torch.Tensor, stream=None, out=None) -> torch.Tensor:
    """Per-row max|x| (float32 [M]) of a (local, K-sharded) activation slice — the
    partial a row-parallel layer all-reduces with MAX before quantizing."""
    x = _cuda(x)
    if x.dtype not in (torch.float32, torch.bfloat16) or x.dim() != 2:
        raise _lib.ParamError("activations must be 2-d float32 or bfloat16")
    m, k = x.shape
    amax = out if out is not None else torch.empty((m,), dtype=torch.float32, device=x.device)
    if amax.dtype != torch.float32 or amax.numel() != m or not amax.is_contiguous():
        raise _lib.ParamError("amax must be a contiguous float32 [M] tensor")
    check(load().isb_row_absmax(_ptr(x), _DT[x.dtype], m, k, _ptr(amax), _stream(stream)))
    return amax


def quantize_per_token_amax(x: torch.Tensor, amax: torch.Tensor, codes=None, scales=None,
                            stream=None):
    """quantize(x, 8, symmetric, per_token) of a K-slice given the FULL-row absmax
    (quantize.cpp:120-125): codes equal the slice of the full-row quantization."""
    x = _cuda(x)
    amax = _cuda(amax, torch.float32)
    if x.dtype not in (torch.float32, torch.bfloat16) or x.dim() != 2:
        raise _lib.ParamError("activations must be 2-d float32 or bfloat16")
    m, k = x.shape
    if amax.numel() != m:
        raise _lib.DimensionError(f"amax has {amax.numel()} rows, activations {m}")
    if codes is None:
        codes = torch.empty((m, k), dtype=torch.int8, device=x.device)
    if scales is None:
        scales = torch.empty((m,), dtype=torch.float64, device=x.device)
    check(load().isb_quantize_per_token_amax(_ptr(x), _DT[x.dtype], m, k, _ptr(amax),
                                             _ptr(codes), _ptr(scales), _stream(stream)))
    return codes, scales


def finalize_acc(acc: torch.Tensor, sa: torch.Tensor, amplifier: int, out_dtype=torch.bfloat16,
                 out=None, stream=None) -> torch.Tensor:
    """Eq. 2 epilogue of an (all-reduced) int32 accumulator (gemm.cpp:252):
    out = float((acc / amplifier) * s_a)."""
    acc = _cuda(acc, torch.int32)
    sa = _cuda(sa, torch.float64)
    m, n = acc.shape
    if out is None:
        out = torch.empty((m, n), dtype=out_dtype, device=acc.device)
    check(load().isb_finalize_acc(_ptr(acc), _ptr(sa), m, n, int(amplifier), _ptr(out),
                                  _DT[out.dtype], _stream(stream)))
    return out


def quantize_weight(w: torch.Tensor, group: int = 128, bit_width: int = 4, stream=None):
    """quantize(w, bits, symmetric, group_of(g)) — quantize.cpp:93-145. Returns
    (codes int16 [K, N], scales float64 [N * K/g], unit n*(K/g)+k/g)."""
    w = _cuda(w, torch.float32)
    k, n = w.shape
    codes = torch.empty((k, n), dtype=torch.int16, device=w.device)
    scales = torch.empty((n * (k // group) if group > 0 and k % group == 0 else 1,),
                         dtype=torch.float64, device=w.device)
    check(load().isb_quantize_weight_groups(_ptr(w), k, n, group, bit_width, _ptr(codes),
                                            _ptr(scales), _stream(stream)))
    return codes, scales


# ---------------------------------------------------------------------------- host helpers
@dataclass
class IntegerScaleSet:
    """integer_scale.hpp:17-21."""
    int_scales: np.ndarray
    amplifier: int
    exponent: int


def search_amplifier_exponent(scales) -> int:
    s = np.ascontiguousarray(np.asarray(scales, np.float64))
    e = C.c_int32()
    check(load().isb_search_amplifier_exponent(s.ctypes.data_as(C.c_void_p), s.size, C.byref(e)))
    return e.value


def search_amplifier(scales) -> int:
    return 1 << search_amplifier_exponent(scales)


def integerize_scales(scales, amplifier: int) -> IntegerScaleSet:
    s = np.ascontiguousarray(np.asarray(scales, np.float64))
    out = np.empty(max(s.size, 1), np.int32)
    e = C.c_int32()
    check(load().isb_integerize_scales(s.ctypes.data_as(C.c_void_p), s.size, int(amplifier),
                                       out.ctypes.data_as(C.c_void_p), C.byref(e)))
    return IntegerScaleSet(out[: s.size], int(amplifier), e.value)


def overflow_analyzer(k: int, group: int, act_bits: int, weight_bits: int, s: IntegerScaleSet):
    ks = np.ascontiguousarray(np.asarray(s.int_scales, np.int32))
    bound, head, safe = C.c_int64(), C.c_double(), C.c_int32()
    check(load().isb_overflow_analyzer(k, group, act_bits, weight_bits,
                                       ks.ctypes.data_as(C.c_void_p), ks.size, C.byref(bound),
                                       C.byref(head), C.byref(safe)))
    return {"static_bound": bound.value, "observed_max": 0, "headroom_bits": head.value,
            "safe": bool(safe.value)}


# ---------------------------------------------------------------------------- K2
class PackedWeight:
    """Device-resident int4 weight in the tiled layout (csrc/layout.cuh) plus its
    group scales and IntegerScaleSet. Owns the C handle."""

    def __init__(self, handle: C.c_void_p, device):
        self._h = handle
        self.device = device
        info = WeightInfo()
        check(load().isb_weight_info(self._h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in WeightInfo._fields_}

    @property
    def handle(self):
        return self._h

    @property
    def k(self):
        return self.info["k"]

    @property
    def n(self):
        return self.info["n"]

    @property
    def group(self):
        return self.info["group"]

    @staticmethod
    def _scales(scales, int_scales, device):
        s = torch.as_tensor(scales, dtype=torch.float64).to(device).contiguous()
        ks = None
        if int_scales is not None:
            ks = torch.as_tensor(np.asarray(int_scales, np.int32) if not isinstance(
                int_scales, torch.Tensor) else int_scales, dtype=torch.int32).to(device).contiguous()
        return s, ks

    @classmethod
    def from_codes(cls, codes: torch.Tensor, group: int, scales, int_scales=None,
                   amplifier: int = 1, stream=None) -> "PackedWeight":
        """Pack reference int16 codes (K x N, row-major)."""
        codes = _cuda(codes, torch.int16)
        k, n = codes.shape
        s, ks = cls._scales(scales, int_scales, codes.device)
        h = C.c_void_p()
        check(load().isb_weight_pack_codes(_ptr(codes), k, n, group, _ptr(s), _ptr(ks),
                                           int(amplifier), _stream(stream), C.byref(h)))
        return cls(h, codes.device)

    @classmethod
    def from_signed4(cls, data: torch.Tensor, k: int, n: int, group: int, scales,
                     int_scales=None, amplifier: int = 1, stream=None) -> "PackedWeight":
        """Pack the reference packed_signed4 byte stream (tensor_io.cpp:179-193)."""
        data = _cuda(data, torch.uint8)
        s, ks = cls._scales(scales, int_scales, data.device)
        h = C.c_void_p()
        check(load().isb_weight_pack_signed4(_ptr(data), data.numel(), k, n, group, _ptr(s),
                                             _ptr(ks), int(amplifier), _stream(stream),
                                             C.byref(h)))
        return cls(h, data.device)

    def unpack_codes(self, stream=None) -> torch.Tensor:
        out = torch.empty((self.k, self.n), dtype=torch.int16, device=self.device)
        check(load().isb_weight_unpack_codes(self._h, _ptr(out), _stream(stream)))
        return out

    def repack_signed4(self, stream=None) -> torch.Tensor:
        out = torch.empty(((self.k * self.n + 1) // 2,), dtype=torch.uint8, device=self.device)
        check(load().isb_weight_repack_signed4(self._h, _ptr(out), _stream(stream)))
        return out

    def close(self):
        if self._h is not None and self._h.value:
            load().isb_weight_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------- workspace
class Workspace:
    """Caller-owned GEMM workspace (tile counters + split partials). Zeroed once;
    the kernels leave it zeroed."""

    def __init__(self, device=None):
        self.device = device
        self.buf = None

    def get(self, nbytes: int, device) -> torch.Tensor:
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = torch.zeros((max(nbytes, 256),), dtype=torch.uint8, device=device)
        return self.buf


_default_ws: dict = {}


def workspace_size(m: int, w: PackedWeight) -> int:
    b = C.c_int64()
    check(load().isb_gemm_workspace_size(m, w.handle, C.byref(b)))
    return b.value


def _ws_for(m, w, workspace):
    need = workspace_size(m, w)
    if workspace is None:
        key = (w.device, torch.cuda.current_stream(w.device).cuda_stream)
        workspace = _default_ws.setdefault(key, Workspace())
    return workspace.get(need, w.device), need


# ---------------------------------------------------------------------------- K3 / K4
def _gemm(path, xq, sa, w: PackedWeight, out_dtype, out, workspace, stream):
    xq = _cuda(xq, torch.int8)
    sa = _cuda(sa, torch.float64)
    m, k = xq.shape
    if out is None:
        out = torch.empty((m, w.n), dtype=out_dtype, device=xq.device)
    ws, need = _ws_for(m, w, workspace)
    fn = load().isb_gemm_integer_scale if path == ISB_PATH_INTEGER_SCALE else \
        load().isb_gemm_float_scale
    check(fn(_ptr(xq), _ptr(sa), m, k, w.handle, _ptr(out), _DT[out.dtype], _ptr(ws), ws.numel(),
             _stream(stream)))
    return out


def gemm_integer_scale(xq, sa, w: PackedWeight, out_dtype=torch.bfloat16, out=None,
                       workspace=None, stream=None):
    """K3 — gemm_integer_scale (gemm.cpp:205-262) on tcgen05. out_dtype=torch.int32
    returns the raw scaled accumulator sum_g P_g k_g (row-parallel TP; see
    finalize_acc)."""
    return _gemm(ISB_PATH_INTEGER_SCALE, xq, sa, w, out_dtype, out, workspace, stream)


def gemm_float_scale(xq, sa, w: PackedWeight, out_dtype=torch.bfloat16, out=None,
                     workspace=None, stream=None):
    """K4 — gemm_float_scale (gemm.cpp:156-203), fp32 I2F+FFMA per group, on tcgen05."""
    return _gemm(ISB_PATH_FLOAT_SCALE, xq, sa, w, out_dtype, out, workspace, stream)


def gemm_coarse(xq, sa, w: PackedWeight, out_dtype=torch.bfloat16, out=None, workspace=None,
                stream=None):
    """gemm_coarse (gemm.hpp:97, gemm.cpp:264-309): per-channel W4A8 (w packed with
    group = K), out = float((double(acc) * s_w[j]) * s_a[i]) — bit-exact."""
    xq = _cuda(xq, torch.int8)
    sa = _cuda(sa, torch.float64)
    m, k = xq.shape
    if out is None:
        out = torch.empty((m, w.n), dtype=out_dtype, device=xq.device)
    ws, _ = _ws_for(m, w, workspace)
    check(load().isb_gemm_coarse(_ptr(xq), _ptr(sa), m, k, w.handle, _ptr(out), _DT[out.dtype],
                                 _ptr(ws), ws.numel(), _stream(stream)))
    return out


def gemm_act_fused(x, w: PackedWeight, path: str = "integer-scale", out_dtype=torch.bfloat16,
                   out=None, sa_out=None, workspace=None, stream=None):
    """K1 (+) K3/K4 in one launch (config C3): float32/bf16 activations in, the
    same output as quantize_per_token + gemm_integer_scale / gemm_float_scale.
    `sa_out` (float64 [M], optional) receives the per-token scales."""
    x = _cuda(x)
    if x.dtype not in (torch.float32, torch.bfloat16) or x.dim() != 2:
        raise _lib.ParamError("activations must be 2-d float32 or bfloat16")
    m, k = x.shape
    if out is None:
        out = torch.empty((m, w.n), dtype=out_dtype, device=x.device)
    if sa_out is not None:
        sa_out = _cuda(sa_out, torch.float64)
    b = C.c_int64()
    check(load().isb_gemm_act_fused_workspace_size(m, w.handle, C.byref(b)))
    if workspace is None:
        key = (w.device, torch.cuda.current_stream(w.device).cuda_stream)
        workspace = _default_ws.setdefault(key, Workspace())
    ws = workspace.get(b.value, w.device)
    p = ISB_PATH_INTEGER_SCALE if path == "integer-scale" else ISB_PATH_FLOAT_SCALE
    check(load().isb_gemm_act_fused(p, _ptr(x), _DT[x.dtype], m, k, w.handle, _ptr(out),
                                    _DT[out.dtype], _ptr(sa_out), _ptr(ws), ws.numel(),
                                    _stream(stream)))
    return out


class GroupedGemm:
    """Grouped layer launch (isb_group_plan_*): up to 8 W4A8 GEMMs — e.g. the
    linears of one decoder layer, or the experts of a MoE layer — in ONE
    persistent tcgen05 launch, per-token activation quantization (K1) included.
    Per problem the output is bit-identical to quantize_per_token followed by
    gemm_integer_scale / gemm_float_scale.

    problems: sequence of dicts with
      weight  PackedWeight (group 128)
      x       float32 / bf16 [M, K] activations (quantized in the launch), or
      xq, sa  int8 codes [M, K] and float64 scales [M] (pre-quantized), and
      out     optional preallocated [M, N] output (else allocated here).
    With `x`, `xq` / `sa` may be given to receive the codes and scales.
    Every pointer is bound at construction: run() replays the launch (CUDA-graph
    safe); keep the tensors alive and update them in place."""

    def __init__(self, problems, path: str = "integer-scale", out_dtype=torch.bfloat16):
        if not 1 <= len(problems) <= 8:
            raise _lib.ParamError("grouped GEMM: 1..8 problems")
        arr = (GroupProblem * len(problems))()
        self.outs, self._keep = [], []
        for i, pr in enumerate(problems):
            w = pr["weight"]
            x, xq, sa = pr.get("x"), pr.get("xq"), pr.get("sa")
            if x is not None:
                x = _cuda(x)
                if x.dtype not in (torch.float32, torch.bfloat16) or x.dim() != 2:
                    raise _lib.ParamError("activations must be 2-d float32 or bfloat16")
                m, k = x.shape
                if xq is not None:
                    xq = _cuda(xq, torch.int8)
                if sa is not None:
                    sa = _cuda(sa, torch.float64)
            else:
                xq, sa = _cuda(xq, torch.int8), _cuda(sa, torch.float64)
                m, k = xq.shape
            if k != w.k:
                raise _lib.DimensionError(f"activation K={k} vs weight rows {w.k}")
            out = pr.get("out")
            if out is None:
                out = torch.empty((m, w.n), dtype=out_dtype, device=w.device)
            elif out.dtype != out_dtype or tuple(out.shape) != (m, w.n):
                raise _lib.ParamError("output tensor shape / dtype mismatch")
            arr[i] = GroupProblem(w.handle.value, m, None if x is None else x.data_ptr(),
                                  _DT[x.dtype] if x is not None else 0,
                                  None if xq is None else xq.data_ptr(),
                                  None if sa is None else sa.data_ptr(), out.data_ptr())
            self.outs.append(out)
            self._keep += [w, x, xq, sa, out]
        self.path = ISB_PATH_INTEGER_SCALE if path == "integer-scale" else ISB_PATH_FLOAT_SCALE
        h = C.c_void_p()
        check(load().isb_group_plan_create(arr, len(problems), self.path, _DT[out_dtype],
                                           C.byref(h)))
        self._h = h
        info = GroupInfo()
        check(load().isb_group_plan_info(h, C.byref(info)))
        self.grid, self.cluster, self.tile_tokens = info.grid, info.cluster, info.tile_tokens
        self.makespan_steps = info.makespan_steps

    def run(self, stream=None):
        check(load().isb_group_run(self._h, _stream(stream)))
        return self.outs

    def nonfinite(self, clear: bool = True) -> bool:
        """Whether any activation quantized by this plan was non-finite (synchronous;
        the reference quantizer's ValueError, quantize.cpp)."""
        r = C.c_int32()
        check(load().isb_group_nonfinite(self._h, 1 if clear else 0, C.byref(r)))
        return bool(r.value)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            load().isb_group_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gemm_checked(path: str, xq, sa, w: PackedWeight, strict=False, want_f64=True, want_acc=True,
                 want_partials=False, stream=None):
    """Checked int64 GEMM with full reference stats semantics. Returns
    (out f32, out_f64, acc int64, partials int64, stats dict)."""
    xq = _cuda(xq, torch.int8)
    sa = _cuda(sa, torch.float64)
    m, k = xq.shape
    dev = xq.device
    p = ISB_PATH_INTEGER_SCALE if path == "integer-scale" else ISB_PATH_FLOAT_SCALE
    out = torch.empty((m, w.n), dtype=torch.float32, device=dev)
    of = torch.empty((m, w.n), dtype=torch.float64, device=dev) if want_f64 else None
    acc = torch.empty((m, w.n), dtype=torch.int64, device=dev) if want_acc and p else None
    part = (torch.empty((m, w.n * (w.k // w.group)), dtype=torch.int64, device=dev)
            if want_partials else None)
    st = GemmStats()
    check(load().isb_gemm_checked(p, _ptr(xq), _ptr(sa), m, k, w.handle, int(strict), _ptr(out),
                                  _ptr(of), _ptr(acc), _ptr(part), C.byref(st), _stream(stream)))
    stats = {f: getattr(st, f) for f, _ in GemmStats._fields_}
    return out, of, acc, part, stats


class DualInner:
    """Device DualInnerQuant (gemm.hpp:22-27): codes K x N int16 in [0, 15], double
    scales and int32 zero points per unit j*G + t, group size."""

    def __init__(self, codes, scales, zero_points, group):
        self.codes, self.scales, self.zero_points, self.group = codes, scales, zero_points, group


def dual_inner_quantize(w8_codes: torch.Tensor, group: int, stream=None) -> DualInner:
    """dual_inner_quantize (gemm.cpp:311-345) on the device: 8-bit per-channel codes
    (K x N) -> asymmetric 4-bit group codes + scales + zero points."""
    w8 = _cuda(w8_codes, torch.int16)
    k, n = w8.shape
    if group < 1 or k % group:
        raise _lib.ParamError("group size must divide the reduction dimension")
    units = n * (k // group)
    codes = torch.empty((k, n), dtype=torch.int16, device=w8.device)
    scales = torch.empty((units,), dtype=torch.float64, device=w8.device)
    zps = torch.empty((units,), dtype=torch.int32, device=w8.device)
    check(load().isb_dual_inner_quantize(_ptr(w8), k, n, group, _ptr(codes), _ptr(scales),
                                         _ptr(zps), _stream(stream)))
    return DualInner(codes, scales, zps, group)


def gemm_dual_quant(xq, sa, inner: DualInner, outer_scales, want_f64=False, stream=None):
    """gemm_dual_quant (gemm.cpp:347-412): the QServe-style comparison path, bit-exact
    float32 output (and the double value when want_f64)."""
    xq = _cuda(xq, torch.int8)
    sa = _cuda(sa, torch.float64)
    so = torch.as_tensor(np.asarray(outer_scales, np.float64) if not isinstance(
        outer_scales, torch.Tensor) else outer_scales, dtype=torch.float64).to(xq.device).contiguous()
    m, k = xq.shape
    n = inner.codes.shape[1]
    if inner.codes.shape[0] != k:
        raise _lib.DimensionError(f"activation K={k} vs weight rows {inner.codes.shape[0]}")
    out = torch.empty((m, n), dtype=torch.float32, device=xq.device)
    of = torch.empty((m, n), dtype=torch.float64, device=xq.device) if want_f64 else None
    check(load().isb_gemm_dual_quant(_ptr(xq), _ptr(sa), m, k, _ptr(inner.codes),
                                     _ptr(inner.scales), _ptr(inner.zero_points), inner.group,
                                     _ptr(so), n, _ptr(out), _ptr(of), _stream(stream)))
    return (out, of) if want_f64 else out


def gemm_dense(x: torch.Tensor, w: torch.Tensor, out_dtype=None, out=None, stream=None):
    """Dense fp16/bf16 baseline (no cuBLAS): x[M][K] @ w[N][K]^T on tcgen05 kind::f16
    with fp32 accumulation (isb_gemm_dense) — the FP16 comparator of the paper's
    W4A8 speed-up claims. Same semantics as torch.nn.functional.linear(x, w)."""
    if x.dtype != w.dtype or x.dtype not in (torch.float16, torch.bfloat16):
        raise _lib.ParamError("dense operands must both be fp16 or bf16")
    x = _cuda(x)
    w = _cuda(w)
    m, k = x.shape
    n, k2 = w.shape
    if k2 != k:
        raise _lib.DimensionError(f"activation K={k} vs weight K={k2}")
    if out is None:
        out = torch.empty((m, n), dtype=out_dtype or x.dtype, device=x.device)
    check(load().isb_gemm_dense(_ptr(x), _ptr(w), _DT[x.dtype], m, n, k, _ptr(out),
                                _DT[out.dtype], _stream(stream)))
    return out


def launch_count() -> int:
    return load().isb_launch_count()
