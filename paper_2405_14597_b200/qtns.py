"""QTNS tensor files + JSON sidecars -> device weights.

Host-side restatement of the reference container (tensor_io.cpp:142-303) and the
quantized-tensor persistence (quantize.cpp:175-270), with the same byte layout,
validation order and error taxonomy:

    "QTNS" | u16 version = 1 | u8 dtype (0 real32, 1 signed8, 2 packed_signed4)
    | u8 ndim (1 or 2) | u64 dims... | payload (little endian)

    <values>.qtns.json: {"bit_width", "scheme", "granularity": {"kind",
    "group_size"}, "scales", "zero_points"}

`load_packed_weight` is the ingestion path of a real checkpoint: the
packed_signed4 payload bytes go to the device untouched and the K2 kernel
(`isb_weight_pack_signed4`) converts the reference nibble order to the tiled
device layout; the sidecar's group scales are integerised on the host (offline,
integer_scale.cpp:40-59) and uploaded with it.
"""
from __future__ import annotations

import json
import struct

import numpy as np

from . import _lib

MAGIC = b"QTNS"
VERSION = 1
REAL32, SIGNED8, PACKED_SIGNED4 = 0, 1, 2
_MAX_DIM = 1 << 32       # tensor_io.cpp:15
_MAX_ELEMENTS = 1 << 40  # tensor_io.cpp:16
_KINDS = {"per_tensor": "per_tensor", "tensor": "per_tensor", "per_token": "per_token",
          "token": "per_token", "per_channel": "per_channel", "channel": "per_channel",
          "group": "group"}  # gran_kind_from_string, quantize.cpp:76-82


class IoError(_lib.IntscaleError):
    """IoError (types.hpp:64-67): the file cannot be opened / read / written."""


def _payload_bytes(dtype, dims):
    n = int(np.prod(dims, dtype=np.uint64))
    return n * 4 if dtype == REAL32 else n if dtype == SIGNED8 else (n + 1) // 2


def encode_header(dtype: int, dims) -> bytes:
    """encode_header, tensor_io.cpp:142-150."""
    return MAGIC + struct.pack("<HBB", VERSION, dtype, len(dims)) + b"".join(
        struct.pack("<Q", int(d)) for d in dims)


def decode_header(buf: bytes, offset: int = 0):
    """decode_header, tensor_io.cpp:152-177 -> (dtype, dims, payload offset)."""
    if len(buf) < offset + 8:
        raise _lib.FormatError("header truncated")
    if buf[offset:offset + 4] != MAGIC:
        raise _lib.FormatError("bad magic, not a QTNS file")
    version, dtype, ndim = struct.unpack_from("<HBB", buf, offset + 4)
    if version != VERSION:
        raise _lib.FormatError(f"unsupported version {version}")
    if dtype > 2:
        raise _lib.FormatError(f"unknown dtype code {dtype}")
    if ndim not in (1, 2):
        raise _lib.FormatError(f"ndim must be 1 or 2, got {ndim}")
    if len(buf) < offset + 8 + 8 * ndim:
        raise _lib.FormatError("header truncated")
    dims, count = [], 1
    for i in range(ndim):
        d = struct.unpack_from("<Q", buf, offset + 8 + 8 * i)[0]
        if d == 0:
            raise _lib.FormatError("zero dimension")
        if d > _MAX_DIM:
            raise _lib.FormatError("dimension too large")
        dims.append(d)
        count *= d
    if count > _MAX_ELEMENTS:
        raise _lib.FormatError("tensor too large")
    return dtype, dims, offset + 8 + 8 * ndim


def _read_file(path) -> bytes:
    try:
        with open(path, "rb") as f:
            return f.read()
    except OSError as e:
        raise IoError(f"cannot open {path}") from e


def _write_file(path, data: bytes):
    try:
        with open(path, "wb") as f:
            f.write(data)
    except OSError as e:
        raise IoError(f"cannot open {path} for writing") from e


def pack_signed4(values) -> bytes:
    """pack_signed4, tensor_io.cpp:179-193 (row-major, even index -> low nibble)."""
    v = np.asarray(values).reshape(-1).astype(np.int64)
    bad = (v < -8) | (v > 7)
    if bad.any():
        raise _lib.ValueError_(f"value {int(v[bad][0])} outside signed 4-bit range")
    nib = (v & 0xF).astype(np.uint8)
    if nib.size % 2:
        nib = np.append(nib, np.uint8(0))
    return (nib[0::2] | (nib[1::2] << 4)).astype(np.uint8).tobytes()


def unpack_signed4(data: bytes, rows: int, cols: int) -> np.ndarray:
    """unpack_signed4, tensor_io.cpp:195-208."""
    n = rows * cols
    if len(data) != (n + 1) // 2:
        raise _lib.LengthError(f"packed payload is {len(data)} bytes, expected {(n + 1) // 2}")
    b = np.frombuffer(data, np.uint8)
    v = np.empty(2 * b.size, np.int16)
    v[0::2] = b & 0xF
    v[1::2] = b >> 4
    v = v[:n]
    v[v >= 8] -= 16
    return v.reshape(rows, cols)


def _shape(dims):
    return (1, int(dims[0])) if len(dims) == 1 else (int(dims[0]), int(dims[1]))


def read_tensor(path):
    """read_tensor, tensor_io.cpp:210-256 -> float32 array, or (bit_width, int16 codes)."""
    buf = _read_file(path)
    dtype, dims, off = decode_header(buf)
    expect = _payload_bytes(dtype, dims)
    if len(buf) - off < expect:
        raise _lib.LengthError(f"payload truncated in {path}")
    if len(buf) - off > expect:
        raise _lib.LengthError(f"trailing bytes after payload in {path}")
    rows, cols = _shape(dims)
    if dtype == REAL32:
        x = np.frombuffer(buf, "<f4", rows * cols, off).astype(np.float32)
        bad = ~np.isfinite(x)
        if bad.any():
            raise _lib.ValueError_(f"non-finite value at element {int(np.argmax(bad))}")
        return x.reshape(rows, cols)
    if dtype == SIGNED8:
        return 8, np.frombuffer(buf, np.int8, rows * cols, off).astype(np.int16).reshape(rows, cols)
    return 4, unpack_signed4(buf[off:], rows, cols)


def write_tensor(x, path, dtype=None):
    """write_tensor, tensor_io.cpp:264-303 (float32 -> real32; codes -> signed8 /
    packed_signed4 as `dtype` says)."""
    x = np.asarray(x)
    if x.ndim != 2 or x.shape[0] < 1 or x.shape[1] < 1:
        raise _lib.ParamError("empty tensor")
    if dtype is None:
        if not np.isfinite(x).all():
            raise _lib.ValueError_("refusing to write non-finite values")
        payload = x.astype("<f4").tobytes()
        dtype = REAL32
    elif dtype == SIGNED8:
        v = x.astype(np.int64)
        bad = (v < -128) | (v > 127)
        if bad.any():
            raise _lib.ValueError_(f"value {int(v[bad][0])} outside signed 8-bit range")
        payload = v.astype(np.int8).tobytes()
    elif dtype == PACKED_SIGNED4:
        payload = pack_signed4(x)
    else:
        raise _lib.ParamError("integer overload cannot write real32")
    _write_file(path, encode_header(dtype, x.shape) + payload)


def write_quantized(codes, bit_width, scheme, kind, group_size, scales, zero_points, path):
    """write_quantized, quantize.cpp:194-220 (values file + `<path>.json` sidecar).
    Asymmetric (unsigned) codes are stored as their two's-complement fold
    (fold_unsigned, quantize.cpp:181-184)."""
    stored = np.asarray(codes).astype(np.int64)
    if scheme == "asymmetric":
        half = 1 << (bit_width - 1)
        stored = np.where(stored >= half, stored - 2 * half, stored)
    write_tensor(stored, path, PACKED_SIGNED4 if bit_width == 4 else SIGNED8)
    side = {"bit_width": int(bit_width), "scheme": scheme,
            "granularity": {"kind": kind, "group_size": int(group_size)},
            "scales": [float(s) for s in np.asarray(scales, np.float64)],
            "zero_points": [int(z) for z in np.asarray(zero_points, np.int64)]}
    try:
        with open(str(path) + ".json", "w") as f:
            f.write(json.dumps(side, indent=2) + "\n")
    except OSError as e:
        raise IoError(f"cannot open {path}.json for writing") from e


def read_quantized(path):
    """read_quantized, quantize.cpp:222-270 -> dict(codes, bit_width, scheme, kind,
    group_size, scales, zero_points). Symmetric payloads only carry signed codes."""
    data = read_tensor(path)
    if not isinstance(data, tuple):
        raise _lib.FormatError(f"{path} holds real values, expected codes")
    bits, codes = data
    try:
        with open(str(path) + ".json") as f:
            side = json.load(f)
    except OSError as e:
        raise IoError(f"cannot open sidecar {path}.json") from e
    except json.JSONDecodeError as e:
        raise _lib.FormatError(f"bad sidecar {path}.json: {e}") from e
    try:
        q = {"bit_width": int(side["bit_width"]), "scheme": str(side["scheme"]),
             "kind": str(side["granularity"]["kind"]),
             "group_size": int(side["granularity"]["group_size"]),
             "scales": np.asarray(side["scales"], np.float64),
             "zero_points": np.asarray(side["zero_points"], np.int32)}
    except (KeyError, TypeError, ValueError) as e:
        raise _lib.FormatError(f"bad sidecar {path}.json: {e}") from e
    if q["scheme"] not in ("symmetric", "asymmetric"):
        raise _lib.ParamError(f"unknown scheme '{q['scheme']}'")
    if q["kind"] not in _KINDS:
        raise _lib.ParamError(f"unknown granularity '{q['kind']}'")
    q["kind"] = _KINDS[q["kind"]]
    if q["bit_width"] not in (4, 8):
        raise _lib.ParamError(f"bit width must be 4 or 8, got {q['bit_width']}")
    if q["bit_width"] != bits:
        raise _lib.FormatError("sidecar bit width disagrees with container dtype")
    if q["scheme"] == "asymmetric":  # unfold_unsigned, quantize.cpp:186-190
        codes = np.where(codes < 0, codes + (1 << q["bit_width"]), codes).astype(np.int16)
    rows, cols = codes.shape
    if q["kind"] == "group" and (q["group_size"] < 1 or rows % q["group_size"]):
        raise _lib.ParamError("group size does not divide the reduction dimension")
    units = {"per_tensor": 1, "per_token": rows, "per_channel": cols,
             "group": cols * (rows // max(q["group_size"], 1))}[q["kind"]]
    if q["scales"].size != units:
        raise _lib.FormatError("sidecar scale count does not match shape")
    if q["scheme"] == "asymmetric" and q["zero_points"].size != q["scales"].size:
        raise _lib.FormatError("sidecar zero point count does not match scale count")
    q["codes"] = codes
    return q


def load_packed_weight(path, amplifier: int | None = None, device="cuda"):
    """A symmetric 4-bit group (or per-channel) weight file -> PackedWeight on the
    device. The nibble payload is uploaded as is and re-laid-out by K2; the integer
    scales are integerize_scales(scales, amplifier) (search_amplifier when None)."""
    import torch

    from . import ops
    buf = _read_file(path)
    dtype, dims, off = decode_header(buf)
    if dtype != PACKED_SIGNED4 or len(dims) != 2:
        raise _lib.FormatError(f"{path}: expected a 2-d packed_signed4 weight")
    if len(buf) - off != _payload_bytes(dtype, dims):
        raise _lib.LengthError(f"payload size mismatch in {path}")
    q = read_quantized(path)  # validates the sidecar against the payload
    if q["scheme"] != "symmetric" or q["kind"] not in ("group", "per_channel"):
        raise _lib.ParamError("weights must be symmetric group or per-channel")
    k, n = int(dims[0]), int(dims[1])
    g = q["group_size"] if q["kind"] == "group" else k
    amp = ops.search_amplifier(q["scales"]) if amplifier is None else int(amplifier)
    s = ops.integerize_scales(q["scales"], amp)
    data = torch.frombuffer(bytearray(buf[off:]), dtype=torch.uint8).to(device)
    return ops.PackedWeight.from_signed4(data, k, n, g, q["scales"], s.int_scales, s.amplifier)
