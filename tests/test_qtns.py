"""QTNS container + JSON sidecar: the reference's tensor I/O
cases (test_tensor_io.cpp:64-226) and quantized persistence cases
(test_quantize.cpp:284-328) against paper_2405_14597_b200.qtns, plus the device
ingestion path (payload bytes -> K2 packer -> K3) against the oracle."""
import json
import struct

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2405_14597_b200 import _lib
from paper_2405_14597_b200 import qtns as Q


def header_bytes(dtype, rows, cols):
    """24-byte header for a 2-d tensor (test_tensor_io.cpp:46-53)."""
    return bytes([ord("Q"), ord("T"), ord("N"), ord("S"), 1, 0, dtype, 2]) + struct.pack(
        "<QQ", rows, cols)


def rowq(vals):
    return np.asarray([vals], np.int16)


# --------------------------------------------------------------- nibble packing
def test_nibble_packing_pins_reference_bytes():
    assert Q.pack_signed4(rowq([-8, 7])) == bytes([0x78])
    assert np.array_equal(Q.unpack_signed4(bytes([0x78]), 1, 2), rowq([-8, 7]))
    assert Q.pack_signed4(rowq([3])) == bytes([0x03])
    assert Q.pack_signed4(rowq([-1])) == bytes([0x0F])
    assert np.array_equal(Q.unpack_signed4(bytes([0x0F]), 1, 1), rowq([-1]))
    v8 = rowq([-8, -1, 0, 1, 2, -2, 7, -7])
    assert Q.pack_signed4(v8) == bytes([0xF8, 0x10, 0xE2, 0x97])
    assert np.array_equal(Q.unpack_signed4(bytes([0xF8, 0x10, 0xE2, 0x97]), 1, 8), v8)
    with pytest.raises(_lib.ValueError_):
        Q.pack_signed4(rowq([8]))
    with pytest.raises(_lib.ValueError_):
        Q.pack_signed4(rowq([-9]))
    with pytest.raises(_lib.LengthError):
        Q.unpack_signed4(bytes([0xF8]), 1, 3)


def test_nibble_packing_matches_oracle_on_random_codes():
    rng = np.random.default_rng(3)
    for rows, cols in [(1, 1), (3, 5), (128, 7), (256, 64)]:
        v = rng.integers(-8, 8, size=(rows, cols)).astype(np.int16)
        assert Q.pack_signed4(v) == bytes(O.pack_signed4(v))
        assert np.array_equal(Q.unpack_signed4(Q.pack_signed4(v), rows, cols), v)


# --------------------------------------------------------------- containers
def test_float_file_pins_header_layout(tmp_path):
    Q.write_tensor(np.zeros((1, 1), np.float32), tmp_path / "z.qtns")
    assert (tmp_path / "z.qtns").read_bytes() == header_bytes(0, 1, 1) + bytes(4)


def test_float_tensors_round_trip_bit_exactly(tmp_path):
    x = np.array([[0.0, -1.5, 3.25e-3], [1.0e30, -1.0e-30, 127.0]], np.float32)
    Q.write_tensor(x, tmp_path / "x.qtns")
    back = Q.read_tensor(tmp_path / "x.qtns")
    assert back.shape == (2, 3)
    assert np.array_equal(back.view(np.int32), x.view(np.int32))


def test_integer_payloads_round_trip_with_sign(tmp_path):
    q = np.array([[-128, 127], [0, -1]], np.int16)
    Q.write_tensor(q, tmp_path / "q.qtns", Q.SIGNED8)
    bits, back = Q.read_tensor(tmp_path / "q.qtns")
    assert bits == 8 and np.array_equal(back, q)
    q4 = rowq([-8, 7, -1])
    Q.write_tensor(q4, tmp_path / "q4.qtns", Q.PACKED_SIGNED4)
    bits, back4 = Q.read_tensor(tmp_path / "q4.qtns")
    assert bits == 4 and np.array_equal(back4, q4)
    assert (tmp_path / "q4.qtns").stat().st_size == 26  # 24-byte header + ceil(3/2)


def test_one_dimensional_file_is_a_single_row(tmp_path):
    b = bytes([ord("Q"), ord("T"), ord("N"), ord("S"), 1, 0, 1, 1, 5, 0, 0, 0, 0, 0, 0, 0])
    (tmp_path / "v.qtns").write_bytes(b + bytes([0x80, 0xFF, 0x00, 0x01, 0x7F]))
    bits, v = Q.read_tensor(tmp_path / "v.qtns")
    assert v.shape == (1, 5)
    assert list(v[0]) == [-128, -1, 0, 1, 127]


GOOD = header_bytes(0, 1, 1) + bytes(4)


def _patch(i, val):
    b = bytearray(GOOD)
    b[i] = val
    return bytes(b)


@pytest.mark.parametrize("data,err", [
    (_patch(0, ord("X")), _lib.FormatError),             # bad magic
    (_patch(4, 2), _lib.FormatError),                    # unsupported version
    (_patch(6, 3), _lib.FormatError),                    # unknown dtype
    (_patch(7, 3), _lib.FormatError),                    # bad rank
    (header_bytes(0, 0, 1), _lib.FormatError),           # zero dimension
    (GOOD[:-1], _lib.LengthError),                       # truncated payload
    (GOOD[:10], _lib.FormatError),                       # truncated header
    (GOOD + b"\0", _lib.LengthError),                    # trailing bytes
    (header_bytes(0, 1, 1) + bytes([0, 0, 0xC0, 0x7F]), _lib.ValueError_),  # NaN payload
    (header_bytes(0, (1 << 32) + 1, 1), _lib.FormatError),  # dimension above kMaxDim
    (header_bytes(1, 1 << 21, 1 << 20), _lib.FormatError),  # 2^41 elements > kMaxElements
], ids=["magic", "version", "dtype", "rank", "zero-dim", "short-payload", "short-header",
        "trailing", "nan", "max-dim", "max-elements"])
def test_malformed_files_raise_matching_error(tmp_path, data, err):
    (tmp_path / "bad.qtns").write_bytes(data)
    with pytest.raises(err):
        Q.read_tensor(tmp_path / "bad.qtns")


def test_missing_file_is_io_error(tmp_path):
    with pytest.raises(Q.IoError):
        Q.read_tensor(tmp_path / "absent.qtns")


def test_writers_reject_unrepresentable_values(tmp_path):
    with pytest.raises(_lib.ValueError_):
        Q.write_tensor(np.full((1, 1), np.nan, np.float32), tmp_path / "nan.qtns")
    with pytest.raises(_lib.ValueError_):
        Q.write_tensor(np.full((1, 1), 200), tmp_path / "big.qtns", Q.SIGNED8)
    with pytest.raises(_lib.ValueError_):
        Q.write_tensor(np.full((1, 1), 8), tmp_path / "big4.qtns", Q.PACKED_SIGNED4)
    with pytest.raises(_lib.ParamError):
        Q.write_tensor(np.full((1, 1), 1), tmp_path / "real.qtns", Q.REAL32)


# --------------------------------------------------------------- sidecars
def _persist_x():
    """test_quantize.cpp:284-291: x(128, 4) = 2*u01 - 1 from mt19937_64(9)."""
    rng = O.Rng(9)
    return (2.0 * rng.u01(128 * 4) - 1.0).astype(np.float32).reshape(128, 4)


def _write(q, path):
    names = {O.PER_TENSOR: "per_tensor", O.PER_TOKEN: "per_token",
             O.PER_CHANNEL: "per_channel", O.GROUP: "group"}
    Q.write_quantized(q.values, q.bit_width,
                      "asymmetric" if q.scheme == O.ASYMMETRIC else "symmetric",
                      names[q.kind], q.group, q.scales, q.zero_points, path)


def test_symmetric_group_round_trips_with_sidecar(tmp_path):
    q = O.quantize(_persist_x(), 4, O.SYMMETRIC, O.GROUP, 32)
    _write(q, tmp_path / "w.qtns")
    assert (tmp_path / "w.qtns.json").exists()
    assert (tmp_path / "w.qtns").stat().st_size == 24 + 256
    side = json.loads((tmp_path / "w.qtns.json").read_text())
    assert list(side) == ["bit_width", "scheme", "granularity", "scales", "zero_points"]
    back = Q.read_quantized(tmp_path / "w.qtns")
    assert np.array_equal(back["codes"], q.values)
    assert back["bit_width"] == 4 and back["scheme"] == "symmetric"
    assert back["kind"] == "group" and back["group_size"] == 32
    assert np.array_equal(back["scales"], q.scales)


@pytest.mark.parametrize("bits,kind", [(4, O.PER_TOKEN), (8, O.PER_CHANNEL)])
def test_asymmetric_codes_survive_signed_container(tmp_path, bits, kind):
    q = O.quantize(_persist_x(), bits, O.ASYMMETRIC, kind, 0)
    assert q.values.min() >= 0
    if bits == 8:
        assert q.values.max() >= 128
    _write(q, tmp_path / "a.qtns")
    back = Q.read_quantized(tmp_path / "a.qtns")
    assert np.array_equal(back["codes"], q.values)
    assert np.array_equal(back["zero_points"], q.zero_points)
    assert np.array_equal(back["scales"], q.scales)


def test_bad_sidecars(tmp_path):
    q = O.quantize(_persist_x(), 4, O.SYMMETRIC, O.GROUP, 32)
    p = tmp_path / "w.qtns"
    _write(q, p)
    side = json.loads((tmp_path / "w.qtns.json").read_text())

    def put(d):
        (tmp_path / "w.qtns.json").write_text(json.dumps(d))

    put({**side, "bit_width": 8})
    with pytest.raises(_lib.FormatError):      # disagrees with the container dtype
        Q.read_quantized(p)
    put({**side, "scales": side["scales"][:-1]})
    with pytest.raises(_lib.FormatError):      # scale count
        Q.read_quantized(p)
    put({k: v for k, v in side.items() if k != "scales"})
    with pytest.raises(_lib.FormatError):      # missing key
        Q.read_quantized(p)
    put({**side, "scheme": "skewed"})
    with pytest.raises(_lib.ParamError):
        Q.read_quantized(p)
    put({**side, "granularity": {"kind": "group", "group_size": 48}})
    with pytest.raises(_lib.ParamError):      # 48 does not divide 128
        Q.read_quantized(p)
    (tmp_path / "w.qtns.json").write_text("{not json")
    with pytest.raises(_lib.FormatError):
        Q.read_quantized(p)
    (tmp_path / "w.qtns.json").unlink()
    with pytest.raises(Q.IoError):
        Q.read_quantized(p)
    Q.write_tensor(np.zeros((2, 2), np.float32), tmp_path / "f.qtns")
    with pytest.raises(_lib.FormatError):      # real values, expected codes
        Q.read_quantized(tmp_path / "f.qtns")


# --------------------------------------------------------------- device ingestion
@pytest.mark.gpu
@pytest.mark.parametrize("m,k,n", [(1, 4096, 512), (16, 11008, 384), (200, 4096, 256)])
def test_qtns_weight_to_device_gemm_bit_exact(tmp_path, m, k, n):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2405_14597_b200 as isb
    from tests.instances import llama_problem
    x, w, s, _, _ = llama_problem(m, k, n, seed_w=61 + n, seed_x=67 + m)
    _write(w, tmp_path / "w.qtns")
    pw = Q.load_packed_weight(tmp_path / "w.qtns", amplifier=1024)
    assert torch.equal(pw.unpack_codes().cpu(), torch.from_numpy(w.values))
    assert bytes(pw.repack_signed4().cpu().numpy()) == (tmp_path / "w.qtns").read_bytes()[24:]
    ref = O.gemm_integer_scale(x, w, s).output
    xq = torch.from_numpy(x.values.astype(np.int8)).cuda()
    sa = torch.from_numpy(x.scales).cuda()
    out = isb.gemm_integer_scale(xq, sa, pw, out_dtype=torch.float32).cpu().numpy()
    assert np.array_equal(out.view(np.int32), ref.view(np.int32))
    # amplifier search from the sidecar scales (llama-like -> 1024)
    assert Q.load_packed_weight(tmp_path / "w.qtns").info["amplifier"] == 1024
