"""CPU checks of the drop-in boundary: the in-tree sm_100a library loads here (no
GPU needed to dlopen it) and exports every entry point include/intscale_b200.h
declares; host-only helpers of the offline path match the oracle."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "intscale_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(isb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["isb_quantize_per_token", "isb_weight_pack_codes", "isb_weight_pack_signed4",
                 "isb_gemm_integer_scale", "isb_gemm_float_scale", "isb_gemm_checked",
                 "isb_overflow_analyzer", "isb_integerize_scales"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2405_14597_b200 import _lib
    lib = C.CDLL(_lib.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the Python mirror binds exactly those
    assert set(_lib.SIGNATURES) == set(declared_functions())


def test_sass_is_tcgen05_native():
    import subprocess
    from paper_2405_14597_b200 import _lib
    try:
        sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True,
                              text=True, timeout=300).stdout
    except FileNotFoundError:
        pytest.skip("cuobjdump not available")
    assert "UTCIMMA" in sass          # tcgen05.mma.kind::i8
    assert "UTMALDG" in sass          # TMA tensor loads
    assert "LDTM" in sass and "STTM" in sass  # TMEM traffic
    assert not re.search(r"(?<![A-Z])(HMMA|IMMA)", sass)  # no legacy mma.sync path


def test_host_helpers_match_oracle(oracle):
    import paper_2405_14597_b200 as isb
    rng = oracle.Rng(7)
    for _ in range(50):
        s = np.array([oracle.exp2(-11.0 + 13.0 * rng.u01()) for _ in range(40)])
        assert isb.search_amplifier(s) == oracle.search_amplifier(s)
        for amp in (1, 8, 1024, 8192):
            a = isb.integerize_scales(s, amp)
            b = oracle.integerize_scales(s, amp)
            assert np.array_equal(a.int_scales, b.int_scales) and a.exponent == b.exponent
    ks = oracle.IntegerScaleSet(np.full(32, 1024, np.int32), 1024, 10)
    r = isb.overflow_analyzer(4096, 128, 8, 4, isb.IntegerScaleSet(ks.int_scales, 1024, 10))
    assert r["static_bound"] == 4261412864 and not r["safe"]
    with pytest.raises(isb.OverflowError_):
        isb.integerize_scales([3.0e6], 1024)
    with pytest.raises(isb.ParamError):
        isb.integerize_scales([0.5], 3)


def test_compute_entry_points_fail_loudly_without_gpu():
    """No CPU fallback: on a host without a GPU the device entry points raise."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2405_14597_b200 as isb
    with pytest.raises(isb.ParamError):
        isb.quantize_per_token(torch.zeros(2, 4))
