"""The C-ABI library: loads, exports every symbol include/bfpgpu.h declares,
and its host-side logic (validation, same-shape, sizes) matches the reference
-- CPU only, no compute calls.  Plus the host mirror of the reference API."""
from __future__ import annotations

import ctypes as C
import math
import re

import numpy as np
import pytest

from conftest import FORMATS, MODES, ROOT

import paper_1602_04716_b200 as bfp
from paper_1602_04716_b200 import _lib


def _declared_symbols() -> list[str]:
    text = (ROOT / "include" / "bfpgpu.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bfp_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def L():
    if not _lib.LIB_PATH.exists():
        from paper_1602_04716_b200.build import build
        build(verbose=False)
    return _lib.lib()


def test_exports_every_declared_symbol(L):
    syms = _declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    # and the Python binding knows the signature of each of them
    assert set(syms) <= set(_lib.SIGNATURES), set(syms) - set(_lib.SIGNATURES)


def fmt(e, s, rn=1, ftz=0, name=b""):
    return _lib.BfpFormat(e, s, rn, ftz, name)


def test_validate_ranges_match_reference(L, ref_oracle):
    """validate(): e in [2, 11], s in [1, 52], 1+e+s <= 64 (format.hpp:57-64)."""
    R = ref_oracle.ref()
    for e in range(0, 14):
        for s in range(0, 56):
            want = R.ref_validate(e, s) == 0
            got = L.bfp_validate(C.byref(fmt(e, s))) == _lib.BFP_OK
            assert want == got, (e, s)


def test_same_shape_compares_name(L):
    """require_same_shape compares the whole spec incl. name (arith.hpp:228-231)."""
    a, b = fmt(4, 3, name=b"fp8"), fmt(4, 3, name=b"fp8")
    assert L.bfp_same_shape(C.byref(a), C.byref(b)) == _lib.BFP_OK
    c = fmt(4, 3, name=b"e4m3")
    assert L.bfp_same_shape(C.byref(a), C.byref(c)) == _lib.BFP_EMISMATCH
    assert L.bfp_same_shape(C.byref(a), C.byref(fmt(4, 3, rn=0, name=b"fp8"))) == _lib.BFP_EMISMATCH
    assert L.bfp_same_shape(C.byref(fmt(4, 3)), C.byref(_lib.BfpFormat(4, 3, 1, 0, None))) == _lib.BFP_OK


def test_sizes(L):
    for (e, s) in FORMATS:
        n = 1 + e + s
        f = fmt(e, s)
        assert L.bfp_is_supported(C.byref(f)) == 1
        for count in (0, 1, 1024, 1025, 5000):
            assert L.bfp_plane_bytes(C.byref(f), count) == ((count + 1023) // 1024) * n * 128
        assert L.bfp_enc_bytes(C.byref(f)) == (1 if n <= 8 else 2 if n <= 16 else 4)
        assert L.bfp_is_compiled(C.byref(f)) == 1
    assert L.bfp_is_compiled(C.byref(fmt(7, 20))) == 0  # legal, not instantiated: NVRTC backend
    assert L.bfp_is_supported(C.byref(fmt(7, 20))) == 1
    assert L.bfp_is_supported(C.byref(fmt(12, 3))) == 0  # illegal


def test_python_mirror_errors():
    with pytest.raises(ValueError):
        bfp.make_spec(1, 3)
    with pytest.raises(ValueError):
        bfp.make_spec(4, 0)
    with pytest.raises(ValueError):
        bfp.make_spec(11, 53)
    f = bfp.make_spec(4, 3)
    assert f.rounding == bfp.rounding_mode.rn and f.subnormals == bfp.subnormal_policy.gradual
    assert (f.bias(), f.emin(), f.emax()) == (7, -6, 7)
    assert f.canonical_nan() == 0x7C and f.inf(1) == 0xF8 and f.max_finite(0) == 0x77
    with pytest.raises(ValueError):
        bfp.require_same_shape(bfp.make_spec(4, 3, name="a"), bfp.make_spec(4, 3, name="b"))


def test_host_scalar_codec_matches_oracle(oracle):
    rng = np.random.default_rng(1)
    vals = list(rng.standard_normal(300) * 100) + [0.0, -0.0, math.inf, -math.inf, math.nan, 1e-30,
                                                   65504.0, 65520.0, 2.0 ** -24, 3 * 2.0 ** -26]
    for (e, s) in FORMATS:
        for (rn, ftz) in MODES:
            f = bfp.make_spec(e, s, rn, ftz)
            for v in vals:
                assert bfp.encode_scalar(v, f) == oracle.orc().orc_encode(v, e, s, rn, ftz), (e, s, v)
        f = bfp.make_spec(e, s)
        for enc in rng.integers(0, 1 << (1 + e + s), size=200):
            a = bfp.decode_scalar(int(enc), f)
            b = oracle.orc().orc_decode(int(enc), e, s)
            assert (math.isnan(a) and math.isnan(b)) or a == b


def test_split_classify_mirror(oracle):
    """split / classify (format.hpp:83-99) agree with the oracle's exact decode
    on every encoding of the <= 9-bit formats and sampled wider ones."""
    rng = np.random.default_rng(7)
    for (e, s) in FORMATS:
        f = bfp.make_spec(e, s)
        nb = 1 + e + s
        encs = range(1 << nb) if nb <= 9 else [int(x) for x in rng.integers(0, 1 << nb, size=2000)]
        for enc in encs:
            sc = bfp.split(enc, f)
            assert sc.sign == enc >> (e + s) and sc.fraction == enc & ((1 << s) - 1)
            assert sc.biased_exp == (enc >> s) & ((1 << e) - 1)
            x = oracle.orc().orc_decode(enc, e, s)
            want = (bfp.value_class.nan if math.isnan(x) else bfp.value_class.infinity if math.isinf(x)
                    else bfp.value_class.zero if x == 0 else bfp.value_class.subnormal
                    if abs(x) < 2.0 ** f.emin() else bfp.value_class.normal)
            assert bfp.classify(enc, f) == want, (e, s, enc)


def test_chain_program_validation(L):
    """bfp_chain rejects malformed programs before touching the device."""
    import ctypes as C
    from paper_1602_04716_b200 import _lib
    f = _lib.BfpFormat(4, 3, 1, 0, b"")
    ptrs = (C.c_void_p * 2)(None, None)
    for prog in (b"a+", b"ab", b"abc+", b"ax+", b"ab%", b"", b"ac+"):
        assert L.bfp_chain(C.byref(f), prog, 2, ptrs, None, 1024, None) == _lib.BFP_EARG, prog
    assert L.bfp_chain(C.byref(f), b"ab+", 9, ptrs, None, 1024, None) == _lib.BFP_EARG
    assert L.bfp_chain(C.byref(f), None, 2, ptrs, None, 1024, None) == _lib.BFP_EARG
    bad = _lib.BfpFormat(1, 3, 1, 0, b"")
    assert L.bfp_chain(C.byref(bad), b"ab+", 2, ptrs, None, 1024, None) == _lib.BFP_EFORMAT
    assert L.bfp_chain(C.byref(f), b" a b + ", 2, ptrs, None, 0, None) == _lib.BFP_OK  # count 0


def test_chain_f32_validation(L):
    import ctypes as C
    from paper_1602_04716_b200 import _lib
    ptrs = (C.c_void_p * 2)(None, None)
    wide = _lib.BfpFormat(8, 23 + 1, 1, 0, b"")  # no float32 codec beyond s = 23
    assert L.bfp_chain_f32(C.byref(wide), b"ab+", 2, ptrs, None, 1024, None) == _lib.BFP_EUNSUPPORTED
    f = _lib.BfpFormat(5, 10, 1, 0, b"")
    assert L.bfp_chain_f32(C.byref(f), b"ab", 2, ptrs, None, 1024, None) == _lib.BFP_EARG


def test_arith_ex_flags_validated(L):
    import ctypes as C
    from paper_1602_04716_b200 import _lib
    f = _lib.BfpFormat(4, 3, 1, 0, b"")
    assert L.bfp_arith_ex(0, C.byref(f), None, None, None, None, 0, None, 4) == _lib.BFP_EARG
    assert L.bfp_arith_ex(0, C.byref(f), None, None, None, None, 0, None, _lib.BFP_INPUTS_READY) == _lib.BFP_OK
    assert L.bfp_arith_ex(4, C.byref(f), None, None, None, None, 0, None,
                          _lib.BFP_INPUTS_READY | _lib.BFP_GENERAL_NETWORK) == _lib.BFP_OK
