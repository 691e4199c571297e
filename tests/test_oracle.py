"""Pin the oracle (oracle/bfp_oracle.c) to the reference before trusting it.

CPU only.  The C restatement is checked against
  * the reference headers compiled in place (oracle/_ref) -- exhaustively for
    every <= 9-bit format in all four modes and all five operations, on
    seeded random + directed operands for the rest;
  * the golden fixtures in tests/golden/ (written by the reference itself);
  * the SPEC known-answer examples that the survey verified against the code
    (SURVEY.md §4), and hardware binary16 conversion for 1/5/10 RN.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import FORMATS, MODES, all_pairs, operands, related, ROOT

GOLDEN = ROOT / "tests" / "golden"


# --------------------------------------------------------------- known answers
def test_spec_known_answers(oracle):
    O = oracle.orc()
    assert O.orc_encode(1.5, 4, 3, 1, 0) == 0x3C
    assert O.orc_encode(512.0, 4, 3, 1, 0) == 0x78  # overflow -> Inf under RN
    assert O.orc_encode(512.0, 4, 3, 0, 0) == 0x77  # max finite under RZ
    assert O.orc_binop(0, 4, 3, 1, 0, 0x3C, 0x42) == 0x48
    assert O.orc_binop(2, 4, 3, 1, 0, 0x3C, 0x42) == 0x47
    assert O.orc_binop(2, 4, 3, 0, 0, 0x3D, 0x3B) == 0x40
    assert O.orc_binop(2, 4, 3, 1, 0, 0x3D, 0x3B) == 0x41
    assert O.orc_binop(3, 4, 3, 1, 0, 0x38, 0x40) == 0x30
    # max finite of 1/4/3 is 240 (format.hpp:46-48, bias 7; SPEC.md:239 says 480)
    assert O.orc_decode(0x77, 4, 3) == 240.0


def test_ieee_conventions(oracle):
    O = oracle.orc()
    e, s = 4, 3
    nan = 0x7C  # canonical: positive, fraction MSB (format.hpp:49-52)
    for rn in (0, 1):
        assert O.orc_binop(0, e, s, rn, 0, 0x78, 0xF8) == nan  # Inf - Inf
        assert O.orc_binop(2, e, s, rn, 0, 0x78, 0x00) == nan  # Inf * 0
        assert O.orc_binop(0, e, s, rn, 0, 0x3C, 0xBC) == 0x00  # x + (-x) = +0
        assert O.orc_binop(0, e, s, rn, 0, 0x80, 0x80) == 0x80  # -0 + -0 = -0
        assert O.orc_binop(0, e, s, rn, 0, 0x7F, 0x01) == nan  # NaN propagates canonical
    assert O.orc_binop(0, e, s, 1, 0, 0x77, 0x77) == 0x78  # RN overflow -> Inf
    assert O.orc_binop(0, e, s, 0, 0, 0x77, 0x77) == 0x77  # RZ overflow -> max finite


# --------------------------------------------------- C restatement vs reference
@pytest.mark.parametrize("fmt2", [(3, 2), (4, 3), (5, 3)])
@pytest.mark.parametrize("mode", MODES)
def test_restatement_exhaustive_vs_reference(ref_oracle, fmt2, mode):
    O = ref_oracle
    e, s = fmt2
    fmt = (e, s) + mode
    x, y = all_pairs(1 + e + s)
    for op in ("add", "sub", "mul", "div"):
        want = O.ref_binop_enc(op, fmt, x, y)
        got = O.binop(op, fmt, x, y)
        bad = np.nonzero(want != got)[0]
        assert len(bad) == 0, (op, fmt, [(hex(int(x[i])), hex(int(y[i])), hex(int(want[i])), hex(int(got[i])))
                                         for i in bad[:5]])


@pytest.mark.parametrize("fmt2", [f for f in FORMATS if 1 + f[0] + f[1] > 9])
@pytest.mark.parametrize("mode", MODES)
def test_restatement_random_vs_reference(ref_oracle, fmt2, mode):
    O = ref_oracle
    e, s = fmt2
    fmt = (e, s) + mode
    rng = np.random.default_rng(hash((e, s) + mode) & 0xFFFFFFFF)
    n = 1 << 14
    x = operands(e, s, n, rng)
    y = operands(e, s, n, rng)
    y[: n // 8] = related(x[: n // 8], e, s, rng)
    c = operands(e, s, n, rng)
    for op in ("add", "sub", "mul", "div", "mul_add"):
        want = O.ref_binop_enc(op, fmt, x, y, c if op == "mul_add" else None)
        got = O.binop(op, fmt, x, y, c)
        assert np.array_equal(want, got), (op, fmt, int((want != got).sum()))


def test_restatement_codec_vs_reference(ref_oracle):
    O = ref_oracle
    rng = np.random.default_rng(7)
    bits = rng.integers(0, 1 << 32, size=1 << 16, dtype=np.uint64).astype(np.uint32)
    xs = bits.view(np.float32)
    for (e, s) in FORMATS:
        for mode in MODES:
            fmt = (e, s) + mode
            assert np.array_equal(O.encode_f32(fmt, xs), O.ref_encode_f32(fmt, xs)), fmt
        encs = rng.integers(0, 1 << (1 + e + s), size=1 << 12, dtype=np.uint64)
        a = O.decode_f32((e, s, 1, 0), encs).view(np.uint32)
        b = O.ref_decode_f32((e, s, 1, 0), encs).view(np.uint32)
        assert np.array_equal(a, b), (e, s)


def test_encode_matches_binary16_hardware(oracle):
    """encode_scalar for 1/5/10 RN gradual == IEEE binary16 RN conversion
    (numpy's float32 -> float16), NaN aside."""
    rng = np.random.default_rng(11)
    bits = rng.integers(0, 1 << 32, size=1 << 18, dtype=np.uint64).astype(np.uint32)
    xs = bits.view(np.float32)
    ok = ~np.isnan(xs)
    want = xs[ok].astype(np.float16).view(np.uint16).astype(np.uint64)
    got = oracle.encode_f32((5, 10, 1, 0), xs[ok])
    assert np.array_equal(want, got)


# ----------------------------------------------------------------------- layout
def test_layout_restatement_vs_reference(ref_oracle):
    O = ref_oracle
    rng = np.random.default_rng(3)
    for (e, s) in [(4, 3), (5, 10), (8, 23)]:
        nb = 1 + e + s
        for n in (1, 31, 32, 1023, 1024, 1025, 3000):
            enc = rng.integers(0, 1 << nb, size=n, dtype=np.uint64)
            p_ref = O.ref_pack_planes((e, s), enc)
            p_orc = O.pack_planes(enc, nb)
            assert np.array_equal(p_ref, p_orc), (e, s, n)
            assert np.array_equal(O.ref_unpack_planes((e, s), p_ref, n), enc)
            assert np.array_equal(O.unpack_planes(p_orc, n, nb), enc)


def test_shipped_pack_defect_recorded(ref_oracle):
    """Defect B: the shipped transpose64 is anti-diagonal, so
    pack([0x3C]) yields all-zero lanes for any format with n <= 32 bits and
    unpack(pack(x)) != x.  Parity therefore uses the documented layout."""
    O = ref_oracle
    enc = np.array([0x3C], dtype=np.uint64)
    shipped = O.ref_pack_planes((4, 3), enc, shipped=True)
    assert not shipped.any()
    documented = O.ref_pack_planes((4, 3), enc)
    lanes = [j for j in range(8) if documented[j * 32] & 1]
    assert lanes == [2, 3, 4, 5]  # SPEC.md:226 says 2,4,5,6 -- also wrong


# ---------------------------------------------------------------------- golden
def test_restatement_vs_golden(oracle):
    g = np.load(GOLDEN / "arith.npz")
    for (e, s) in FORMATS:
        for (rn, ftz) in MODES:
            key = f"{e}_{s}_{rn}_{ftz}"
            fmt = (e, s, rn, ftz)
            x, y, c = (g[f"{k}_{key}"].astype(np.uint64) for k in "xyc")
            for op in ("add", "sub", "mul", "div", "mul_add"):
                got = oracle.binop(op, fmt, x, y, c)
                assert np.array_equal(got, g[f"{op}_{key}"].astype(np.uint64)), (op, key)


def test_codec_vs_golden(oracle):
    g = np.load(GOLDEN / "codec.npz")
    for (e, s) in FORMATS:
        for (rn, ftz) in MODES:
            key = f"{e}_{s}_{rn}_{ftz}"
            fmt = (e, s, rn, ftz)
            xs = g[f"f32in_{key}"].view(np.float32)
            assert np.array_equal(oracle.encode_f32(fmt, xs), g[f"enc_{key}"].astype(np.uint64)), key
            dec = oracle.decode_f32(fmt, g[f"decin_{key}"].astype(np.uint64)).view(np.uint32)
            assert np.array_equal(dec, g[f"dec_{key}"]), key


def test_layout_vs_golden(oracle):
    g = np.load(GOLDEN / "layout.npz")
    for (e, s) in [(4, 3), (5, 10), (8, 15), (8, 23)]:
        nb = 1 + e + s
        enc = g[f"enc_{e}_{s}"].astype(np.uint64)
        assert np.array_equal(oracle.pack_planes(enc, nb), g[f"planes_{e}_{s}"])
        assert not np.array_equal(g[f"shipped_{e}_{s}"], g[f"planes_{e}_{s}"])
