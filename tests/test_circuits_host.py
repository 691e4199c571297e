"""The device networks (csrc/bfp_circuits.cuh, bfp_layout.cuh) compiled for
the host and checked against the oracle -- CPU only, exhaustive where the
format is small.  The same source is what runs on the B200; the GPU tests
(test_gpu_parity.py) repeat the checks through the C ABI."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import FORMATS, MODES, all_pairs, fast_domain, fast_domain_operands, operands, related, ROOT

GOLDEN = ROOT / "tests" / "golden"


def _check(O, host, op, fmt, x, y, c=None, generated=(False, True)):
    """templates AND the generated LOP3 covers (the code the kernels run)."""
    nb = 1 + fmt[0] + fmt[1]
    px, py = O.pack_planes(x, nb), O.pack_planes(y, nb)
    pc = O.pack_planes(c, nb) if c is not None else None
    want = O.binop(op, fmt, x, y, c)
    for gen in generated:
        got = O.unpack_planes(host.binop(op, fmt, px, py, pc, gen), len(x), nb)
        bad = np.nonzero(want != got)[0]
        assert len(bad) == 0, (op, fmt, gen, len(bad),
                               [(hex(int(x[i])), hex(int(y[i])), hex(int(want[i])), hex(int(got[i])))
                                for i in bad[:5]])


@pytest.mark.parametrize("fmt2", [(3, 2), (4, 3), (5, 3)])
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("op", ["add", "sub", "mul", "div"])
def test_exhaustive_small(oracle, host, fmt2, mode, op):
    x, y = all_pairs(1 + fmt2[0] + fmt2[1])
    _check(oracle, host, op, fmt2 + mode, x, y)


@pytest.mark.parametrize("op", ["add", "mul", "div"])
def test_exhaustive_13bit(oracle, host, op):
    """1/5/7: all 2^26 pairs, RN + gradual."""
    x, y = all_pairs(13)
    _check(oracle, host, op, (5, 7, 1, 0), x, y, generated=(False,))  # covers: GPU suite


@pytest.mark.parametrize("fmt2", [f for f in FORMATS if 1 + f[0] + f[1] > 9])
@pytest.mark.parametrize("mode", MODES)
def test_random_wide(oracle, host, fmt2, mode):
    e, s = fmt2
    rng = np.random.default_rng((e * 64 + s) * 4 + mode[0] * 2 + mode[1])
    n = 1 << 16
    x = operands(e, s, n, rng)
    y = operands(e, s, n, rng)
    y[: n // 8] = related(x[: n // 8], e, s, rng)
    c = operands(e, s, n, rng)
    for op in ("add", "sub", "mul", "div", "mul_add"):
        _check(oracle, host, op, fmt2 + mode, x, y, c if op == "mul_add" else None)


def test_mul_add_small_exhaustive_c(oracle, host):
    """chain round(round(a*b)+c) for 1/3/2: all (a, b) against 8 c values."""
    x, y = all_pairs(6)
    rng = np.random.default_rng(5)
    for cval in rng.integers(0, 64, size=8):
        c = np.full_like(x, cval)
        for mode in MODES:
            _check(oracle, host, "mul_add", (3, 2) + mode, x, y, c)


# ------------------------------------------------- mul_add: the fast domain
def _check_fast(O, host, fmt, a, b, c, min_inside, generated=(False, True)):
    """Predicate = its restatement; inside the domain the fast template and the
    fast cover equal the oracle's chain (outside they are never run)."""
    e, s = fmt[:2]
    nb = 1 + e + s
    pa, pb, pc = (O.pack_planes(v, nb) for v in (a, b, c))
    dom = O.unpack_planes(host.binop("mul_add_domain", fmt, pa, pb, pc), len(a), nb) & np.uint64(1)
    inside = fast_domain(e, s, a, b, c)
    assert np.array_equal(dom.astype(bool), inside), fmt
    assert int(inside.sum()) >= min_inside, (fmt, int(inside.sum()))
    want = O.binop("mul_add", fmt, a, b, c)
    for gen in generated:
        got = O.unpack_planes(host.binop("mul_add_fast", fmt, pa, pb, pc, gen), len(a), nb)
        bad = np.nonzero((want != got) & inside)[0]
        assert len(bad) == 0, (fmt, gen, len(bad), [(hex(int(a[i])), hex(int(b[i])), hex(int(c[i])),
                                                     hex(int(want[i])), hex(int(got[i]))) for i in bad[:5]])


@pytest.mark.parametrize("mode", [(1, 0), (0, 1)])  # the GPU suite runs all four modes over the same triples
def test_mul_add_fast_domain_exhaustive_1_4_3(oracle, host, mode):
    """Every (a, b, c) triple of 1/4/3 (2^24): the fast network is only ever run
    inside its domain, and there it must equal bfp_add(bfp_mul(a, b), c)."""
    v = np.arange(1 << 8, dtype=np.uint64)
    a, b, c = (g.ravel() for g in np.meshgrid(v, v, v, indexing="ij"))
    _check_fast(oracle, host, (4, 3) + mode, a, b, c, min_inside=1 << 19)


@pytest.mark.parametrize("mode", [(1, 0), (0, 1)])  # all four modes: 35 s, 0 mismatches
def test_mul_add_fast_cover_exhaustive_1_5_3(oracle, host, mode):
    """The generated fast-domain cover of 1/5/3 on EVERY (a, b, c) inside its
    domain (27.4 M triples of the 2^27), enumerated from the exponent ranges."""
    e, s = 5, 3
    fmt = (e, s) + mode
    v = np.arange(1 << 9, dtype=np.uint64)
    ex = (v >> np.uint64(s)) & np.uint64(31)
    A, Cv = v[(ex >= 1) & (ex < 24)], v[(ex >= 8) & (ex < 24)]
    total = 0
    for a8 in A.reshape(-1, 8):
        a, b, c = (g.ravel() for g in np.meshgrid(a8, A, Cv, indexing="ij"))
        keep = fast_domain(e, s, a, b, c)
        a, b, c = a[keep], b[keep], c[keep]
        if not len(a):
            continue
        total += len(a)
        pad = -len(a) % 1024
        a, b, c = (np.concatenate([x, np.repeat(x[-1:], pad)]) for x in (a, b, c))
        want = oracle.binop("mul_add", fmt, a, b, c)
        got = oracle.unpack_planes(host.binop("mul_add_fast", fmt, *(oracle.pack_planes(x, 9) for x in (a, b, c)),
                                              True), len(a), 9)
        assert np.array_equal(got, want), (fmt, int((got != want).sum()))
    assert total == 27394048


@pytest.mark.parametrize("fmt2", [f for f in FORMATS if 1 + f[0] + f[1] > 8])
@pytest.mark.parametrize("mode", [(1, 0), (0, 1)])  # all four modes: test_gpu_parity.py, same generator
def test_mul_add_fast_domain_random(oracle, host, fmt2, mode):
    """Wider formats: special-weighted operands (mostly outside the domain: the
    predicate must say so) and operands generated inside it, weighted towards
    its edges, with c correlated to the product (cancellation, ties)."""
    e, s = fmt2
    rng = np.random.default_rng((e * 64 + s) * 4 + mode[0] * 2 + mode[1] + 77)
    n = 1 << 17
    a, b, c = (operands(e, s, n, rng) for _ in range(3))
    a[n // 2:], b[n // 2:], c[n // 2:] = (v[n // 2:] for v in fast_domain_operands(oracle, fmt2 + mode, n, rng))
    c[: n // 2] = fast_domain_operands(oracle, fmt2 + mode, n // 2, rng)[2]  # a, b decide
    _check_fast(oracle, host, fmt2 + mode, a, b, c, min_inside=n // 2)
    _check_fast(oracle, host, fmt2 + mode, *fast_domain_operands(oracle, fmt2 + mode, n, rng), min_inside=n)


def test_golden_host(oracle, host):
    g = np.load(GOLDEN / "arith.npz")
    for (e, s) in FORMATS:
        nb = 1 + e + s
        for (rn, ftz) in MODES:
            key = f"{e}_{s}_{rn}_{ftz}"
            x, y, c = (g[f"{k}_{key}"].astype(np.uint64) for k in "xyc")
            px, py, pc = (oracle.pack_planes(v, nb) for v in (x, y, c))
            for op in ("add", "sub", "mul", "div", "mul_add"):
                for generated in (False, True):
                    z = host.binop(op, (e, s, rn, ftz), px, py, pc if op == "mul_add" else None,
                                   generated)
                    got = oracle.unpack_planes(z, len(x), nb)
                    assert np.array_equal(got, g[f"{op}_{key}"].astype(np.uint64)), (op, key)


# ----------------------------------------------------------------------- codec
@pytest.mark.parametrize("fmt2", FORMATS)
def test_codec_host(oracle, host, fmt2):
    e, s = fmt2
    rng = np.random.default_rng(e * 100 + s)
    bits = rng.integers(0, 1 << 32, size=1 << 16, dtype=np.uint64).astype(np.uint32)
    bits[: 1 << 14] = (bits[: 1 << 14] & 0x807FFFFF) | (
        rng.integers(90, 165, size=1 << 14, dtype=np.uint64).astype(np.uint32) << 23)
    for mode in MODES:
        fmt = fmt2 + mode
        want = oracle.encode_f32(fmt, bits.view(np.float32))
        for direction in (0, 2):  # restatement and branch-free kernel codec
            got = host.codec(direction, fmt, bits).astype(np.uint64)
            assert np.array_equal(got, want), (fmt, direction, int((got != want).sum()))
    nb = 1 + e + s
    encs = (np.arange(1 << nb, dtype=np.uint64) if nb <= 16
            else rng.integers(0, 1 << nb, size=1 << 16, dtype=np.uint64))
    want = oracle.decode_f32((e, s, 1, 0), encs).view(np.uint32)
    for direction in (1, 3):
        got = host.codec(direction, (e, s, 1, 0), encs.astype(np.uint32))
        assert np.array_equal(got, want), direction


# ---------------------------------------------------------------------- layout
@pytest.mark.parametrize("eb,nb", [(1, 6), (1, 8), (2, 9), (2, 16), (3, 24), (4, 24), (4, 32),
                                   (5, 40), (6, 41), (7, 56), (8, 33), (8, 64)])
def test_transpose_host(oracle, host, eb, nb):
    rng = np.random.default_rng(nb)
    for n in (1, 33, 1024, 2500):
        enc = rng.integers(0, 1 << nb, size=n, dtype=np.uint64)
        planes = host.pack_enc(eb, nb, enc)
        assert np.array_equal(planes, oracle.pack_planes(enc, nb)), (eb, nb, n)
        assert np.array_equal(host.unpack_enc(eb, nb, planes, n), enc)


def test_layout_golden_host(host):
    g = np.load(GOLDEN / "layout.npz")
    for (e, s) in [(4, 3), (5, 10), (8, 15), (8, 23)]:
        nb = 1 + e + s
        eb = 1 if nb <= 8 else 2 if nb <= 16 else 4
        enc = g[f"enc_{e}_{s}"].astype(np.uint64)
        assert np.array_equal(host.pack_enc(eb, nb, enc), g[f"planes_{e}_{s}"])


def test_bfpraw_stride3_host(host):
    """3-byte .bfpraw records (pack.hpp:78-109) <-> 32-bit encodings."""
    import ctypes as C
    host.L.host_raw3.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(24)
    for _ in range(50):
        raw = rng.integers(0, 256, size=96, dtype=np.uint8)
        enc = np.zeros(32, dtype=np.uint32)
        back = np.zeros(96, dtype=np.uint8)
        host.L.host_raw3(raw.ctypes.data, enc.ctypes.data, back.ctypes.data)
        want = raw.reshape(32, 3).astype(np.uint32)
        want = want[:, 0] | (want[:, 1] << 8) | (want[:, 2] << 16)
        assert np.array_equal(enc, want)
        assert np.array_equal(back, raw)


@pytest.mark.parametrize("fmt2", FORMATS + [(11, 52), (10, 40), (11, 20), (2, 1)])
def test_codec64_host(oracle, ref_oracle, host, fmt2):
    """encode_scalar(double) / decode_scalar (format.hpp:101-188) for any legal
    format, against the C restatement and (sampled) the reference itself."""
    e, s = fmt2
    rng = np.random.default_rng(e * 1000 + s)
    bits = rng.integers(0, 1 << 63, size=1 << 15, dtype=np.uint64) * np.uint64(2) + \
        rng.integers(0, 2, size=1 << 15, dtype=np.uint64)
    ex = rng.integers(1023 - 1100, 1023 + 1100, size=1 << 14).clip(0, 2047).astype(np.uint64)
    bits[: 1 << 14] = (bits[: 1 << 14] & np.uint64(0x800FFFFFFFFFFFFF)) | (ex << np.uint64(52))
    xs = bits.view(np.float64)
    for mode in MODES:
        fmt = fmt2 + mode
        want = oracle.encode_f64(fmt, xs)
        assert np.array_equal(host.codec64(0, fmt, bits), want), fmt
        R = ref_oracle.ref()
        for v in xs[:200]:
            assert R.ref_encode_f64(float(v), e, s, mode[0], mode[1]) == oracle.orc().orc_encode(
                float(v), e, s, mode[0], mode[1])
    nb = 1 + e + s
    encs = rng.integers(0, 1 << min(nb, 63), size=1 << 14, dtype=np.uint64)
    if nb == 64:
        encs = encs * np.uint64(2) + rng.integers(0, 2, size=len(encs), dtype=np.uint64)
    got = host.codec64(1, fmt2 + (1, 0), encs)
    want = oracle.decode_f64(fmt2 + (1, 0), encs).view(np.uint64)
    nan = np.isnan(want.view(np.float64))
    assert np.array_equal(got[~nan], want[~nan])
    assert np.all(got[nan] == np.uint64(0x7FF8000000000000))  # quiet_NaN()


@pytest.mark.parametrize("s", list(range(2, 31)))
def test_significand_products_exact(host, s):
    """Array and radix-4 Booth (constexpr Dadda schedule) significand products
    equal the exact integer product lane by lane, S = 2..30 (mul_w uses Booth
    for S >= 9), with random significands and the all-ones top bits mul_w feeds."""
    import ctypes as C
    L = host.L
    L.host_product.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
    rng = np.random.default_rng(100 + s)
    for trial in range(24):
        a = rng.integers(0, 1 << 32, s + 1, dtype=np.uint64).astype(np.uint32)
        b = rng.integers(0, 1 << 32, s + 1, dtype=np.uint64).astype(np.uint32)
        if trial % 2:
            a[s] = b[s] = 0xFFFFFFFF
        if trial == 2:
            a[:] = b[:] = 0xFFFFFFFF
        # per-lane values (bit j of lane k = bit k of word j)
        av = [sum(((int(a[j]) >> k) & 1) << j for j in range(s + 1)) for k in range(32)]
        bv = [sum(((int(b[j]) >> k) & 1) << j for j in range(s + 1)) for k in range(32)]
        want = [x * y for x, y in zip(av, bv)]
        for which in (0, 1):
            p = np.zeros(2 * s + 2, dtype=np.uint32)
            assert L.host_product(s, which, a.ctypes.data, b.ctypes.data, p.ctypes.data) == 0
            got = [sum(((int(p[j]) >> k) & 1) << j for j in range(2 * s + 2)) for k in range(32)]
            assert got == want, (s, which, trial)


def test_template_format_sweep(tmp_path, oracle):
    """The template networks (what the NVRTC backend compiles) over ~60
    formats incl. 1/2/5, 1/3/11, 1/2/24 (working exponent wider than E + 2)
    and both RN + gradual and RZ + FTZ, against the oracle."""
    import subprocess
    from conftest import ROOT
    exe = tmp_path / "format_sweep"
    subprocess.run(["g++", "-O1", "-std=c++17", str(ROOT / "tests" / "native" / "format_sweep.cpp"),
                    f"-L{ROOT / 'oracle'}", "-loracle", f"-Wl,-rpath,{ROOT / 'oracle'}", "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip().endswith("total bad 0"), r.stdout


def test_runtime_cover_generator(tmp_path):
    """tools/lutmap/gen.cpp in GEN_ONE mode (what BFP_JIT_MAP=1 runs for a
    runtime format): its header equals the template networks bit for bit."""
    import subprocess
    from conftest import ROOT
    csrc = ROOT / "paper_1602_04716_b200" / "csrc"
    lut = ROOT / "tools" / "lutmap"
    e, s, rn, ftz = 3, 11, 1, 0
    gen = tmp_path / "gen"
    subprocess.run(["g++", "-O2", "-std=c++17", f"-I{csrc}", f"-I{lut}", f"-DGEN_ONE_E={e}", f"-DGEN_ONE_S={s}",
                    f"-DGEN_ONE_RN={rn}", f"-DGEN_ONE_FTZ={ftz}", str(lut / "gen.cpp"), "-o", str(gen)], check=True)
    subprocess.run([str(gen), str(tmp_path)], check=True)
    hdr = tmp_path / f"gen_{e}_{s}_{rn}_{ftz}.cuh"
    assert hdr.exists()
    src = tmp_path / "check.cpp"
    src.write_text(f"""
#include "bfp_circuits.cuh"
#include "{hdr.name}"
#include <cstdio>
#include <random>
using namespace bfpg;
using F = Format<{e}, {s}, {str(bool(rn)).lower()}, {str(bool(ftz)).lower()}>;
int main() {{
  std::mt19937 r(3);
  long bad = 0;
  for (int it = 0; it < 4000; ++it) {{
    w32 X[F::N], Y[F::N], C[F::N], Z1[F::N], Z2[F::N];
    for (int j = 0; j < F::N; ++j) {{ X[j] = r(); Y[j] = r(); C[j] = r(); }}
    Gen<F, 0>::run(X, Y, C, Z1); add_w<F, false>(X, Y, Z2); for (int j = 0; j < F::N; ++j) bad += Z1[j] != Z2[j];
    Gen<F, 1>::run(X, Y, C, Z1); add_w<F, true>(X, Y, Z2); for (int j = 0; j < F::N; ++j) bad += Z1[j] != Z2[j];
    Gen<F, 2>::run(X, Y, C, Z1); mul_w<F>(X, Y, Z2); for (int j = 0; j < F::N; ++j) bad += Z1[j] != Z2[j];
    Gen<F, 3>::run(X, Y, C, Z1); div_w<F>(X, Y, Z2); for (int j = 0; j < F::N; ++j) bad += Z1[j] != Z2[j];
    Gen<F, 4>::run(X, Y, C, Z1); mul_add_w<F>(X, Y, C, Z2); for (int j = 0; j < F::N; ++j) bad += Z1[j] != Z2[j];
  }}
  std::printf("bad %ld\\n", bad);
  return bad != 0;
}}
""")
    exe = tmp_path / "check"
    subprocess.run(["g++", "-O1", "-std=c++17", f"-I{csrc}", f"-I{tmp_path}", str(src), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "bad 0" in r.stdout, r.stdout + r.stderr
