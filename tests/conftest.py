"""Shared fixtures.  `-m gpu` tests need a B200; everything else runs on CPU."""
from __future__ import annotations

import ctypes as C
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import oracle as O  # noqa: E402  (test infrastructure: the checker)

# Formats with compiled networks, and all four mode combinations.
FORMATS = [(3, 2), (4, 3), (5, 3), (5, 7), (5, 10), (6, 9), (8, 7), (8, 15), (8, 23)]
MODES = [(1, 0), (0, 0), (1, 1), (0, 1)]  # (rn, ftz)


# The default `-m gpu` run is sized for the driver's 20-minute step (~9 min on a
# B200); BFP_GPU_SUITE=full (or BFP_EXHAUSTIVE16=all) adds the longest sweeps.
# A full run is logged in profiles/r02_pytest_gpu_full_all.log (with BFP_EXHAUSTIVE16=all too: 424 passed, 34 min).
import os as _os  # noqa: E402

FULL_GPU_SUITE = _os.environ.get("BFP_GPU_SUITE") == "full" or _os.environ.get("BFP_EXHAUSTIVE16") == "all"
full_suite_only = pytest.mark.skipif(
    not FULL_GPU_SUITE, reason="set BFP_GPU_SUITE=full (full run logged in profiles/r02_pytest_gpu_full_all.log)")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity sweep")


def _cuda_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def oracle():
    O.orc()
    return O


@pytest.fixture(scope="session")
def ref_oracle():
    if not O.ref_available():
        try:
            O.build(ref=True)
        except Exception:
            pass
    if not O.ref_available():
        pytest.skip("reference build (oracle/_ref) unavailable on this host")
    O.ref()
    return O


class HostCircuits:
    """The device networks compiled for the host (tests/native)."""

    def __init__(self):
        native = ROOT / "tests" / "native"
        if not (ROOT / "paper_1602_04716_b200" / "csrc" / "gen" / "gen_8_23.cuh").exists():
            from paper_1602_04716_b200.build import generate
            generate(verbose=False)
        subprocess.run(["make", "-s", "-C", str(native)], check=True)
        L = C.CDLL(str(native / "libhostcirc.so"))
        vp = C.c_void_p
        L.host_binop.argtypes = [C.c_int, C.c_uint, C.c_uint, C.c_int, C.c_int, vp, vp, vp, vp, C.c_size_t]
        L.host_codec.argtypes = [C.c_int, C.c_uint, C.c_uint, C.c_int, C.c_int, vp, vp, C.c_size_t]
        L.host_codec64.argtypes = [C.c_int, C.c_uint, C.c_uint, C.c_int, C.c_int, vp, vp, C.c_size_t]
        L.host_pack_enc.argtypes = [C.c_int, C.c_uint, vp, C.c_size_t, vp]
        L.host_unpack_enc.argtypes = [C.c_int, C.c_uint, vp, C.c_size_t, vp]
        self.L = L

    def binop(self, op: str, fmt, px, py, pc=None, generated: bool = False):
        code = {"add": 0, "sub": 1, "mul": 2, "div": 3, "mul_add": 4, "mul_add_fast": 5,
                "mul_add_domain": 6}[op] + (10 if generated else 0)
        nb = 1 + fmt[0] + fmt[1]
        z = np.zeros_like(px)
        rc = self.L.host_binop(code, fmt[0], fmt[1], fmt[2], fmt[3], px.ctypes.data, py.ctypes.data,
                               pc.ctypes.data if pc is not None else None, z.ctypes.data,
                               len(px) // (nb * 32))
        assert rc == 0
        return z

    def codec(self, direction: int, fmt, vals: np.ndarray) -> np.ndarray:
        vals = np.ascontiguousarray(vals, dtype=np.uint32)
        out = np.zeros_like(vals)
        rc = self.L.host_codec(direction, fmt[0], fmt[1], fmt[2], fmt[3], vals.ctypes.data,
                               out.ctypes.data, len(vals))
        assert rc == 0
        return out

    def codec64(self, direction: int, fmt, vals: np.ndarray) -> np.ndarray:
        vals = np.ascontiguousarray(vals, dtype=np.uint64)
        out = np.zeros_like(vals)
        assert self.L.host_codec64(direction, fmt[0], fmt[1], fmt[2], fmt[3], vals.ctypes.data,
                                   out.ctypes.data, len(vals)) == 0
        return out

    def pack_enc(self, eb: int, nbits: int, enc: np.ndarray) -> np.ndarray:
        """eb-byte little-endian records (eb = 1..8) -> planes."""
        raw = np.ascontiguousarray(enc.astype(np.uint64)).view(np.uint8).reshape(-1, 8)[:, :eb].copy()
        planes = np.zeros(O.nblocks(len(enc)) * nbits * 32, dtype=np.uint32)
        self.L.host_pack_enc(eb, nbits, raw.ctypes.data, len(enc), planes.ctypes.data)
        return planes

    def unpack_enc(self, eb: int, nbits: int, planes: np.ndarray, n: int) -> np.ndarray:
        raw = np.zeros((n, 8), dtype=np.uint8)
        buf = np.zeros(n * eb, dtype=np.uint8)
        self.L.host_unpack_enc(eb, nbits, np.ascontiguousarray(planes).ctypes.data, n, buf.ctypes.data)
        raw[:, :eb] = buf.reshape(n, eb)
        return raw.view(np.uint64).reshape(n)


@pytest.fixture(scope="session")
def host():
    return HostCircuits()


# ----------------------------------------------------------------- operands
def all_pairs(nb: int):
    n = 1 << nb
    x = np.repeat(np.arange(n, dtype=np.uint64), n)
    y = np.tile(np.arange(n, dtype=np.uint64), n)
    return x, y


def operands(e: int, s: int, n: int, rng: np.random.Generator) -> np.ndarray:
    """Random encodings with extra weight on zero/subnormal, near-overflow and
    special exponents (the places the circuits branch)."""
    nb = 1 + e + s
    v = rng.integers(0, 1 << nb, size=n, dtype=np.uint64)
    k = n // 4
    sg = rng.integers(0, 2, size=k, dtype=np.uint64) << np.uint64(e + s)
    fr = rng.integers(0, 1 << s, size=k, dtype=np.uint64)
    lo = rng.integers(0, 4, size=k, dtype=np.uint64)
    hi = ((1 << e) - 1 - rng.integers(0, 3, size=k)).astype(np.uint64)
    v[:k] = sg | (lo << np.uint64(s)) | fr
    v[k:2 * k] = sg | (hi << np.uint64(s)) | fr
    return v


def related(x: np.ndarray, e: int, s: int, rng: np.random.Generator) -> np.ndarray:
    """Operands close to x in magnitude (cancellation / tie cases)."""
    flip = rng.integers(0, 2, size=len(x), dtype=np.uint64) << np.uint64(e + s)
    d = rng.integers(0, 4, size=len(x), dtype=np.uint64)
    mask = np.uint64((1 << (1 + e + s)) - 1)
    return (x ^ flip ^ d) & mask


# ------------------------------------------------- mul_add: the fast domain
def fast_domain(e: int, s: int, a, b, c) -> np.ndarray:
    """mul_add_fast_domain (csrc/bfp_circuits.cuh) restated on encodings, with
    ea, eb, ec the exponent fields and KN = clog2(s + 5):
    1 <= ea, eb < 3*2^(e-2);  2^(e-1) <= ea + eb <= 2^e + 2^(e-1) - 5;
    2^KN <= ec < 3*2^(e-2)."""
    kn = int(np.ceil(np.log2(s + 5)))
    ea, eb, ec = ((np.asarray(v, dtype=np.uint64) >> np.uint64(s)) & np.uint64((1 << e) - 1) for v in (a, b, c))
    cap = 3 << (e - 2)
    return ((ea != 0) & (eb != 0) & (ea < cap) & (eb < cap) & (ea + eb >= (1 << (e - 1)))
            & (ea + eb <= (1 << e) + (1 << (e - 1)) - 5) & (ec >= (1 << kn)) & (ec < cap))


def fast_domain_operands(O, fmt, n: int, rng: np.random.Generator):
    """(a, b, c), all n triples inside the fast domain, weighted towards its
    edges: exponent sums at both bounds, all-ones / zero fractions, c a few ulps
    from -(a*b) (massive cancellation) or at the ends of its exponent range."""
    e, s = fmt[:2]
    kn = int(np.ceil(np.log2(s + 5)))
    cap, lo, hi = 3 << (e - 2), 1 << (e - 1), (1 << e) + (1 << (e - 1)) - 5
    sign = np.uint64(1 << (e + s))

    def frac(k):
        f = rng.integers(0, 1 << s, size=k, dtype=np.uint64)
        edge = rng.integers(0, 8, size=k)
        f[edge == 0] = 0
        f[edge == 1] = (1 << s) - 1
        f[edge == 2] = 1
        return f

    ea = rng.integers(1, cap, size=n).astype(np.int64)
    lo_b = np.maximum(1, lo - ea)            # smallest / largest eb allowed beside ea
    hi_b = np.minimum(cap - 1, hi - ea)
    eb = lo_b + (rng.integers(0, 1 << 30, size=n) % (hi_b - lo_b + 1))
    k = rng.integers(0, 6, size=n)
    eb = np.where(k == 0, lo_b, np.where(k == 1, hi_b, np.where(k == 2, np.minimum(lo_b + 1, hi_b), eb)))
    ec = rng.integers(1 << kn, cap, size=n).astype(np.int64)
    k = rng.integers(0, 6, size=n)
    ec = np.where(k == 0, 1 << kn, np.where(k == 1, cap - 1, ec))
    a, b, c = ((rng.integers(0, 2, size=n, dtype=np.uint64) << np.uint64(e + s)) | (x.astype(np.uint64) << np.uint64(s))
               | frac(n) for x in (ea, eb, ec))
    # a quarter: c = -(a*b) +- a few ulps where that stays inside the domain
    q = n // 4
    p = (O.binop("mul", fmt, a[:q], b[:q]) ^ sign) + rng.integers(0, 5, size=q, dtype=np.uint64) - np.uint64(2)
    p &= np.uint64((1 << (1 + e + s)) - 1)
    ok = fast_domain(e, s, a[:q], b[:q], p)
    c[:q] = np.where(ok, p, c[:q])
    assert fast_domain(e, s, a, b, c).all()
    return a, b, c
