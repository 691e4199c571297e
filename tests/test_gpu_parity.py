"""Parity of the B200 kernels, called through the C ABI (libbfpgpu.so), with
the oracle -- bit-exact, since all of this is integer/bit work.

  * arithmetic: exhaustive for every <= 9-bit format (all modes, add / sub /
    mul / mul_add), all 2^26 pairs of 1/5/7, every x against sampled y for the
    16-bit formats, seeded random + directed operands for 24 / 32-bit;
  * the golden fixtures written by the reference itself;
  * layout: pack / unpack of raw encodings and of float32 against
    field_from_elements / element_of + encode_scalar / decode_scalar, with
    ragged counts and unaligned buffers;
  * BASELINE configs at full size: C1 and C2 fully against the oracle, C3-C5
    through size-independent properties plus sampled oracle checks.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from conftest import FORMATS, MODES, ROOT, all_pairs, fast_domain, fast_domain_operands, operands, related

import paper_1602_04716_b200 as bfp
from paper_1602_04716_b200 import _lib, workloads as W

pytestmark = pytest.mark.gpu
GOLDEN = ROOT / "tests" / "golden"
OPS = {"add": 0, "sub": 1, "mul": 2, "div": 3, "mul_add": 4}


def dev(a: np.ndarray) -> torch.Tensor:
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a).cuda()


def cfmt(fmt):
    return _lib.BfpFormat(fmt[0], fmt[1], fmt[2], fmt[3], b"")


def gpu_arith(op: str, fmt, px, py, pc=None, flags: int = 0) -> np.ndarray:
    L = _lib.lib()
    nb = 1 + fmt[0] + fmt[1]
    count = (len(px) // (nb * 32)) * 1024
    dx, dy = dev(px), dev(py)
    dc = dev(pc) if pc is not None else None
    dz = torch.empty_like(dx)
    f = cfmt(fmt)
    rc = L.bfp_arith_ex(OPS[op], C.byref(f), dx.data_ptr(), dy.data_ptr(),
                        dc.data_ptr() if dc is not None else None, dz.data_ptr(), count,
                        torch.cuda.current_stream().cuda_stream, flags)
    assert rc == 0, _lib.lib().bfp_last_error()
    return dz.cpu().numpy().view(np.uint32)


def fast_blocks(fmt, pa, pb, pc) -> int:
    """bfp_mul_add_fast_blocks: blocks of the call that run the fast-domain cover."""
    nb = 1 + fmt[0] + fmt[1]
    count = (len(pa) // (nb * 32)) * 1024
    da, db, dc = dev(pa), dev(pb), dev(pc)
    out = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    f = cfmt(fmt)
    rc = _lib.lib().bfp_mul_add_fast_blocks(C.byref(f), da.data_ptr(), db.data_ptr(), dc.data_ptr(), count,
                                            out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert rc == 0, _lib.lib().bfp_last_error()
    return int(out.item())


def check(O, op, fmt, x, y, c=None):
    nb = 1 + fmt[0] + fmt[1]
    px, py = O.pack_planes(x, nb), O.pack_planes(y, nb)
    pc = O.pack_planes(c, nb) if c is not None else None
    got = O.unpack_planes(gpu_arith(op, fmt, px, py, pc), len(x), nb)
    want = O.binop(op, fmt, x, y, c)
    bad = np.nonzero(want != got)[0]
    assert len(bad) == 0, (op, fmt, len(bad), [(hex(int(x[i])), hex(int(y[i])), hex(int(want[i])),
                                                hex(int(got[i]))) for i in bad[:5]])


# ------------------------------------------------------------------ arithmetic
@pytest.mark.parametrize("fmt2", [(3, 2), (4, 3), (5, 3)])
@pytest.mark.parametrize("mode", MODES)
def test_exhaustive_small(oracle, fmt2, mode):
    e, s = fmt2
    x, y = all_pairs(1 + e + s)
    rng = np.random.default_rng(e + s)
    c = rng.integers(0, 1 << (1 + e + s), size=len(x), dtype=np.uint64)
    for op in ("add", "sub", "mul", "div", "mul_add"):
        check(oracle, op, fmt2 + mode, x, y, c if op == "mul_add" else None)


@pytest.mark.parametrize("mode", [(1, 0), (0, 1)])
def test_exhaustive_13bit(oracle, mode):
    x, y = all_pairs(13)
    for op in ("add", "mul", "div"):
        check(oracle, op, (5, 7) + mode, x, y)


@pytest.mark.parametrize("fmt2", [(5, 10), (6, 9), (8, 7)])
def test_16bit_every_x(oracle, fmt2):
    """every 16-bit x against 48 sampled y (RN + gradual)."""
    rng = np.random.default_rng(fmt2[0])
    xs = np.arange(1 << 16, dtype=np.uint64)
    ys = operands(*fmt2, 48, rng)
    x = np.repeat(xs, len(ys))
    y = np.tile(ys, len(xs))
    for op in ("add", "sub", "mul", "div"):
        check(oracle, op, fmt2 + (1, 0), x, y)


@pytest.mark.parametrize("fmt2", [f for f in FORMATS if 1 + f[0] + f[1] > 9])
@pytest.mark.parametrize("mode", MODES)
def test_random_wide(oracle, fmt2, mode):
    e, s = fmt2
    rng = np.random.default_rng(1000 + e * 64 + s + 7 * mode[0] + 13 * mode[1])
    n = 1 << 18
    x = operands(e, s, n, rng)
    y = operands(e, s, n, rng)
    y[: n // 8] = related(x[: n // 8], e, s, rng)
    c = operands(e, s, n, rng)
    for op in ("add", "sub", "mul", "div", "mul_add"):
        check(oracle, op, fmt2 + mode, x, y, c if op == "mul_add" else None)


# mul_add kernels carry two covers (include/bfpgpu.h, BFP_GENERAL_NETWORK): a
# warp runs the fast-domain one when its whole 1024-element block is inside
# the domain.  Blocks wholly inside, blocks with one element outside, and the
# general cover forced on the same operands: all equal the oracle's chain.
FAST_FMTS = [f for f in FORMATS if f != (3, 2)]  # 1/3/2 has no fast cover (E = KN)


@pytest.mark.parametrize("fmt2", FAST_FMTS)
@pytest.mark.parametrize("mode", MODES)
def test_mul_add_fast_and_general_covers(oracle, fmt2, mode):
    fmt = fmt2 + mode
    e, s = fmt2
    nb = 1 + e + s
    rng = np.random.default_rng(4242 + e * 64 + s + 7 * mode[0] + 13 * mode[1])
    n = 1 << 19
    a, b, c = fast_domain_operands(oracle, fmt, n, rng)
    want = oracle.binop("mul_add", fmt, a, b, c)
    planes = [oracle.pack_planes(v, nb) for v in (a, b, c)]
    for flags in (0, 2):  # every block on the fast cover / the general cover forced
        got = oracle.unpack_planes(gpu_arith("mul_add", fmt, *planes, flags=flags), n, nb)
        assert np.array_equal(got, want), (fmt, flags, int((got != want).sum()))
    assert fast_blocks(fmt, *planes) == n // 1024  # the kernel's own predicate + vote: every warp
    # every other block gets ONE element outside the domain (a zero, a
    # subnormal a, a tiny c): those warps take the general cover
    a2, b2, c2 = a.copy(), b.copy(), c.copy()
    blk = np.arange(0, n // 1024, 2)
    pos = blk * 1024 + rng.integers(0, 1024, size=len(blk))
    kind = rng.integers(0, 5, size=len(blk))
    special = np.uint64(((1 << e) - 1) << s)
    a2[pos[kind == 0]] = 0
    a2[pos[kind == 1]] &= np.uint64((1 << s) - 1)
    c2[pos[kind == 2]] &= np.uint64((1 << s) - 1) | np.uint64(1 << (e + s))
    b2[pos[kind == 3]] |= special          # Inf / NaN
    c2[pos[kind == 4]] = special           # +Inf
    inside = fast_domain(e, s, a2, b2, c2).reshape(-1, 1024).all(axis=1)
    assert inside[1::2].all() and not inside[0::2].any()
    want2 = oracle.binop("mul_add", fmt, a2, b2, c2)
    planes2 = [oracle.pack_planes(v, nb) for v in (a2, b2, c2)]
    got2 = oracle.unpack_planes(gpu_arith("mul_add", fmt, *planes2), n, nb)
    assert np.array_equal(got2, want2), (fmt, int((got2 != want2).sum()))
    assert fast_blocks(fmt, *planes2) == n // 2048
    # special-weighted random operands: the device count equals the restated predicate's
    x, y, z = (operands(e, s, 1 << 16, rng) for _ in range(3))
    x[: 1 << 15], y[: 1 << 15], z[: 1 << 15] = a[: 1 << 15], b[: 1 << 15], c[: 1 << 15]
    perm = rng.permutation(64)  # whole blocks shuffled
    x, y, z = (v.reshape(64, 1024)[perm].ravel() for v in (x, y, z))
    want_blocks = int(fast_domain(e, s, x, y, z).reshape(-1, 1024).all(axis=1).sum())
    assert 16 <= want_blocks < 64
    assert fast_blocks(fmt, *(oracle.pack_planes(v, nb) for v in (x, y, z))) == want_blocks


def test_fast_blocks_without_a_fast_cover(oracle):
    """1/3/2 has no fast-domain cover (E = KN): every block runs the general one."""
    rng = np.random.default_rng(3)
    planes = [oracle.pack_planes(rng.integers(0, 64, size=4096, dtype=np.uint64), 6) for _ in range(3)]
    assert fast_blocks((3, 2, 1, 0), *planes) == 0


@pytest.mark.parametrize("mode", MODES)
def test_mul_add_fast_cover_every_triple_1_4_3(oracle, mode):
    """Every (a, b, c) of 1/4/3 inside the fast domain, packed so that each
    block is wholly inside it: the fast cover over its entire domain."""
    fmt = (4, 3) + mode
    v = np.arange(1 << 8, dtype=np.uint64)
    a, b, c = (g.ravel() for g in np.meshgrid(v, v, v, indexing="ij"))
    keep = fast_domain(4, 3, a, b, c)
    a, b, c = a[keep], b[keep], c[keep]
    pad = -len(a) % 1024  # repeat the last triple: the tail block stays inside
    a, b, c = (np.concatenate([x, np.repeat(x[-1:], pad)]) for x in (a, b, c))
    assert len(a) >= 1 << 19
    want = oracle.binop("mul_add", fmt, a, b, c)
    got = oracle.unpack_planes(gpu_arith("mul_add", fmt, *(oracle.pack_planes(x, 8) for x in (a, b, c))), len(a), 8)
    assert np.array_equal(got, want), (fmt, int((got != want).sum()))


def test_golden_gpu(oracle):
    g = np.load(GOLDEN / "arith.npz")
    for (e, s) in FORMATS:
        nb = 1 + e + s
        for (rn, ftz) in MODES:
            key = f"{e}_{s}_{rn}_{ftz}"
            x, y, c = (g[f"{k}_{key}"].astype(np.uint64) for k in "xyc")
            px, py, pc = (oracle.pack_planes(v, nb) for v in (x, y, c))
            for op in ("add", "sub", "mul", "div", "mul_add"):
                z = gpu_arith(op, (e, s, rn, ftz), px, py, pc if op == "mul_add" else None)
                got = oracle.unpack_planes(z, len(x), nb)
                assert np.array_equal(got, g[f"{op}_{key}"].astype(np.uint64)), (op, key)


# ---------------------------------------------------------------------- layout
@pytest.mark.parametrize("fmt2", FORMATS)
def test_pack_unpack_enc(oracle, fmt2):
    e, s = fmt2
    nb = 1 + e + s
    spec = bfp.make_spec(e, s)
    rng = np.random.default_rng(nb)
    for n in (1, 31, 32, 33, 1000, 1024, 1025, 4096, 70001):
        enc = rng.integers(0, 1 << nb, size=n + 1, dtype=np.uint64)
        # offset view by one element: unaligned for the vector path
        for off in (0, 1):
            e_np = enc[off:off + n]
            t = torch.from_numpy(e_np.astype(np.int64)).cuda()
            v = bfp.pack(t, spec)
            planes = v.planes.cpu().numpy().view(np.uint32)
            assert np.array_equal(planes, oracle.pack_planes(e_np, nb)), (n, off)
            back = bfp.to_u64(bfp.unpack(v), spec).cpu().numpy().astype(np.uint64)
            assert np.array_equal(back, e_np), (n, off)


def test_unaligned_buffers(oracle):
    spec = bfp.make_spec(5, 10)
    nb = spec.total_bits()
    n = 5000
    rng = np.random.default_rng(9)
    enc = rng.integers(0, 1 << nb, size=n, dtype=np.uint64)
    buf = torch.zeros(n + 8, dtype=torch.int16, device="cuda")
    buf[1:n + 1] = torch.from_numpy(enc.astype(np.uint16).view(np.int16)).cuda()
    sub = buf[1:n + 1]  # 2-byte aligned only
    v = bfp.pack(sub, spec)
    assert np.array_equal(v.planes.cpu().numpy().view(np.uint32), oracle.pack_planes(enc, nb))
    out = torch.zeros(n + 8, dtype=torch.int16, device="cuda")
    L = _lib.lib()
    rc = L.bfp_unpack_enc(spec.c, v.planes.data_ptr(), out[1:].data_ptr(), n,
                          torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    assert np.array_equal(out[1:n + 1].cpu().numpy().view(np.uint16).astype(np.uint64), enc)


@pytest.mark.parametrize("fmt2", FORMATS)
@pytest.mark.parametrize("mode", MODES)
def test_pack_unpack_f32(oracle, fmt2, mode):
    e, s = fmt2
    nb = 1 + e + s
    fmt = fmt2 + mode
    spec = bfp.make_spec(e, s, mode[0], mode[1])
    rng = np.random.default_rng(nb * 4 + mode[0] * 2 + mode[1])
    n = (1 << 16) + 77
    bits = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
    bits[: n // 2] = (bits[: n // 2] & 0x807FFFFF) | (
        rng.integers(90, 165, size=n // 2, dtype=np.uint64).astype(np.uint32) << 23)
    xs = bits.view(np.float32)
    v = bfp.pack_f32(torch.from_numpy(xs).cuda(), spec)
    want = oracle.encode_f32(fmt, xs)
    assert np.array_equal(v.planes.cpu().numpy().view(np.uint32), oracle.pack_planes(want, nb))
    back = bfp.unpack_f32(v).cpu().numpy().view(np.uint32)
    assert np.array_equal(back, oracle.decode_f32(fmt, want).view(np.uint32))
    if nb <= 16:  # every encoding through unpack_f32
        encs = np.arange(1 << nb, dtype=np.uint64)
        ve = bfp.pack(torch.from_numpy(encs.astype(np.int64)).cuda(), spec)
        got = bfp.unpack_f32(ve).cpu().numpy().view(np.uint32)
        assert np.array_equal(got, oracle.decode_f32(fmt, encs).view(np.uint32))


def test_codec_golden_gpu():
    g = np.load(GOLDEN / "codec.npz")
    for (e, s) in FORMATS:
        nb = 1 + e + s
        for (rn, ftz) in MODES:
            key = f"{e}_{s}_{rn}_{ftz}"
            spec = bfp.make_spec(e, s, rn, ftz)
            xs = g[f"f32in_{key}"].view(np.float32)
            v = bfp.pack_f32(torch.from_numpy(xs.copy()).cuda(), spec)
            got = bfp.to_u64(bfp.unpack(v), spec).cpu().numpy()
            assert np.array_equal(got.astype(np.uint32), g[f"enc_{key}"]), key
            ve = bfp.pack(torch.from_numpy(g[f"decin_{key}"].astype(np.int64)).cuda(), spec)
            assert np.array_equal(bfp.unpack_f32(ve).cpu().numpy().view(np.uint32), g[f"dec_{key}"])


# ------------------------------------------------------------ API / errors
def test_python_api_roundtrip(oracle):
    spec = bfp.make_spec(4, 3)
    x = torch.linspace(-20, 20, 3000, device="cuda")
    y = torch.linspace(7, -3, 3000, device="cuda")
    vx, vy = bfp.pack_f32(x, spec), bfp.pack_f32(y, spec)
    ex = oracle.encode_f32((4, 3, 1, 0), x.cpu().numpy())
    ey = oracle.encode_f32((4, 3, 1, 0), y.cpu().numpy())
    for fn, op in ((bfp.bfp_add, "add"), (bfp.bfp_sub, "sub"), (bfp.bfp_mul, "mul")):
        z = bfp.to_u64(bfp.unpack(fn(vx, vy)), spec).cpu().numpy().astype(np.uint64)
        assert np.array_equal(z, oracle.binop(op, (4, 3, 1, 0), ex, ey)), op
    with pytest.raises(ValueError):
        bfp.bfp_add(vx, bfp.pack_f32(y, bfp.make_spec(4, 3, name="other")))
    # out= must match the operands' spec, count and plane size (no OOB writes)
    good = bfp.empty(spec, 3000)
    assert bfp.bfp_mul(vx, vy, out=good) is good
    bad = [bfp.empty(bfp.make_spec(3, 2), 3000),                        # narrower format
           bfp.empty(spec, 1000),                                       # fewer elements
           bfp.bfp_vector(spec, good.planes[:good.planes.numel() // 2], 3000),  # short planes
           bfp.bfp_vector(spec, good.planes.cpu(), 3000)]               # host memory
    for out in bad:
        with pytest.raises(ValueError):
            bfp.bfp_mul(vx, vy, out=out)
        with pytest.raises(ValueError):
            bfp.chain("ab*", vx, vy, out=out)


def test_unsupported_and_errors():
    L = _lib.lib()
    t = torch.zeros(4096, dtype=torch.int32, device="cuda")
    f = _lib.BfpFormat(12, 20, 1, 0, b"")  # illegal (validate: e <= 11)
    assert L.bfp_add(C.byref(f), t.data_ptr(), t.data_ptr(), t.data_ptr(), 10, None) == _lib.BFP_EFORMAT
    f = _lib.BfpFormat(1, 3, 1, 0, b"")
    assert L.bfp_add(C.byref(f), t.data_ptr(), t.data_ptr(), t.data_ptr(), 10, None) == _lib.BFP_EFORMAT
    f = _lib.BfpFormat(4, 3, 1, 0, b"")
    assert L.bfp_add(C.byref(f), None, t.data_ptr(), t.data_ptr(), 10, None) == _lib.BFP_EARG
    assert L.bfp_add(C.byref(f), t.data_ptr(), t.data_ptr(), t.data_ptr(), 0, None) == _lib.BFP_OK


@pytest.mark.parametrize("chunk,n", [(1 << 20, 3 * (1 << 20) + 5000),  # ctx chunk binds
                                     (1 << 24, 9 * (1 << 20) + 123)])  # split into 8 ragged chunks
def test_host_pipeline_matches_device(oracle, chunk, n):
    L = _lib.lib()
    fmt = (5, 10, 1, 0)
    nb = 16
    rng = np.random.default_rng(4)
    x, y = operands(5, 10, n, rng), operands(5, 10, n, rng)
    px, py = oracle.pack_planes(x, nb), oracle.pack_planes(y, nb)
    pz = np.zeros_like(px)
    ctx = L.bfp_host_ctx_create(chunk)
    try:
        f = cfmt(fmt)
        rc = L.bfp_arith_host(ctx, 2, C.byref(f), px.ctypes.data, py.ctypes.data, None, pz.ctypes.data, n)
        assert rc == 0
        assert np.array_equal(oracle.unpack_planes(pz, n, nb), oracle.binop("mul", fmt, x, y))
        xs = (rng.standard_normal(n) * 100).astype(np.float32)
        pp = np.zeros_like(px)
        assert L.bfp_pack_f32_host(ctx, C.byref(f), xs.ctypes.data, pp.ctypes.data, n) == 0
        assert np.array_equal(pp, oracle.pack_planes(oracle.encode_f32(fmt, xs), nb))
        back = np.zeros(n, dtype=np.float32)
        assert L.bfp_unpack_f32_host(ctx, C.byref(f), pp.ctypes.data, back.ctypes.data, n) == 0
        assert np.array_equal(back.view(np.uint32),
                              oracle.decode_f32(fmt, oracle.encode_f32(fmt, xs)).view(np.uint32))
    finally:
        L.bfp_host_ctx_destroy(ctx)


# -------------------------------------------------------- BASELINE configs
def _enc_np(t: torch.Tensor, spec) -> np.ndarray:
    return bfp.to_u64(t, spec).cpu().numpy().astype(np.uint64)


def test_config1_full(oracle):
    """C1: 1/4/3 add, N=2^24, uniform [-16,16] -> encode_scalar -> planes."""
    spec = bfp.make_spec(4, 3)
    n = 1 << 24
    a = W.c1_floats(0, n, W.SEED_A)
    b = W.c1_floats(0, n, W.SEED_B)
    va, vb = bfp.pack_f32(a, spec), bfp.pack_f32(b, spec)
    z = bfp.bfp_add(va, vb)
    ea = oracle.encode_f32((4, 3, 1, 0), a.cpu().numpy())
    eb = oracle.encode_f32((4, 3, 1, 0), b.cpu().numpy())
    assert np.array_equal(_enc_np(bfp.unpack(va), spec), ea)
    assert np.array_equal(_enc_np(bfp.unpack(z), spec), oracle.binop("add", (4, 3, 1, 0), ea, eb))


def test_config2_full(oracle):
    """C2: 1/4/3 mul and sub, N=2^26 raw encodings incl. subnormals and 1% zeros."""
    spec = bfp.make_spec(4, 3)
    n = 1 << 26
    a = W.c2_encodings(0, n, W.SEED_A)
    b = W.c2_encodings(0, n, W.SEED_B)
    va, vb = bfp.pack(a, spec), bfp.pack(b, spec)
    ea, eb = a.cpu().numpy().astype(np.uint64), b.cpu().numpy().astype(np.uint64)
    for fn, op in ((bfp.bfp_mul, "mul"), (bfp.bfp_sub, "sub")):
        got = _enc_np(bfp.unpack(fn(va, vb)), spec)
        assert np.array_equal(got, oracle.binop(op, (4, 3, 1, 0), ea, eb)), op


def _sample_check(oracle, fmt, spec, ea_t, eb_t, z_t, op, k=1 << 20, ec_t=None):
    n = ea_t.numel()
    idx = torch.randint(0, n, (k,), device="cuda", generator=torch.Generator("cuda").manual_seed(5))
    ea, eb = _enc_np(ea_t[idx], spec), _enc_np(eb_t[idx], spec)
    ec = _enc_np(ec_t[idx], spec) if ec_t is not None else None
    assert np.array_equal(_enc_np(z_t[idx], spec), oracle.binop(op, fmt, ea, eb, ec)), op


@pytest.mark.slow
def test_config3_properties(oracle):
    """C3: 1/5/10, N=2^28: pack_f32 == IEEE binary16 RN (NaN-free input),
    add/mul commutative, x - y == x + (-y), unpack_f32(pack_f32(x)) exact on
    representable values; sampled oracle parity of every op."""
    spec = bfp.make_spec(5, 10)
    fmt = (5, 10, 1, 0)
    n = 1 << 28
    a = W.c3_floats(0, n, W.SEED_A)
    b = W.c3_floats(0, n, W.SEED_B)
    va, vb = bfp.pack_f32(a, spec), bfp.pack_f32(b, spec)
    ea, eb = bfp.unpack(va), bfp.unpack(vb)
    assert torch.equal(ea, a.to(torch.float16).view(torch.int16))
    s = bfp.bfp_add(va, vb)
    assert torch.equal(s.planes, bfp.bfp_add(vb, va).planes)
    m = bfp.bfp_mul(va, vb)
    assert torch.equal(m.planes, bfp.bfp_mul(vb, va).planes)
    d = bfp.bfp_sub(va, vb)
    nb = bfp.pack(eb ^ torch.tensor(-32768, dtype=torch.int16, device="cuda"), spec)
    assert torch.equal(d.planes, bfp.bfp_add(va, nb).planes)
    back = bfp.unpack_f32(va)
    assert torch.equal(back, a.to(torch.float16).to(torch.float32))
    _sample_check(oracle, fmt, spec, ea, eb, bfp.unpack(s), "add")
    _sample_check(oracle, fmt, spec, ea, eb, bfp.unpack(m), "mul")


@pytest.mark.slow
@pytest.mark.parametrize("fmt2", [(3, 2), (5, 3), (5, 7), (8, 7), (8, 15)])
def test_config4_sampled(oracle, fmt2):
    e, s = fmt2
    spec = bfp.make_spec(e, s)
    n = 1 << 26  # a quarter of the bench size keeps the test fast; same kernels
    a = W.c4_encodings(e, s, 0, n, W.SEED_A)
    b = W.c4_encodings(e, s, 0, n, W.SEED_B)
    va, vb = bfp.pack(a, spec), bfp.pack(b, spec)
    for fn, op in ((bfp.bfp_add, "add"), (bfp.bfp_mul, "mul")):
        z = fn(va, vb)
        _sample_check(oracle, fmt2 + (1, 0), spec, bfp.unpack(va), bfp.unpack(vb), bfp.unpack(z), op)


@pytest.mark.slow
def test_config5_shards(oracle):
    """C5: the fused 1/6/9 chain computed on 4 block-aligned shards
    concatenates to the unsharded result (no exchange step), with sampled
    oracle parity (the bench runs 2^32 / G per GPU)."""
    spec = bfp.make_spec(6, 9)
    n = (1 << 26) + 3 * 1024 + 17
    ops = [bfp.pack_f32(W.c5_floats(0, n, sd), spec) for sd in (W.SEED_A, W.SEED_B, W.SEED_C)]
    full = bfp.bfp_mul_add(*ops)
    parts = []
    for r in range(4):
        lo, hi = W.shard(n, r, 4)
        sh = [bfp.pack_f32(W.c5_floats(lo, hi, sd), spec) for sd in (W.SEED_A, W.SEED_B, W.SEED_C)]
        parts.append(bfp.bfp_mul_add(*sh).planes)
    assert torch.equal(torch.cat(parts), full.planes)
    ea, eb, ec = (bfp.unpack(v) for v in ops)
    _sample_check(oracle, (6, 9, 1, 0), spec, ea, eb, bfp.unpack(full), "mul_add", ec_t=ec)


def test_launch_counter():
    L = _lib.lib()
    before = L.bfp_launch_count()
    spec = bfp.make_spec(4, 3)
    v = bfp.pack(torch.arange(2048, device="cuda") % 256, spec)
    bfp.bfp_add(v, v)
    assert L.bfp_launch_count() == before + 2


@pytest.mark.slow
def test_pack_f32_all_binary32_1_5_10():
    """encode_scalar for 1/5/10 RN + gradual on ALL 2^32 float32 inputs (the
    hardware-cvt path) equals IEEE binary16 RN conversion (torch's own
    float -> half kernel); NaNs must be the canonical 0x7e00."""
    spec = bfp.make_spec(5, 10)
    chunk = 1 << 28
    nan_canon = torch.tensor(0x7E00, dtype=torch.int16, device="cuda")
    for lo in range(0, 1 << 32, chunk):
        bits = torch.arange(lo, lo + chunk, dtype=torch.int64, device="cuda").to(torch.int32)
        x = bits.view(torch.float32)
        got = bfp.unpack(bfp.pack_f32(x, spec))
        want = x.to(torch.float16).view(torch.int16)
        want = torch.where(torch.isnan(x), nan_canon, want)
        assert torch.equal(got, want), hex(lo)


@pytest.mark.slow
@pytest.mark.parametrize("fmt2", FORMATS)
@pytest.mark.parametrize("mode", MODES)
def test_pack_f32_strided_sweep(oracle, fmt2, mode):
    """every 4099th binary32 bit pattern (~1M inputs spanning all exponents,
    both signs, subnormals, Inf, NaN) through pack_f32 / unpack_f32."""
    e, s = fmt2
    spec = bfp.make_spec(e, s, mode[0], mode[1])
    fmt = fmt2 + mode
    bits = (np.arange(0, 1 << 32, 4099, dtype=np.uint64)).astype(np.uint32)
    xs = bits.view(np.float32)
    v = bfp.pack_f32(torch.from_numpy(xs).cuda(), spec)
    want = oracle.encode_f32(fmt, xs)
    got = bfp.to_u64(bfp.unpack(v), spec).cpu().numpy().astype(np.uint64)
    assert np.array_equal(got, want), int((got != want).sum())
    back = bfp.unpack_f32(v).cpu().numpy().view(np.uint32)
    assert np.array_equal(back, oracle.decode_f32(fmt, want).view(np.uint32))


@pytest.mark.parametrize("fmt2", [f for f in FORMATS if 1 + f[0] + f[1] <= 32])
def test_bfpraw_roundtrip_vs_reference(ref_oracle, fmt2):
    """.bfpraw bytes written by the reference's to_bfpraw (pack.hpp:86-95) ->
    pack_bfpraw == field_from_elements planes; unpack_bfpraw == the bytes."""
    O = ref_oracle
    e, s = fmt2
    nb = 1 + e + s
    spec = bfp.make_spec(e, s)
    stride = bfp.bfpraw_stride(spec)
    rng = np.random.default_rng(nb + 100)
    for n in (1, 33, 1024, 3001, 1 << 16):
        enc = rng.integers(0, 1 << nb, size=n, dtype=np.uint64)
        raw = np.zeros(n * stride, dtype=np.uint8)
        O.ref().ref_to_bfpraw(enc.ctypes.data_as(O._u64p), n, raw.ctypes.data_as(O._u8p), e, s)
        v = bfp.pack_bfpraw(torch.from_numpy(raw).cuda(), spec)
        assert np.array_equal(v.planes.cpu().numpy().view(np.uint32), O.pack_planes(enc, nb)), n
        back = bfp.unpack_bfpraw(v).cpu().numpy()
        assert np.array_equal(back, raw), n
    if stride > 1:  # from_bfpraw rejects a ragged byte count (pack.hpp:98-100)
        with pytest.raises(ValueError):
            bfp.pack_bfpraw(torch.zeros(stride * 10 + 1, dtype=torch.uint8, device="cuda"), spec)


@pytest.mark.parametrize("fmt2", [f for f in FORMATS if f[0] <= 8 and f[1] <= 23])
@pytest.mark.parametrize("mode", MODES)
def test_arith_f32_fused(oracle, fmt2, mode):
    """Fused float32-in/out ops == decode(op(encode(x), encode(y))) per the
    oracle, and == the unfused pack_f32 / op / unpack_f32 composition."""
    e, s = fmt2
    fmt = fmt2 + mode
    spec = bfp.make_spec(e, s, mode[0], mode[1])
    rng = np.random.default_rng(e * 31 + s + mode[0] * 7 + mode[1])
    n = (1 << 15) + 1234  # ragged tail
    def floats():
        bits = rng.integers(0, 1 << 32, size=n, dtype=np.uint64).astype(np.uint32)
        bits[: n // 2] = (bits[: n // 2] & 0x807FFFFF) | (
            rng.integers(110, 145, size=n // 2, dtype=np.uint64).astype(np.uint32) << 23)
        return bits.view(np.float32)
    xs, ys, cs = floats(), floats(), floats()
    ex, ey, ec = (oracle.encode_f32(fmt, v) for v in (xs, ys, cs))
    tx, ty, tc = (torch.from_numpy(v).cuda() for v in (xs, ys, cs))
    for op, code in (("add", 0), ("sub", 1), ("mul", 2), ("div", 3), ("mul_add", 4)):
        got = bfp.arith_f32(code, spec, tx, ty, tc if code == 4 else None).cpu().numpy().view(np.uint32)
        want = oracle.decode_f32(fmt, oracle.binop(op, fmt, ex, ey, ec)).view(np.uint32)
        assert np.array_equal(got, want), (op, int((got != want).sum()))


def test_arith_f32_unaligned():
    spec = bfp.make_spec(5, 10)
    n = 5000
    buf = torch.randn(3 * n + 3, device="cuda") * 50
    x, y, z = buf[1:n + 1], buf[n + 2:2 * n + 2], torch.empty(n + 1, device="cuda")[1:]
    L = _lib.lib()
    assert L.bfp_arith_f32(2, spec.c, x.data_ptr(), y.data_ptr(), None, z.data_ptr(), n,
                           torch.cuda.current_stream().cuda_stream) == 0
    ref = bfp.unpack_f32(bfp.bfp_mul(bfp.pack_f32(x, spec), bfp.pack_f32(y, spec)))
    assert torch.equal(z.view(torch.int32), ref.view(torch.int32))


def test_host_batch_matches_device(oracle):
    """bfp_arith_host_batch: several ops over one H2D of shared host operands."""
    L = _lib.lib()
    fmt = (4, 3, 1, 0)
    n = 5 * (1 << 20) + 777
    rng = np.random.default_rng(8)
    x, y = operands(4, 3, n, rng), operands(4, 3, n, rng)
    px, py = oracle.pack_planes(x, 8), oracle.pack_planes(y, 8)
    outs = [np.zeros_like(px) for _ in range(3)]
    ops = [2, 1, 3]
    ctx = L.bfp_host_ctx_create(1 << 24)  # the call splits itself into ragged chunks
    try:
        f = cfmt(fmt)
        arr = (C.c_int * 3)(*ops)
        ptrs = (C.c_void_p * 3)(*[o.ctypes.data for o in outs])
        assert L.bfp_arith_host_batch(ctx, 3, arr, C.byref(f), px.ctypes.data, py.ctypes.data, None,
                                      ptrs, n) == 0
    finally:
        L.bfp_host_ctx_destroy(ctx)
    for o, op in zip(outs, ("mul", "sub", "div")):
        assert np.array_equal(oracle.unpack_planes(o, n, 8), oracle.binop(op, fmt, x, y)), op


@pytest.mark.gpu
def test_host_mul_add_many_chunks(oracle):
    """Three-input host pipeline (mul_add) over more chunks than buffer slots:
    slot reuse is ordered by the k_done / out_done events."""
    L = _lib.lib()
    fmt = (6, 9, 1, 0)
    n = 11 * (1 << 19) + 4321
    rng = np.random.default_rng(12)
    a, b, c = (operands(6, 9, n, rng) for _ in range(3))
    pa, pb, pc = (oracle.pack_planes(v, 16) for v in (a, b, c))
    pz = np.zeros_like(pa)
    ctx = L.bfp_host_ctx_create(1 << 19)
    try:
        f = cfmt(fmt)
        assert L.bfp_arith_host(ctx, 4, C.byref(f), pa.ctypes.data, pb.ctypes.data, pc.ctypes.data,
                                pz.ctypes.data, n) == 0
    finally:
        L.bfp_host_ctx_destroy(ctx)
    assert np.array_equal(oracle.unpack_planes(pz, n, 16), oracle.binop("mul_add", fmt, a, b, c))


def _pinned_like(L, arr: np.ndarray):
    """A page-locked (mapped) copy of arr from bfp_host_alloc, viewed as numpy."""
    p = L.bfp_host_alloc(arr.nbytes)
    assert p
    view = np.ctypeslib.as_array((C.c_uint8 * arr.nbytes).from_address(p)).view(arr.dtype)
    view[:] = arr.reshape(-1)
    return p, view


def test_host_pipeline_pinned_outputs_written_in_place(oracle):
    """Outputs in mapped pinned memory are written by the kernels directly
    (no D2H stage); results equal the pageable-buffer path and the oracle."""
    L = _lib.lib()
    fmt = (5, 10, 1, 0)
    n = 7 * (1 << 19) + 999
    rng = np.random.default_rng(21)
    x, y = operands(5, 10, n, rng), operands(5, 10, n, rng)
    px, py = oracle.pack_planes(x, 16), oracle.pack_planes(y, 16)
    ptrs = []
    try:
        (hx, _), (hy, _) = _pinned_like(L, px), _pinned_like(L, py)
        outs = [_pinned_like(L, np.zeros_like(px)) for _ in range(2)]
        ptrs += [hx, hy] + [o[0] for o in outs]
        ctx = L.bfp_host_ctx_create(1 << 20)
        try:
            f = cfmt(fmt)
            arr = (C.c_int * 2)(2, 1)
            zp = (C.c_void_p * 2)(*[o[0] for o in outs])
            assert L.bfp_arith_host_batch(ctx, 2, arr, C.byref(f), hx, hy, None, zp, n) == 0
            for (_, v), op in zip(outs, ("mul", "sub")):
                assert np.array_equal(oracle.unpack_planes(v.copy(), n, 16), oracle.binop(op, fmt, x, y)), op
            xs = (rng.standard_normal(n) * 100).astype(np.float32)
            hxs, _ = _pinned_like(L, xs)
            hpp, vpp = _pinned_like(L, np.zeros_like(px))
            hback, vback = _pinned_like(L, np.zeros(n, dtype=np.float32))
            ptrs += [hxs, hpp, hback]
            assert L.bfp_pack_f32_host(ctx, C.byref(f), hxs, hpp, n) == 0
            assert np.array_equal(vpp, oracle.pack_planes(oracle.encode_f32(fmt, xs), 16))
            assert L.bfp_unpack_f32_host(ctx, C.byref(f), hpp, hback, n) == 0
            assert np.array_equal(vback.view(np.uint32),
                                  oracle.decode_f32(fmt, oracle.encode_f32(fmt, xs)).view(np.uint32))
        finally:
            L.bfp_host_ctx_destroy(ctx)
    finally:
        for p in ptrs:
            L.bfp_host_free(p)


@pytest.mark.parametrize("fmt2", [(5, 10), (8, 7)])
@pytest.mark.parametrize("mode", MODES)
def test_pack_f32_hw_path_underflow_boundary(oracle, fmt2, mode):
    """The hardware-cvt encoders (binary16 / bfloat16 layouts, every mode incl.
    FTZ = convert then flush subnormal results) around the subnormal range and
    the normal boundary: every 7th float32 of both signs over the exponents
    from 12 below the smallest subnormal to 2 above the smallest normal."""
    e, s = fmt2
    spec = bfp.make_spec(e, s, mode[0], mode[1])
    fmt = fmt2 + mode
    emin = 2 - (1 << (e - 1))  # unbiased exponent of the smallest normal
    lo_exp, hi_exp = max(0, 127 + emin - s - 12), 127 + emin + 2  # bfloat16: float32 subnormals
    man = np.arange(0, 1 << 23, 7, dtype=np.uint32)
    exps = np.arange(lo_exp, hi_exp + 1, dtype=np.uint32)
    bits = (exps[:, None] << 23 | man[None, :]).reshape(-1)
    bits = np.concatenate([bits, bits | np.uint32(0x80000000)])
    xs = bits.view(np.float32)
    v = bfp.pack_f32(torch.from_numpy(xs).cuda(), spec)
    want = oracle.encode_f32(fmt, xs)
    got = bfp.to_u64(bfp.unpack(v), spec).cpu().numpy().astype(np.uint64)
    assert np.array_equal(got, want), int((got != want).sum())


@pytest.mark.parametrize("fmt2", [(4, 3), (5, 10), (6, 9)])
def test_inputs_ready_flag_back_to_back(oracle, fmt2):
    """BFP_INPUTS_READY (loads before the PDL wait): back-to-back launches on
    one stream over resident operands give the same bits as the oracle."""
    e, s = fmt2
    nb = 1 + e + s
    fmt = fmt2 + (1, 0)
    spec = bfp.make_spec(e, s)
    rng = np.random.default_rng(31 + nb)
    n = (1 << 20) + 333
    xs = [operands(e, s, n, rng) for _ in range(3)]
    vs = [bfp.pack(torch.from_numpy(x.astype(np.int64)).cuda(), spec) for x in xs]
    outs = [bfp.empty(spec, n) for _ in range(6)]
    ops = [(0, "add"), (2, "mul"), (4, "mul_add"), (1, "sub"), (2, "mul"), (0, "add")]
    for k, (code, _) in enumerate(ops):  # no sync in between: PDL chains the kernels
        bfp.arith(code, vs[k % 3], vs[(k + 1) % 3], vs[(k + 2) % 3], out=outs[k], inputs_ready=True)
    torch.cuda.synchronize()
    for k, (code, name) in enumerate(ops):
        got = bfp.to_u64(bfp.unpack(outs[k]), spec).cpu().numpy().astype(np.uint64)
        want = oracle.binop(name, fmt, xs[k % 3], xs[(k + 1) % 3], xs[(k + 2) % 3])
        assert np.array_equal(got, want), name


@pytest.mark.parametrize("seed", range(6))
def test_host_pipeline_random_shapes(oracle, seed):
    """Host-buffer entry points over random counts, context chunk sizes, op
    batches and pageable / pinned buffers == the device-buffer calls."""
    L = _lib.lib()
    rng = np.random.default_rng(1000 + seed)
    (e, s) = [(4, 3), (5, 10), (6, 9), (3, 2)][seed % 4]
    nb = 1 + e + s
    fmt = (e, s, 1, 0)
    spec = bfp.make_spec(e, s)
    n = int(rng.integers(1, 3 << 20))
    chunk = int(1 << int(rng.integers(19, 23)))
    ops = [int(o) for o in rng.choice([0, 1, 2, 3], size=int(rng.integers(1, 4)), replace=False)]
    pinned = bool(seed % 2)
    x, y = operands(e, s, n, rng), operands(e, s, n, rng)
    px, py = oracle.pack_planes(x, nb), oracle.pack_planes(y, nb)
    ptrs = []
    try:
        if pinned:
            (hx, _), (hy, _) = _pinned_like(L, px), _pinned_like(L, py)
            outs = [_pinned_like(L, np.zeros_like(px)) for _ in ops]
            ptrs += [hx, hy] + [o[0] for o in outs]
            zp = [o[0] for o in outs]
            views = [o[1] for o in outs]
        else:
            hx, hy = px.ctypes.data, py.ctypes.data
            views = [np.zeros_like(px) for _ in ops]
            zp = [v.ctypes.data for v in views]
        ctx = L.bfp_host_ctx_create(chunk)
        try:
            arr = (C.c_int * len(ops))(*ops)
            outp = (C.c_void_p * len(ops))(*zp)
            assert L.bfp_arith_host_batch(ctx, len(ops), arr, C.byref(cfmt(fmt)), hx, hy, None, outp, n) == 0
        finally:
            L.bfp_host_ctx_destroy(ctx)
        vx, vy = (bfp.pack(torch.from_numpy(v.astype(np.int64)).cuda(), spec) for v in (x, y))
        for op, v in zip(ops, views):
            want = bfp.arith(op, vx, vy).planes.cpu().numpy().view(np.uint32)
            assert np.array_equal(np.asarray(v).view(np.uint32).reshape(-1), want.reshape(-1)), (op, n, chunk, pinned)
    finally:
        for p in ptrs:
            L.bfp_host_free(p)
