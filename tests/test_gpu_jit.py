"""Runtime-format backend: legal formats WITHOUT a
compiled network run the same templates JIT-compiled by NVRTC on first use.
Checked against the reference itself (oracle/_ref: exact for every width,
where the binary64 restatement is not)."""
from __future__ import annotations

import ctypes as C

import numpy as np
import pytest
import torch

from conftest import operands, related

import paper_1602_04716_b200 as bfp
from paper_1602_04716_b200 import _lib

pytestmark = pytest.mark.gpu

JIT_FORMATS = [(2, 1), (6, 3), (7, 20), (11, 20), (10, 40), (2, 5), (3, 11), (2, 30)]  # last three: working exponent wider than E + 2
OPS = {"add": 0, "sub": 1, "mul": 2, "div": 3, "mul_add": 4}


def _arith(op, fmt, px, py, pc):
    L = _lib.lib()
    nb = 1 + fmt[0] + fmt[1]
    count = (len(px) // (nb * 32)) * 1024
    dev = lambda a: torch.from_numpy(a.view(np.int32)).cuda()  # noqa: E731
    dx, dy, dc = dev(px), dev(py), dev(pc)
    dz = torch.empty_like(dx)
    f = _lib.BfpFormat(fmt[0], fmt[1], fmt[2], fmt[3], b"")
    assert L.bfp_is_compiled(C.byref(f)) == 0
    rc = L.bfp_arith(OPS[op], C.byref(f), dx.data_ptr(), dy.data_ptr(), dc.data_ptr(), dz.data_ptr(),
                     count, torch.cuda.current_stream().cuda_stream)
    assert rc == 0, L.bfp_last_error()
    return dz.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("fmt2", JIT_FORMATS)
@pytest.mark.parametrize("mode", [(1, 0), (0, 1)])
def test_jit_arith_vs_reference(ref_oracle, fmt2, mode):
    O = ref_oracle
    e, s = fmt2
    fmt = fmt2 + mode
    nb = 1 + e + s
    rng = np.random.default_rng(nb * 3 + mode[0])
    n = 4096 if nb > 32 else 1 << 14
    if nb <= 12:
        x = np.repeat(np.arange(1 << nb, dtype=np.uint64), 1 << nb)[: n * 16]
        y = np.tile(np.arange(1 << nb, dtype=np.uint64), 1 << nb)[: n * 16]
        n = len(x)
    else:
        x, y = operands(e, s, n, rng), operands(e, s, n, rng)
        y[: n // 8] = related(x[: n // 8], e, s, rng)
    c = operands(e, s, n, rng)
    px, py, pc = (O.pack_planes(v, nb) for v in (x, y, c))
    for op in OPS:
        got = _arith(op, fmt, px, py, pc)
        want = O.ref_binop_planes(op, fmt, px, py, pc if op == "mul_add" else None)
        assert np.array_equal(got, want), (op, fmt)


@pytest.mark.parametrize("fmt2", [(6, 3), (7, 20), (11, 20), (10, 40)])
@pytest.mark.parametrize("mode", [(1, 0), (0, 1)])
def test_jit_mul_add_fast_domain(ref_oracle, oracle, fmt2, mode):
    """Runtime formats run mul_add's fast-domain TEMPLATE on blocks inside the
    domain (csrc/bfp_kernels.cuh, has_fast_cover): operands generated inside it,
    every other block with one element outside, and the general network forced
    -- all equal the reference's bfp_add(bfp_mul(a, b), c)."""
    from conftest import fast_domain, fast_domain_operands
    e, s = fmt2
    fmt = fmt2 + mode
    nb = 1 + e + s
    rng = np.random.default_rng(900 + nb + mode[0])
    n = 1 << 13
    a, b, c = fast_domain_operands(oracle, fmt, n, rng)
    pos = np.arange(0, n // 1024, 2) * 1024 + rng.integers(0, 1024, size=n // 2048)
    a[pos[0::2]] = 0
    c[pos[1::2]] &= np.uint64((1 << s) - 1)
    assert fast_domain(e, s, a, b, c).reshape(-1, 1024).all(axis=1).sum() == n // 2048
    pa, pb, pc = (ref_oracle.pack_planes(v, nb) for v in (a, b, c))
    want = ref_oracle.ref_binop_planes("mul_add", fmt, pa, pb, pc)
    L = _lib.lib()
    f = _lib.BfpFormat(e, s, mode[0], mode[1], b"")
    da, db, dc = (torch.from_numpy(p.view(np.int32)).cuda() for p in (pa, pb, pc))
    for flags in (0, 2):
        dz = torch.empty_like(da)
        assert L.bfp_arith_ex(4, C.byref(f), da.data_ptr(), db.data_ptr(), dc.data_ptr(), dz.data_ptr(), n,
                              torch.cuda.current_stream().cuda_stream, flags) == 0, L.bfp_last_error()
        assert np.array_equal(dz.cpu().numpy().view(np.uint32), want), (fmt, flags)


@pytest.mark.parametrize("fmt2", [(2, 1), (6, 3), (7, 16), (2, 5), (3, 11), (2, 20), (4, 22)])
def test_jit_codec(oracle, fmt2):
    e, s = fmt2
    nb = 1 + e + s
    for mode in [(1, 0), (0, 1)]:
        spec = bfp.make_spec(e, s, *mode)
        rng = np.random.default_rng(nb)
        bits = rng.integers(0, 1 << 32, size=70001, dtype=np.uint64).astype(np.uint32)
        bits[:35000] = (bits[:35000] & 0x807FFFFF) | (
            rng.integers(100, 160, size=35000, dtype=np.uint64).astype(np.uint32) << 23)
        xs = bits.view(np.float32)
        v = bfp.pack_f32(torch.from_numpy(xs).cuda(), spec)
        want = oracle.encode_f32(fmt2 + mode, xs)
        assert np.array_equal(v.planes.cpu().numpy().view(np.uint32), oracle.pack_planes(want, nb))
        got = bfp.to_u64(bfp.unpack(v), spec).cpu().numpy().astype(np.uint64)
        assert np.array_equal(got, want)
        back = bfp.unpack_f32(v).cpu().numpy().view(np.uint32)
        assert np.array_equal(back, oracle.decode_f32(fmt2 + mode, want).view(np.uint32))


def test_jit_unsupported_f32_codec():
    """float32 conversion needs e <= 8, s <= 23: EUNSUPPORTED beyond (binary64 works)."""
    L = _lib.lib()
    f = _lib.BfpFormat(10, 40, 1, 0, b"")
    t = torch.zeros(1 << 16, dtype=torch.float32, device="cuda")
    p = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")
    assert L.bfp_pack_f32(C.byref(f), t.data_ptr(), p.data_ptr(), 100, None) == _lib.BFP_EUNSUPPORTED


WIDE = [(7, 30), (9, 35), (10, 40), (11, 52), (6, 3), (8, 23)]  # n = 38, 45, 51, 64, 10, 32


@pytest.mark.parametrize("fmt2", WIDE)
def test_wide_layout_and_bfpraw(ref_oracle, fmt2):
    """64-bit encodings and .bfpraw strides 5..8 through the layout kernels
    (JIT for the uncompiled formats) against field_from_elements and the
    reference's own to_bfpraw."""
    O = ref_oracle
    e, s = fmt2
    nb = 1 + e + s
    spec = bfp.make_spec(e, s)
    stride = bfp.bfpraw_stride(spec)
    rng = np.random.default_rng(nb)
    n = 3000
    enc = rng.integers(0, 1 << min(nb, 63), size=n, dtype=np.uint64)
    if nb == 64:
        enc = enc * np.uint64(2) + rng.integers(0, 2, size=n, dtype=np.uint64)
    t = torch.from_numpy(enc.view(np.int64).copy()).cuda()
    v = bfp.pack(t, spec)
    assert np.array_equal(v.planes.cpu().numpy().view(np.uint32), O.pack_planes(enc, nb))
    assert np.array_equal(bfp.to_u64(bfp.unpack(v), spec).cpu().numpy().view(np.uint64), enc)
    raw = np.zeros(n * stride, dtype=np.uint8)
    O.ref().ref_to_bfpraw(enc.ctypes.data_as(O._u64p), n, raw.ctypes.data_as(O._u8p), e, s)
    vr = bfp.pack_bfpraw(torch.from_numpy(raw).cuda(), spec)
    assert np.array_equal(vr.planes.cpu().numpy().view(np.uint32), O.pack_planes(enc, nb))
    assert np.array_equal(bfp.unpack_bfpraw(vr).cpu().numpy(), raw)


@pytest.mark.parametrize("fmt2", [(11, 52), (10, 40)])
def test_host_pipeline_wide_formats(ref_oracle, fmt2):
    """Host-buffer pipeline on formats wider than 32 planes (up to 8 KiB per
    block), over more chunks than buffer slots: each chunk must fit the
    context's staging buffers (sized for 32 planes / float32 per block), so
    a wide format runs fewer blocks per chunk.  The result equals the device
    path over the same planes and the reference on both ends."""
    O = ref_oracle
    L = _lib.lib()
    e, s = fmt2
    nb = 1 + e + s
    fmt = (e, s, 1, 0)
    chunk = 1 << 19
    n = 9 * chunk + 77  # > 8 chunks of the context, ragged tail
    rng = np.random.default_rng(nb)
    x, y = operands(e, s, n, rng), operands(e, s, n, rng)
    px, py = O.pack_planes(x, nb), O.pack_planes(y, nb)
    f = _lib.BfpFormat(e, s, 1, 0, b"")
    ctx = L.bfp_host_ctx_create(chunk)
    assert ctx
    outs = [np.zeros_like(px) for _ in range(2)]
    try:
        arr = (C.c_int * 2)(2, 0)
        zp = (C.c_void_p * 2)(*[o.ctypes.data for o in outs])
        assert L.bfp_arith_host_batch(ctx, 2, arr, C.byref(f), px.ctypes.data, py.ctypes.data, None,
                                      zp, n) == 0, L.bfp_last_error()
    finally:
        L.bfp_host_ctx_destroy(ctx)
    for o, op in zip(outs, ("mul", "add")):
        assert np.array_equal(o, _arith(op, fmt, px, py, px)), op
        k = 4096
        for lo in (0, n - k):  # the reference itself on the first / last blocks
            blo = lo // 1024
            pxs = px[blo * nb * 32:(blo + O.nblocks(k)) * nb * 32]
            pys = py[blo * nb * 32:(blo + O.nblocks(k)) * nb * 32]
            want = O.ref_binop_planes(op, fmt, pxs, pys, None)
            assert np.array_equal(o[blo * nb * 32:blo * nb * 32 + len(want)], want), (op, lo)


@pytest.mark.parametrize("fmt2", [(4, 3), (5, 10), (8, 23), (7, 30), (11, 52), (2, 1), (2, 5), (3, 11), (2, 40)])
@pytest.mark.parametrize("mode", [(1, 0), (0, 1)])
def test_pack_unpack_f64(oracle, fmt2, mode):
    """binary64 -> encode_scalar -> planes and planes -> decode_scalar (exact
    binary64), compiled and JIT formats, against the C restatement."""
    e, s = fmt2
    fmt = fmt2 + mode
    nb = 1 + e + s
    spec = bfp.make_spec(e, s, mode[0], mode[1])
    rng = np.random.default_rng(nb * 7 + mode[0])
    n = 40000 + 123
    bits = rng.integers(0, 1 << 63, size=n, dtype=np.uint64) * np.uint64(2) + \
        rng.integers(0, 2, size=n, dtype=np.uint64)
    ex = rng.integers(1023 - 1100, 1023 + 1100, size=n // 2).clip(0, 2047).astype(np.uint64)
    bits[: n // 2] = (bits[: n // 2] & np.uint64(0x800FFFFFFFFFFFFF)) | (ex << np.uint64(52))
    xs = bits.view(np.float64)
    v = bfp.pack_f64(torch.from_numpy(xs.copy()).cuda(), spec)
    want = oracle.encode_f64(fmt, xs)
    assert np.array_equal(v.planes.cpu().numpy().view(np.uint32), oracle.pack_planes(want, nb))
    back = bfp.unpack_f64(v).cpu().numpy()
    ref = oracle.decode_f64(fmt, want)
    nan = np.isnan(ref)
    assert np.array_equal(back.view(np.uint64)[~nan], ref.view(np.uint64)[~nan])
    assert np.all(back.view(np.uint64)[nan] == np.uint64(0x7FF8000000000000))


def test_jit_disk_cache(tmp_path):
    """NVRTC kernels are cached as CUBIN files: a second process loads them
    instead of compiling, with the same results."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    code = ("import torch, numpy as np, paper_1602_04716_b200 as bfp\n"
            "spec = bfp.make_spec(7, 20)\n"
            "v = [bfp.pack(torch.arange(5000, dtype=torch.int64, device='cuda') * k + 12345, spec) for k in (3, 7)]\n"
            "z = bfp.chain('ab*ab+-', *v)\n"
            "print(int(z.planes.to(torch.int64).sum()))\n")
    env = dict(os.environ, BFP_JIT_CACHE=str(tmp_path), PYTHONPATH=str(ROOT))
    out = [subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
           for _ in range(2)]
    assert all(o.returncode == 0 for o in out), out[0].stderr + out[1].stderr
    assert out[0].stdout == out[1].stdout
    files = list(tmp_path.glob("*.cubin"))
    assert len(files) >= 2  # the pack kernel and the chain program
    mtimes = {f: f.stat().st_mtime_ns for f in files}
    out3 = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert out3.returncode == 0 and out3.stdout == out[0].stdout
    assert {f: f.stat().st_mtime_ns for f in tmp_path.glob("*.cubin")} == mtimes  # loaded, not rewritten


@pytest.mark.slow
@pytest.mark.skipif(not __import__("os").environ.get("BFP_FUZZ_WIDE"), reason="set BFP_FUZZ_WIDE=<count>")
def test_jit_wide_format_fuzz(ref_oracle):
    """Random legal formats with wide significands (s in [20, 52], n <= 64),
    random modes, every op, against the reference templates themselves."""
    import os
    O = ref_oracle
    rng = np.random.default_rng(77)
    for t in range(int(os.environ["BFP_FUZZ_WIDE"])):
        e = int(rng.integers(2, 12))
        s = int(rng.integers(20, min(52, 63 - e) + 1))
        fmt = (e, s, int(rng.integers(2)), int(rng.integers(2)))
        nb = 1 + e + s
        n = 2048
        x, y, c = (operands(e, s, n, rng) for _ in range(3))
        y[: n // 8] = related(x[: n // 8], e, s, rng)
        px, py, pc = (O.pack_planes(v, nb) for v in (x, y, c))
        for op in OPS:
            got = _arith(op, fmt, px, py, pc)
            want = O.ref_binop_planes(op, fmt, px, py, pc if op == "mul_add" else None)
            assert np.array_equal(got, want), (t, op, fmt)


@pytest.mark.slow
@pytest.mark.skipif(not __import__("os").environ.get("BFP_FUZZ_LAYOUT"), reason="set BFP_FUZZ_LAYOUT=<count>")
def test_layout_fuzz(oracle):
    """Random legal formats (n <= 64), counts and buffer offsets through the
    layout paths: encodings -> planes (oracle pack_planes), planes ->
    encodings, .bfpraw bytes round trip, binary64 codec (oracle encode_f64 /
    decode_f64) and, where e <= 8 and s <= 23, the float32 codec."""
    import os
    rng = np.random.default_rng(99)
    for t in range(int(os.environ["BFP_FUZZ_LAYOUT"])):
        e = int(rng.integers(2, 12))
        s = int(rng.integers(1, min(52, 63 - e) + 1))
        mode = (int(rng.integers(2)), int(rng.integers(2)))
        fmt = (e, s) + mode
        nb = 1 + e + s
        spec = bfp.make_spec(e, s, *mode)
        n = int(rng.integers(1, 6000))
        enc = operands(e, s, n, rng)
        v = bfp.pack(torch.from_numpy(enc.astype(np.int64)).cuda(), spec)
        assert np.array_equal(v.planes.cpu().numpy().view(np.uint32), oracle.pack_planes(enc, nb)), (t, fmt)
        assert np.array_equal(bfp.to_u64(bfp.unpack(v), spec).cpu().numpy().astype(np.uint64), enc), (t, fmt)
        stride = bfp.bfpraw_stride(spec)
        off = int(rng.integers(0, 16))  # unaligned byte view
        raw_buf = torch.zeros(n * stride + 16, dtype=torch.uint8, device="cuda")
        raw = raw_buf[off: off + n * stride]
        raw.copy_(bfp.unpack_bfpraw(v))
        assert torch.equal(bfp.pack_bfpraw(raw, spec).planes, v.planes), (t, fmt, "bfpraw")
        xs = (rng.standard_normal(n) * float(2.0 ** float(rng.integers(-40, 41)))).astype(np.float64)
        xs[: n // 10] = rng.choice([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-300, -5e-324], size=n // 10)
        v64 = bfp.pack_f64(torch.from_numpy(xs).cuda(), spec)
        want = oracle.encode_f64(fmt, xs)
        assert np.array_equal(bfp.to_u64(bfp.unpack(v64), spec).cpu().numpy().astype(np.uint64), want), (t, fmt, "f64")
        back = bfp.unpack_f64(v64).cpu().numpy().view(np.uint64)
        assert np.array_equal(back, oracle.decode_f64(fmt, want).view(np.uint64)), (t, fmt, "f64 back")
        if e <= 8 and s <= 23:
            xf = xs.astype(np.float32)
            vf = bfp.pack_f32(torch.from_numpy(xf).cuda(), spec)
            wf = oracle.encode_f32(fmt, xf)
            assert np.array_equal(bfp.to_u64(bfp.unpack(vf), spec).cpu().numpy().astype(np.uint64), wf), (t, fmt, "f32")
            bf = bfp.unpack_f32(vf).cpu().numpy().view(np.uint32)
            assert np.array_equal(bf, oracle.decode_f32(fmt, wf).view(np.uint32)), (t, fmt, "f32 back")


@__import__("conftest").full_suite_only
def test_jit_runtime_covers(tmp_path, ref_oracle):
    """BFP_JIT_MAP=1: a runtime format gets LOP3-mapped covers generated on
    first use (tools/lutmap, GEN_ONE mode) -- same bits as the reference."""
    import os
    import subprocess
    import sys
    from conftest import ROOT
    code = (
        "import sys, numpy as np, torch, ctypes as C\n"
        "sys.path.insert(0, 'tests'); sys.path.insert(0, 'oracle')\n"
        "import oracle as O\n"
        "from conftest import operands\n"
        "from paper_1602_04716_b200 import _lib\n"
        "L = _lib.lib()\n"
        "rng = np.random.default_rng(5)\n"
        "for fmt in [(3, 11, 1, 0), (7, 20, 0, 1)]:\n"
        "    e, s = fmt[:2]; nb = 1 + e + s; n = 1 << 13\n"
        "    x, y, c = (operands(e, s, n, rng) for _ in range(3))\n"
        "    px, py, pc = (O.pack_planes(v, nb) for v in (x, y, c))\n"
        "    f = _lib.BfpFormat(*fmt, b'')\n"
        "    for op, name in enumerate(['add', 'sub', 'mul', 'div', 'mul_add']):\n"
        "        dx, dy, dc = (torch.from_numpy(a.view(np.int32)).cuda() for a in (px, py, pc))\n"
        "        dz = torch.empty_like(dx)\n"
        "        assert L.bfp_arith(op, C.byref(f), dx.data_ptr(), dy.data_ptr(), dc.data_ptr(), dz.data_ptr(),\n"
        "                           n, None) == 0\n"
        "        want = O.ref_binop_planes(name, fmt, px, py, pc if name == 'mul_add' else None)\n"
        "        assert np.array_equal(dz.cpu().numpy().view(np.uint32), want), (fmt, name)\n"
        "print('ok')\n")
    env = dict(os.environ, BFP_JIT_CACHE=str(tmp_path), BFP_JIT_MAP="1", PYTHONPATH=str(ROOT))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
    hdrs = sorted(p.name for p in (tmp_path / "gen").glob("*.cuh"))
    assert hdrs == ["gen_3_11_1_0.cuh", "gen_7_20_0_1.cuh"], hdrs
