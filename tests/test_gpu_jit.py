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

JIT_FORMATS = [(2, 1), (6, 3), (7, 20), (11, 20), (10, 40)]
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


@pytest.mark.parametrize("fmt2", [(2, 1), (6, 3), (7, 16)])
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


def test_jit_unsupported_layout():
    """Encodings wider than 32 bits have no device layout kernel: EUNSUPPORTED."""
    L = _lib.lib()
    f = _lib.BfpFormat(10, 40, 1, 0, b"")
    t = torch.zeros(1 << 16, dtype=torch.int64, device="cuda")
    p = torch.zeros(1 << 16, dtype=torch.int32, device="cuda")
    assert L.bfp_pack_enc(C.byref(f), t.data_ptr(), p.data_ptr(), 100, None) == _lib.BFP_EUNSUPPORTED
