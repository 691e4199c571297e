"""Bit-exact parity at the BASELINE configs' full bench sizes, every element
against the oracle (the C restatement, pinned to the reference in
tests/test_oracle.py) on all host threads (orc_verify):

  * C5: 1/6/9 z = round(round(a*b) + c) over all 2^32 elements in ONE
    mul_add launch (the bench's launch size on one GPU), the three pack_f32
    operands too; then every block-aligned shard of G = 2, 4, 8 GPUs launched
    on its own equals the unsharded result;
  * C3: 1/5/10 pack_f32 of both operands, add, mul and unpack_f32 at 2^28;
  * C4: add and mul of every sweep format at 2^28;
  * the fused mul_add network (its own LOP3 cover, not the composition of the
    mul and add covers; both of them, the general and the fast-domain one):
    1/6/9 over (a, b) pairs for 36 c values (signed zeros, subnormals, 1, max
    finite, Inf, NaN, random, both ends of the fast domain's c range) -- every
    4th chunk of 1024 a values by default (2^30 pairs, RN + gradual: the
    default run fits the driver's 20-minute step); ALL 2^32 pairs, and RZ +
    FTZ too, with BFP_GPU_SUITE=full or BFP_EXHAUSTIVE16=all (~5 min each;
    logged in profiles/r02_pytest_gpu_full_all.log) -- and ALL 2^24 (a, b, c)
    triples of 1/4/3 and 2^18 of 1/3/2 in every mode.

Inputs are generated on the device by the bench's own generators
(workloads.py, torch ops -- not our kernels) and copied to the host for the
oracle; the results are compared as plane images (field_from_elements,
bitfield.hpp:33-52).  Log of a run: profiles/r02_fullsize.log.
"""
from __future__ import annotations

import os
import time

import numpy as np
import pytest
import torch

from conftest import FULL_GPU_SUITE

import paper_1602_04716_b200 as bfp
from paper_1602_04716_b200 import _lib, workloads as W

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
CHUNK = 1 << 26  # elements per host round trip


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _planes_slice(v: bfp.bfp_vector, lo: int, hi: int) -> torch.Tensor:
    nb = v.spec.total_bits()
    return v.planes[(lo // 1024) * nb * 32:((hi + 1023) // 1024) * nb * 32]


def _pack_f32_chunked(gen, n, spec):
    """Bench-style pack_f32 of gen(lo, hi) through the C ABI into one vector."""
    v = bfp.empty(spec, n)
    for lo in range(0, n, CHUNK):
        hi = min(n, lo + CHUNK)
        x = gen(lo, hi)
        sub = _planes_slice(v, lo, hi)
        assert _lib.lib().bfp_pack_f32(spec.c, x.data_ptr(), sub.data_ptr(), hi - lo, _stream()) == 0
    return v


def _check(oracle, op, fmt, ins, got, n, what):
    bad, i, g, w = oracle.verify(op, fmt, *ins, got, n)
    assert bad == 0, f"{what}: {bad} mismatches, first at {i}: got {g:#x} want {w:#x}"


def test_c5_full_2e32(oracle):
    spec = bfp.make_spec(6, 9)
    fmt = (6, 9, 1, 0)
    n = 1 << 32
    seeds = (W.SEED_A, W.SEED_B, W.SEED_C)
    t0 = time.time()
    ops = [_pack_f32_chunked(lambda lo, hi, sd=sd: W.c5_floats(lo, hi, sd), n, spec) for sd in seeds]
    z = bfp.bfp_mul_add(*ops)  # one launch over all 2^32 elements
    torch.cuda.synchronize()
    for lo in range(0, n, CHUNK):
        hi = min(n, lo + CHUNK)
        xs = [W.c5_floats(lo, hi, sd).cpu().numpy() for sd in seeds]
        for k, v in enumerate(ops):
            _check(oracle, "pack", fmt, (xs[k], None, None), _planes_slice(v, lo, hi).cpu().numpy(), hi - lo,
                   f"C5 pack_f32 operand {k} [{lo}, {hi})")
        _check(oracle, "mul_add", fmt, tuple(xs), _planes_slice(z, lo, hi).cpu().numpy(), hi - lo,
               f"C5 mul_add [{lo}, {hi})")
    # the bench's shards: each block-aligned range launched on its own
    for g in (2, 4, 8):
        zs = bfp.empty(spec, n)
        for r in range(g):
            lo, hi = W.shard(n, r, g)
            args = [_planes_slice(v, lo, hi).data_ptr() for v in ops]
            assert _lib.lib().bfp_mul_add(spec.c, *args, _planes_slice(zs, lo, hi).data_ptr(), hi - lo,
                                          _stream()) == 0
        assert torch.equal(zs.planes, z.planes), f"C5 shards of {g}"
        del zs
    print(f"C5: all 2^32 elements bit-exact vs the oracle (+ shards of 2/4/8), {time.time() - t0:.1f} s")


def test_c3_full_2e28(oracle):
    spec = bfp.make_spec(5, 10)
    fmt = (5, 10, 1, 0)
    n = 1 << 28
    xa, xb = W.c3_floats(0, n, W.SEED_A), W.c3_floats(0, n, W.SEED_B)
    va, vb = bfp.pack_f32(xa, spec), bfp.pack_f32(xb, spec)
    s, m, u = bfp.bfp_add(va, vb), bfp.bfp_mul(va, vb), bfp.unpack_f32(va)
    ha, hb = xa.cpu().numpy(), xb.cpu().numpy()
    del xa, xb
    _check(oracle, "pack", fmt, (ha, None, None), va.planes.cpu().numpy(), n, "C3 pack_f32 a")
    _check(oracle, "pack", fmt, (hb, None, None), vb.planes.cpu().numpy(), n, "C3 pack_f32 b")
    _check(oracle, "add", fmt, (ha, hb, None), s.planes.cpu().numpy(), n, "C3 add")
    _check(oracle, "mul", fmt, (ha, hb, None), m.planes.cpu().numpy(), n, "C3 mul")
    _check(oracle, "unpack_f32", fmt, (ha, None, None), u.cpu().numpy().view(np.uint32), n, "C3 unpack_f32")


@pytest.mark.parametrize("fmt2", [(3, 2), (5, 3), (5, 7), (8, 7), (8, 15)])
def test_c4_full_2e28(oracle, fmt2):
    e, s = fmt2
    spec = bfp.make_spec(e, s)
    fmt = fmt2 + (1, 0)
    n = 1 << 28
    a, b = W.c4_encodings(e, s, 0, n, W.SEED_A), W.c4_encodings(e, s, 0, n, W.SEED_B)
    va, vb = bfp.pack(a, spec), bfp.pack(b, spec)
    ha, hb = a.cpu().numpy().view(np.uint32), b.cpu().numpy().view(np.uint32)
    del a, b
    for fn, op in ((bfp.bfp_add, "add"), (bfp.bfp_mul, "mul")):
        _check(oracle, op, fmt, (ha, hb, None), fn(va, vb).planes.cpu().numpy(), n, f"C4 1/{e}/{s} {op}")


# c values for the all-pairs sweep of 1/6/9 (sign 15, exponent 9..14, fraction 0..8)
C_1_6_9 = [0x0000, 0x8000, 0x0001, 0x8001, 0x01FF, 0x81FF, 0x0200, 0x8200, 0x3E00, 0xBE00, 0x3E01, 0xBDFF,
           0x7DFF, 0xFDFF, 0x7C00, 0xFC01, 0x7E00, 0xFE00, 0x7F00, 0x7E01, 0xFF00, 0x0400, 0x0401, 0x2001,
           0x5A5A, 0xA5A5, 0x1234, 0x9876, 0x4321, 0xC0DE, 0x3FFF, 0x0100,
           # both ends of the fast domain's c range (exponent fields 16 and 47): with the 11 values above whose
           # field lies in [16, 48), every block of (a, b) inside the domain runs the fast-domain cover
           0x2000, 0xA1FF, 0x5FFF, 0xDE00]


MODES_PAIRS = [(1, 0), (0, 1)] if FULL_GPU_SUITE else [(1, 0)]


@pytest.mark.parametrize("mode", MODES_PAIRS)
def test_mul_add_all_pairs_1_6_9(oracle, mode):
    """The fused covers (general and fast-domain) over every (a, b) of 1/6/9 for 36 fixed c values."""
    rn, ftz = mode
    spec = bfp.make_spec(6, 9, rn, ftz)
    fmt = (6, 9, rn, ftz)
    na = 1024  # a values per chunk -> 2^26 pairs
    m = na << 16
    vb = bfp.pack(torch.arange(1 << 16, dtype=torch.int64, device="cuda").repeat(na), spec)
    vcs = [bfp.pack(torch.full((m,), c, dtype=torch.int64, device="cuda"), spec) for c in C_1_6_9]
    L = _lib.lib()
    outs = [bfp.empty(spec, m) for _ in C_1_6_9]
    t0, bad = time.time(), 0
    # default: every 4th chunk of 1024 a values (16 of 64: a-exponent fields 0-1, 8-9, 16-17, ... of both
    # signs, 2^30 pairs); BFP_GPU_SUITE=full / BFP_EXHAUSTIVE16=all: all 2^32 pairs (~5 min)
    step = na if FULL_GPU_SUITE else 4 * na
    for a0 in range(0, 1 << 16, step):
        va = bfp.pack(torch.arange(a0, a0 + na, dtype=torch.int64, device="cuda").repeat_interleave(1 << 16),
                      spec)
        for vc, o in zip(vcs, outs):
            assert L.bfp_mul_add(spec.c, va.planes.data_ptr(), vb.planes.data_ptr(), vc.planes.data_ptr(),
                                 o.planes.data_ptr(), m, _stream()) == 0
        got = [o.planes.cpu().numpy().view(np.uint32) for o in outs]
        nbad, info = oracle.verify_mul_add_pairs(fmt, a0, na, np.array(C_1_6_9, dtype=np.uint64), got)
        if nbad:
            i, k, g, w = info
            print(f"mismatch a={a0 + (i >> 16):#x} b={i & 0xffff:#x} c={C_1_6_9[k]:#x}: got {g:#x} want {w:#x}")
        bad += nbad
    print(f"mul_add 1/6/9 {fmt}: {'all 2^32' if FULL_GPU_SUITE else '2^30 (every 4th a chunk)'} (a, b) x "
          f"{len(C_1_6_9)} c, {bad} mismatches, {time.time() - t0:.1f} s")
    assert bad == 0


@pytest.mark.parametrize("fmt2", [(3, 2), (4, 3)])
@pytest.mark.parametrize("mode", [(1, 0), (0, 0), (1, 1), (0, 1)])
def test_mul_add_all_triples(oracle, fmt2, mode):
    """Every (a, b, c) of the <= 8-bit formats through the fused cover."""
    e, s = fmt2
    nb = 1 + e + s
    fmt = fmt2 + mode
    spec = bfp.make_spec(e, s, mode[0], mode[1])
    t = torch.arange(1 << (3 * nb), dtype=torch.int64, device="cuda")
    mask = (1 << nb) - 1
    a, b, c = t >> (2 * nb), (t >> nb) & mask, t & mask
    z = bfp.bfp_mul_add(bfp.pack(a, spec), bfp.pack(b, spec), bfp.pack(c, spec))
    ha, hb, hc = (v.to(torch.int32).cpu().numpy().view(np.uint32) for v in (a, b, c))
    _check(oracle, "mul_add", fmt, (ha, hb, hc), z.planes.cpu().numpy(), len(ha), f"mul_add {fmt} all triples")
