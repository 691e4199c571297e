"""bfp_chain (fused expression programs, NVRTC-compiled): bit-identical to the
same sequence of single-op calls, and to the oracle's composition."""
from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import operands

import paper_1602_04716_b200 as bfp

pytestmark = pytest.mark.gpu

OPS = {"+": bfp.bfp_add, "-": bfp.bfp_sub, "*": bfp.bfp_mul, "/": bfp.bfp_div}
ONAME = {"+": "add", "-": "sub", "*": "mul", "/": "div"}


def _eval_seq(prog, vs):
    st = []
    for ch in prog:
        if ch.isalpha():
            st.append(vs[ord(ch) - 97])
        else:
            y, x = st.pop(), st.pop()
            st.append(OPS[ch](x, y))
    return st[0]


def _eval_oracle(oracle, prog, fmt, encs):
    st = []
    for ch in prog:
        if ch.isalpha():
            st.append(encs[ord(ch) - 97])
        else:
            y, x = st.pop(), st.pop()
            st.append(oracle.binop(ONAME[ch], fmt, x, y))
    return st[0]


PROGRAMS = ["ab*c+", "ab*cd*+", "ab+c/", "ab-ab+*", "abc**d-", "ab/ba/-", "aa*a*a*", "ab*c+d*e-"]


@pytest.mark.parametrize("fmt", [(4, 3, 1, 0), (5, 10, 1, 0), (6, 9, 0, 1), (8, 15, 1, 0), (7, 20, 1, 0)])
@pytest.mark.parametrize("prog", PROGRAMS)
def test_chain_matches_sequence_and_oracle(oracle, fmt, prog):
    e, s, rn, ftz = fmt
    spec = bfp.make_spec(e, s, rn, ftz)
    k = max(ord(c) - 96 for c in prog if c.isalpha())
    rng = np.random.default_rng(hash((fmt, prog)) & 0xFFFF)
    n = 3 * 1024 + 77
    encs = [operands(e, s, n, rng) for _ in range(k)]
    vs = [bfp.pack(torch.from_numpy(x.astype(np.int64)).cuda(), spec) for x in encs]
    z = bfp.chain(prog, *vs)
    seq = _eval_seq(prog, vs)
    assert torch.equal(z.planes, seq.planes), "chain != sequence of single-op calls"
    got = bfp.to_u64(bfp.unpack(z), spec).cpu().numpy().astype(np.uint64)
    assert np.array_equal(got, _eval_oracle(oracle, prog, fmt, encs))


def test_chain_mul_add_equals_fused_kernel():
    spec = bfp.make_spec(6, 9)
    rng = np.random.default_rng(5)
    n = 1 << 20
    vs = [bfp.pack(torch.from_numpy(operands(6, 9, n, rng).astype(np.int64)).cuda(), spec) for _ in range(3)]
    assert torch.equal(bfp.chain("ab*c+", *vs).planes, bfp.bfp_mul_add(*vs).planes)


def test_chain_errors():
    spec = bfp.make_spec(4, 3)
    other = bfp.make_spec(4, 3, name="other")
    a = bfp.empty(spec, 100)
    with pytest.raises(ValueError):
        bfp.chain("ab+", a, bfp.empty(other, 100))  # require_same_shape, name included
    with pytest.raises(ValueError):
        bfp.chain("ab+", a, bfp.empty(spec, 99))
    with pytest.raises(ValueError):
        bfp.chain("a+", a, a)


@pytest.mark.parametrize("fmt", [(4, 3, 1, 0), (5, 10, 1, 1), (8, 7, 0, 0), (6, 9, 1, 0), (7, 20, 1, 0)])
@pytest.mark.parametrize("prog", ["ab*c+", "ab+ab-*", "ab/"])
def test_chain_f32_matches_planes_chain(fmt, prog):
    e, s, rn, ftz = fmt
    spec = bfp.make_spec(e, s, rn, ftz)
    g = torch.Generator(device="cuda").manual_seed(e * 100 + s)
    n = 5 * 1024 + 333  # ragged tail
    k = max(ord(c) - 96 for c in prog if c.isalpha())
    xs = [(torch.randn(n, device="cuda", generator=g) * 50).float() for _ in range(k)]
    xs[0][:7] = torch.tensor([0.0, -0.0, float("inf"), float("nan"), 1e-30, -3e38, 65504.0], device="cuda")
    got = bfp.chain_f32(prog, spec, *xs)
    want = bfp.unpack_f32(bfp.chain(prog, *[bfp.pack_f32(x, spec) for x in xs]))
    assert torch.equal(got.view(torch.int32), want.view(torch.int32))


def _random_program(rng, k: int, nops: int) -> str:
    """A random well-formed postfix program over inputs a.. (k of them)."""
    out, depth = [], 0
    while nops > 0 or depth != 1:
        if depth >= 2 and (nops > 0 and rng.random() < 0.45 or depth > nops + 1):
            out.append("+-*/"[int(rng.integers(4))])
            depth -= 1
            nops -= 1
        elif nops > 0 or depth < 1:
            out.append(chr(97 + int(rng.integers(k))))
            depth += 1
        else:
            out.append("+-*/"[int(rng.integers(4))])
            depth -= 1
    return "".join(out)


@pytest.mark.slow
@pytest.mark.skipif(not __import__("os").environ.get("BFP_FUZZ_CHAIN"), reason="set BFP_FUZZ_CHAIN=<count>")
def test_chain_fuzz(oracle):
    """Random programs x random legal formats (compiled and NVRTC-only) x modes
    against the oracle's composition of single ops."""
    import os
    rng = np.random.default_rng(2024)
    for t in range(int(os.environ["BFP_FUZZ_CHAIN"])):
        e = int(rng.integers(2, 9))
        s = int(rng.integers(1, 24))
        rn, ftz = int(rng.integers(2)), int(rng.integers(2))
        k = int(rng.integers(1, 6))
        prog = _random_program(rng, k, int(rng.integers(1, 7)))
        fmt = (e, s, rn, ftz)
        spec = bfp.make_spec(e, s, rn, ftz)
        n = int(rng.integers(1, 5000))
        encs = [operands(e, s, n, rng) for _ in range(k)]
        vs = [bfp.pack(torch.from_numpy(x.astype(np.int64)).cuda(), spec) for x in encs]
        got = bfp.to_u64(bfp.unpack(bfp.chain(prog, *vs)), spec).cpu().numpy().astype(np.uint64)
        want = _eval_oracle(oracle, prog, fmt, encs)
        assert np.array_equal(got, want), (t, fmt, prog)
        if e <= 8 and s <= 23:  # the float32 form: == decode(chain(encode(x), ...))
            scale = float(2.0 ** float(rng.integers(-8, 9)))
            xs = [torch.from_numpy((rng.standard_normal(n) * scale).astype(np.float32)).cuda() for _ in range(k)]
            zf = bfp.chain_f32(prog, spec, *xs)
            zp = bfp.unpack_f32(bfp.chain(prog, *[bfp.pack_f32(x, spec) for x in xs]))
            assert torch.equal(zf.view(torch.int32), zp.view(torch.int32)), (t, fmt, prog, "f32")
            if k >= 2:  # the fused single-op float32 kernel (bfp_arith_f32) of the same format
                op = int(rng.integers(4))
                za = bfp.arith_f32(op, spec, xs[0], xs[1])
                zr = bfp.unpack_f32(bfp.arith(op, bfp.pack_f32(xs[0], spec), bfp.pack_f32(xs[1], spec)))
                assert torch.equal(za.view(torch.int32), zr.view(torch.int32)), (t, fmt, op, "arith_f32")
