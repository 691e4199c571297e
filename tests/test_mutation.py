"""Mutation smoke test: the parity checks must FAIL on corrupted networks.

A copy of the circuits (paper_1602_04716_b200/csrc) is corrupted and the RN +
gradual networks of one format are rebuilt for the host from it
(tests/native/mutant_harness.cpp), then put through the comparisons the
parity suite runs, against the oracle:

  * round-stage mutants of the templates (1/4/3, exhaustive: all 2^16 pairs
    of add / sub / mul / div, all 2^24 triples of mul_add): round-half-up
    instead of half-to-even, and the sticky bits dropped, in the adder and
    in the shared finish_round of mul / div / mul_add -- every one killed;
  * single-LUT mutants of the generated 1/4/3 LOP3 covers (the code the
    kernels run): one reachable truth-table bit (no constant input involved)
    of a seeded random lop3 flipped.  Over the exhaustive domain a survivor
    is an EQUIVALENT mutant (that minterm never occurs at that node); most
    are killed;
  * single-LUT mutants of the 1/6/9 mul_add cover (C5's network), where the
    suite is sampled: the parity suite's operand generator (2^16 triples
    with zero / subnormal / near-overflow / special weighting) must kill
    every mutant that a 64x larger uniform sample kills.

  * the same for mul_add's SECOND cover (the fast-domain one, Gen<F, 5>), run
    as the kernels run it -- inside the domain, the general cover elsewhere:
    1/4/3 over all 2^24 triples, 1/6/9 with the suite's in-domain operand
    generator against a 32x larger uniform in-domain sample.

The unmutated copy passes, so the kills are the mutations'.
Log of a run: profiles/r02_mutation.log.
"""
from __future__ import annotations

import ctypes as C
import re
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT, fast_domain_operands, operands

CSRC = ROOT / "paper_1602_04716_b200" / "csrc"
HARNESS = ROOT / "tests" / "native" / "mutant_harness.cpp"
OPC = {"add": 0, "sub": 1, "mul": 2, "div": 3, "mul_add": 4}


def _build(tmp, name, fmt2=(4, 3), mutate_circuits=None, mutate_gen=None):
    e, s = fmt2
    d = tmp / name
    (d / "gen").mkdir(parents=True)
    for f in list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")):
        shutil.copy(f, d / f.name)
    gname = f"gen_{e}_{s}.cuh"
    src = (CSRC / "gen" / gname).read_text()
    if mutate_gen:
        src = mutate_gen(src)
    (d / "gen" / gname).write_text(src)
    if mutate_circuits:
        p = d / "bfp_circuits.cuh"
        txt = p.read_text()
        new = mutate_circuits(txt)
        assert new != txt, "mutation did not apply"
        p.write_text(new)
    so = d / "libmut.so"
    subprocess.run(["g++", "-std=c++17", "-O1", "-fPIC", "-shared", f"-I{d}", f"-DMUT_E={e}", f"-DMUT_S={s}",
                    f'-DMUT_GEN="gen/{gname}"', str(HARNESS), "-o", str(so)], check=True, timeout=600)
    L = C.CDLL(str(so))
    L.mut_binop.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]
    return L


class Cases:
    """Operand sets with the oracle's expected planes, per op."""

    def __init__(self, oracle, fmt, sets: dict):
        self.nb = 1 + fmt[0] + fmt[1]
        self.ins, self.want = {}, {}
        for op, (x, y, c) in sets.items():
            self.ins[op] = [oracle.pack_planes(v, self.nb) if v is not None else None for v in (x, y, c)]
            self.want[op] = oracle.pack_planes(oracle.binop(op, fmt, x, y, c), self.nb)

    def killed(self, L, base: int, ops=None) -> list[str]:
        out = []
        for op in ops or list(self.ins):
            a, b, c = self.ins[op]
            z = np.zeros_like(a)
            assert L.mut_binop(base + OPC[op], a.ctypes.data, b.ctypes.data,
                               c.ctypes.data if c is not None else None, z.ctypes.data,
                               len(a) // (self.nb * 32)) == 0
            if not np.array_equal(z, self.want[op]):
                out.append(op)
        return out


@pytest.fixture(scope="module")
def exhaustive_4_3(oracle):
    if not (CSRC / "gen" / "gen_4_3.cuh").exists():
        from paper_1602_04716_b200.build import generate
        generate(verbose=False)
    x = np.repeat(np.arange(256, dtype=np.uint64), 256)
    y = np.tile(np.arange(256, dtype=np.uint64), 256)
    t = np.arange(1 << 24, dtype=np.uint64)
    tr = (t >> np.uint64(16), (t >> np.uint64(8)) & np.uint64(255), t & np.uint64(255))
    sets = {op: (x, y, None) for op in ("add", "sub", "mul", "div")}
    sets["mul_add"] = tr
    return Cases(oracle, (4, 3, 1, 0), sets)


def test_unmutated_copy_passes(tmp_path, exhaustive_4_3):
    L = _build(tmp_path, "clean")
    assert exhaustive_4_3.killed(L, 0) == [] and exhaustive_4_3.killed(L, 10) == []


ROUND_MUTANTS = {
    # add: round-half-up (the LSB no longer breaks ties)
    "add_ties_away": (lambda s: s.replace("rnd = x[3] & (x[0] | x[1] | x[2] | sig[0]);",
                                          "rnd = x[3] & (x[0] | x[1] | x[2] | ONES);"), {"add", "sub", "mul_add"}),
    # add: the sticky bits forgotten (ties-to-even applied to above-half)
    "add_no_sticky": (lambda s: s.replace("rnd = x[3] & (x[0] | x[1] | x[2] | sig[0]);",
                                          "rnd = x[3] & sig[0];"), {"add", "sub", "mul_add"}),
    # finish_round (mul / div / mul_add): round-half-up, then sticky dropped
    "finish_ties_away": (lambda s: s.replace("rnd = R[1] & (R[0] | sig[0]);", "rnd = R[1];"),
                         {"mul", "div", "mul_add"}),
    "finish_no_sticky": (lambda s: s.replace("rnd = R[1] & (R[0] | sig[0]);", "rnd = R[1] & sig[0];"),
                         {"mul", "div", "mul_add"}),
}


@pytest.mark.parametrize("name", sorted(ROUND_MUTANTS))
def test_round_stage_mutants_killed(tmp_path, exhaustive_4_3, name):
    mut, ops = ROUND_MUTANTS[name]
    L = _build(tmp_path, name, mutate_circuits=mut)
    k = exhaustive_4_3.killed(L, 0, sorted(ops))
    print(f"round-stage mutant {name}: killed by {k} (of {sorted(ops)})")
    assert k, f"mutant {name} survived the parity checks of {sorted(ops)}"


def _flip_lut(src: str, fmt2, op: int, which: int, rng) -> tuple[str, str]:
    """Flip one reachable truth-table bit of the `which`-th lop3 of the RN +
    gradual cover of `op`: minterm k = 4a + 2b + c, and a constant-0 input
    (the emitter's `0u` for a cut of fewer than three leaves) fixes its bit."""
    e, s = fmt2
    head = f"template <> struct Gen<Format<{e}, {s}, true, false>, {op}> {{"
    i0 = src.index(head)
    nxt = src.find("template <>", i0 + len(head))
    i1 = nxt if nxt >= 0 else len(src)
    block = src[i0:i1]
    ms = list(re.finditer(r"lop3<0x([0-9A-F]{2})>\(([^,]+), ([^,]+), ([^)]+)\)", block))
    m = ms[which % len(ms)]
    const = [m.group(g).strip() == "0u" for g in (2, 3, 4)]
    bits = [k for k in range(8) if not any(const[j] and (k >> (2 - j)) & 1 for j in range(3))]
    bit = int(rng.choice(bits))
    tt = int(m.group(1), 16) ^ (1 << bit)
    new_block = block[:m.start()] + f"lop3<0x{tt:02X}>" + block[m.start() + len("lop3<0xXX>"):]
    line = block[block.rfind("\n", 0, m.start()) + 1:block.find("\n", m.end())].strip()
    return src[:i0] + new_block + src[i1:], f"bit {bit} of `{line}`"


def test_cover_lut_mutants_4_3(tmp_path, exhaustive_4_3):
    rng = np.random.default_rng(0x160204716)
    src = (CSRC / "gen" / "gen_4_3.cuh").read_text()
    res = []
    for op in OPC:
        for k in range(4):
            mutated, what = _flip_lut(src, (4, 3), OPC[op], int(rng.integers(0, 10_000)), rng)
            L = _build(tmp_path, f"lut_{op}_{k}", mutate_gen=lambda s, m=mutated: m)
            res.append((op, what, bool(exhaustive_4_3.killed(L, 10, [op]))))
    for op, what, kd in res:
        print(f"1/4/3 {op:8s} {what}: {'killed' if kd else 'equivalent (survives the exhaustive domain)'}")
    nk = sum(kd for *_, kd in res)
    print(f"1/4/3 cover LUT mutants: {nk}/{len(res)} killed, the rest proven equivalent over all inputs")
    assert nk >= 0.6 * len(res)


def test_cover_lut_mutants_6_9_mul_add(tmp_path, oracle):
    """C5's network, sampled suite: the parity suite's operands catch every
    mutant a 64x larger uniform sample catches."""
    fmt = (6, 9, 1, 0)
    rng = np.random.default_rng(7)
    n = 1 << 16
    suite = Cases(oracle, fmt, {"mul_add": tuple(operands(6, 9, n, rng) for _ in range(3))})
    big_rng = np.random.default_rng(8)
    big = Cases(oracle, fmt, {"mul_add": tuple(big_rng.integers(0, 1 << 16, size=64 * n, dtype=np.uint64)
                                               for _ in range(3))})
    L = _build(tmp_path, "clean69", (6, 9))
    assert suite.killed(L, 14 - OPC["mul_add"], ["mul_add"]) == [] and big.killed(L, 10, ["mul_add"]) == []
    src = (CSRC / "gen" / "gen_6_9.cuh").read_text()
    res = []
    for k in range(12):
        mutated, what = _flip_lut(src, (6, 9), OPC["mul_add"], int(rng.integers(0, 10_000)), rng)
        L = _build(tmp_path, f"lut69_{k}", (6, 9), mutate_gen=lambda s, m=mutated: m)
        ks, kb = bool(suite.killed(L, 10)), bool(big.killed(L, 10))
        res.append((what, ks, kb))
        print(f"1/6/9 mul_add {what}: suite {'killed' if ks else 'survived'}, "
              f"64x sample {'killed' if kb else 'survived'}")
    assert not [r for r in res if r[2] and not r[1]], "a mutant escaped the suite's sample but not a larger one"
    assert sum(r[1] for r in res) >= 0.6 * len(res)


# ------------------------------------------- mul_add's fast-domain cover
def test_fast_cover_lut_mutants_4_3(tmp_path, exhaustive_4_3):
    """Gen<F, 5> of 1/4/3 over every triple (it runs on the 1.54 M inside the
    domain): survivors are equivalent on the whole domain."""
    rng = np.random.default_rng(0x5eed5)
    src = (CSRC / "gen" / "gen_4_3.cuh").read_text()
    L = _build(tmp_path, "clean_fast43")
    assert exhaustive_4_3.killed(L, 15 - OPC["mul_add"], ["mul_add"]) == []
    res = []
    for k in range(4):
        mutated, what = _flip_lut(src, (4, 3), 5, int(rng.integers(0, 10_000)), rng)
        L = _build(tmp_path, f"fast43_{k}", mutate_gen=lambda s, m=mutated: m)
        res.append((what, bool(exhaustive_4_3.killed(L, 15 - OPC["mul_add"], ["mul_add"]))))
    for what, kd in res:
        print(f"1/4/3 mul_add fast cover {what}: {'killed' if kd else 'equivalent on the whole domain'}")
    assert sum(kd for _, kd in res) >= 0.6 * len(res)


def test_fast_cover_lut_mutants_6_9(tmp_path, oracle):
    """C5's cover: the suite's in-domain operand generator (2^16 triples,
    edge-weighted) kills every mutant a 32x larger uniform in-domain sample kills
    (profiles/r02_mutation_fastcover.log: 12 mutants against a 64x sample)."""
    fmt = (6, 9, 1, 0)
    rng = np.random.default_rng(17)
    n = 1 << 16
    suite = Cases(oracle, fmt, {"mul_add": fast_domain_operands(oracle, fmt, n, rng)})
    br = np.random.default_rng(18)
    m = 32 * n
    sg = lambda: br.integers(0, 2, size=m, dtype=np.uint64) << np.uint64(15)
    fr = lambda: br.integers(0, 512, size=m, dtype=np.uint64)
    ea = br.integers(1, 48, size=m)
    lo_b, hi_b = np.maximum(1, 32 - ea), np.minimum(47, 91 - ea)
    eb = lo_b + br.integers(0, 1 << 30, size=m) % (hi_b - lo_b + 1)
    ec = br.integers(16, 48, size=m)
    big = Cases(oracle, fmt, {"mul_add": tuple(sg() | (x.astype(np.uint64) << np.uint64(9)) | fr()
                                               for x in (ea, eb, ec))})
    code = 15 - OPC["mul_add"]
    L = _build(tmp_path, "clean_fast69", (6, 9))
    assert suite.killed(L, code, ["mul_add"]) == [] and big.killed(L, code, ["mul_add"]) == []
    src = (CSRC / "gen" / "gen_6_9.cuh").read_text()
    res = []
    for k in range(5):
        mutated, what = _flip_lut(src, (6, 9), 5, int(rng.integers(0, 10_000)), rng)
        L = _build(tmp_path, f"fast69_{k}", (6, 9), mutate_gen=lambda s, mm=mutated: mm)
        ks, kb = bool(suite.killed(L, code, ["mul_add"])), bool(big.killed(L, code, ["mul_add"]))
        res.append((what, ks, kb))
        print(f"1/6/9 mul_add fast cover {what}: suite {'killed' if ks else 'survived'}, "
              f"32x sample {'killed' if kb else 'survived'}")
    assert not [r for r in res if r[2] and not r[1]], "a mutant escaped the suite's sample but not a larger one"
    assert sum(r[1] for r in res) >= 0.6 * len(res)
