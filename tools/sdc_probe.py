"""Satisfiability-don't-care probe of a generated LOP3 cover (tools only):
simulate the cover bit-parallel on 2^22 random operand triples (a quarter with
the exponent forced to 0, 1, 2, max-1 or max) and, per LUT, find the input
minterms never observed.  Under those don't-cares, count LUTs that collapse to
a constant or a wire (one input or its complement) or lose an input -- an
upper estimate of what a proven (SAT) don't-care optimisation could remove.

    python tools/sdc_probe.py "6, 9" 4      # format "E, S", op (0 add .. 4 mul_add)
"""
import re, numpy as np, sys, collections
fmt = sys.argv[1] if len(sys.argv) > 1 else "6, 9"
op = sys.argv[2] if len(sys.argv) > 2 else "4"
src = open(f"paper_1602_04716_b200/csrc/gen/gen_{fmt.replace(', ','_')}.cuh").read()
i0 = src.index(f"template <> struct Gen<Format<{fmt}, true, false>, {op}>")
i1 = src.find("template <>", i0 + 10); blk = src[i0:i1 if i1 > 0 else None]
luts = re.findall(r"const w32 (t\d+) = lop3<0x([0-9A-F]{2})>\(([^,]+), ([^,]+), ([^)]+)\)", blk)
outs = re.findall(r"(Z\[\d+\]) = (~?)(\w+(?:\[\d+\])?);", blk)
e, s = map(int, fmt.split(", ")); N = 1 + e + s
W = 1 << 16  # uint64 words -> 2^22 samples
rng = np.random.default_rng(1)
def rand_planes():
    # random encodings with extra weight on special exponent values
    enc = rng.integers(0, 1 << N, size=W * 64, dtype=np.uint64)
    k = len(enc) // 4
    ex = rng.choice(np.array([0, 1, 2, (1 << e) - 2, (1 << e) - 1], dtype=np.uint64), size=k)
    enc[:k] = (enc[:k] & ~np.uint64(((1 << e) - 1) << s)) | (ex << np.uint64(s))
    bits = [((enc >> np.uint64(j)) & np.uint64(1)).astype(np.uint8) for j in range(N)]
    return [np.packbits(b, bitorder="little").view(np.uint64) for b in bits]
env = {}
for nm, P in (("X", rand_planes()), ("Y", rand_planes()), ("C", rand_planes())):
    for j in range(N): env[f"{nm}[{j}]"] = P[j]
env["0u"] = np.zeros(W, dtype=np.uint64)
ONE = np.uint64(0xFFFFFFFFFFFFFFFF)
red = collections.Counter()
for t, tt, a, b, c in luts:
    A, B, Cc = env[a.strip()], env[b.strip()], env[c.strip()]
    tt = int(tt, 16)
    r = np.zeros(W, dtype=np.uint64); seen = 0
    for k in range(8):
        m = (A if k & 4 else ~A) & (B if k & 2 else ~B) & (Cc if k & 1 else ~Cc)
        if np.any(m): seen |= 1 << k
        if (tt >> k) & 1: r |= m
    env[t] = r
    # with unseen minterms as don't cares: is the LUT a constant / a buffer of one input?
    care = seen
    f = tt & care
    def eq(g): return (g & care) == f
    ins = [(a.strip(), 0xF0), (b.strip(), 0xCC), (c.strip(), 0xAA)]
    kind = None
    if eq(0) or eq(0xFF): kind = "const"
    else:
        for nm, v in ins:
            if nm != "0u" and (eq(v) or eq(~v & 0xFF)): kind = "buffer"; break
    if kind is None:
        # depends on only two inputs under the cares?
        for drop in range(3):
            ok = True
            for k in range(8):
                k2 = k ^ (4 >> drop)
                if (care >> k) & 1 and (care >> k2) & 1 and ((tt >> k) & 1) != ((tt >> k2) & 1): ok = False
            if ok and ins[drop][0] != "0u": kind = "drops_an_input"; break
    red[kind or "full"] += 1
    red["unseen_minterms"] += 8 - bin(seen).count("1")
print(fmt, op, len(luts), dict(red))
