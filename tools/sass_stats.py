"""Static SASS instruction mix per kernel of libbfpgpu.so (cuobjdump -sass).

    python tools/sass_stats.py [--filter REGEX] [--json out.json]

For the arithmetic kernels the loop body is one 32-element unit per thread,
so (LOP3 count in the body) / 32 is the LOP3 work per element -- the logic
leg of the roofline.  The body is everything between the
first and the last global load/store of the kernel; the count reported is
the whole function, which only adds the loop/address prologue.
"""
from __future__ import annotations

import argparse
import json
import os
import re
import subprocess
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LIB = Path(os.environ.get("BFP_LIB") or ROOT / "paper_1602_04716_b200" / "libbfpgpu.so")

ALU_PIPE = {"LOP3", "IADD3", "SHF", "PRMT", "ISETP", "SEL", "IMNMX", "FLO", "LEA", "LOP",
            "VIADD", "IABS", "POPC", "BREV", "PLOP3", "VIMNMX", "SGXT", "BMSK", "FSEL", "FSETP", "P2R", "R2P"}
FMA_PIPE = {"IMAD", "FFMA", "FMUL", "FADD", "HFMA2", "HADD2", "HMUL2", "IMUL", "IADD"}
MEM = {"LDG", "STG", "LDS", "STS", "LDL", "STL", "LD", "ST"}


def demangle(names: list[str]) -> dict[str, str]:
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
        return dict(zip(names, out.splitlines()))
    except OSError:
        return {n: n for n in names}


def sass_functions(lib: Path) -> dict[str, list[str]]:
    txt = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", str(lib)],
                         capture_output=True, text=True, check=True).stdout
    funcs: dict[str, list[str]] = {}
    cur = None
    for line in txt.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*([0-9a-f]+)\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)(.*)", line)
        if m:
            funcs[cur].append((int(m.group(1), 16), m.group(3), m.group(4), (m.group(2) or "").strip()))
    return funcs


def loop_body(ins: list) -> list[str]:
    """Opcodes of the main loop: the span of the widest backward branch (the
    grid-stride loop of the kernels; empty if there is none)."""
    best = None
    for a, op, rest, _ in ins:
        if op.startswith("BRA"):
            t = re.search(r"0x([0-9a-f]+)", rest)
            if t and int(t.group(1), 16) < a:
                lo = int(t.group(1), 16)
                if best is None or a - lo > best[1] - best[0]:
                    best = (lo, a)
    if best is None:
        return []
    return [op for a, op, _, _ in ins if best[0] <= a <= best[1]]


def cover_paths(ins: list) -> dict | None:
    """mul_add kernels hold two LOP3 covers behind one warp-uniform branch
    (`@P BRA else; <cover 1>; BRA join; else: <cover 2>; join:`, both forward,
    inside the loop).  Returns the LOP3 count a unit executes on each side --
    the whole function minus the OTHER cover -- as {"fast", "general"} (the
    fast-domain cover is the smaller one), or None without that shape."""
    addr = {i[0]: k for k, i in enumerate(ins)}

    def target(rest):
        t = re.search(r"0x([0-9a-f]+)", rest)
        return int(t.group(1), 16) if t else None

    best = None
    for k, (a, op, rest, pred) in enumerate(ins):
        if not (op.startswith("BRA") and pred):  # predicated forward branch
            continue
        els = target(rest)
        if els is None or els <= a or els not in addr:
            continue
        ke = addr[els]
        jop = ins[ke - 1]
        if not jop[1].startswith("BRA") or jop[3]:
            continue
        join = target(jop[2])
        if join is None or join <= els or join not in addr:
            continue
        c1 = sum(1 for i in ins[k + 1:ke] if i[1].startswith("LOP3"))
        c2 = sum(1 for i in ins[ke:addr[join]] if i[1].startswith("LOP3"))
        if min(c1, c2) >= 64 and (best is None or c1 + c2 > sum(best)):
            best = (c1, c2)
    if best is None:
        return None
    total = sum(1 for i in ins if i[1].startswith("LOP3"))
    return {"fast": total - max(best), "general": total - min(best), "covers": sorted(best)}


def stats(lib: Path = LIB, pattern: str | None = None) -> dict[str, dict]:
    funcs = sass_functions(lib)
    dm = demangle(list(funcs))
    res = {}
    for name, tins in funcs.items():
        pretty = dm.get(name, name)
        if pattern and not re.search(pattern, pretty):
            continue
        ins = [op for _, op, _, _ in tins]
        body = Counter(i.split(".")[0] for i in loop_body(tins))
        base = Counter(i.split(".")[0] for i in ins)
        alu = sum(v for k, v in base.items() if k in ALU_PIPE)
        fma = sum(v for k, v in base.items() if k in FMA_PIPE)
        res[pretty] = {
            "mangled": name,
            "total": len(ins),
            "LOP3": base.get("LOP3", 0),
            "alu_pipe": alu,
            "fma_pipe": fma,
            "mem": sum(v for k, v in base.items() if k in MEM),
            "loop_LOP3": body.get("LOP3", 0),
            "loop_alu_pipe": sum(v for k, v in body.items() if k in ALU_PIPE),
            "loop_total": sum(body.values()),
            "top": base.most_common(8),
        }
        paths = cover_paths(tins)
        if paths:
            res[pretty]["paths"] = paths
    return res


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=str(LIB))
    ap.add_argument("--filter", default=r"k_arith")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    res = stats(Path(a.lib), a.filter)
    for name, r in sorted(res.items()):
        short = re.sub(r"bfpg::|Format<|unsigned int|const", "", name)[:90]
        print(f"{short:90s} tot={r['total']:5d} LOP3={r['LOP3']:5d} alu={r['alu_pipe']:5d} "
              f"fma={r['fma_pipe']:4d} mem={r['mem']:3d} loop: LOP3={r['loop_LOP3']:5d} "
              f"alu={r['loop_alu_pipe']:5d}  LOP3/elem={r['LOP3'] / 32:.2f}"
              + (f"  two covers {r['paths']['covers']}: fast path {r['paths']['fast'] / 32:.2f}, "
                 f"general {r['paths']['general'] / 32:.2f} LOP3/elem" if r.get("paths") else ""))
    if a.json:
        Path(a.json).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
