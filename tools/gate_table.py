"""Gate-count parity tooling: the reference's own
counted_lane tally (lane.hpp:119-188, via oracle/_ref) next to the SASS LOP3
count of our compiled network, per format x op x mode, per element.

    python tools/gate_table.py [--md out.md]

Reference gates are 2-input AND/OR/XOR + NOT per 32-element word (the
reference counts one op per lane operation); ours are 3-input LOP3 per
32-element word.  Both are divided by 32 (per element).
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tools"))

FORMATS = [(3, 2), (4, 3), (5, 3), (5, 7), (5, 10), (6, 9), (8, 7), (8, 15), (8, 23)]
OPS = {"add": 0, "sub": 1, "mul": 2, "div": 3, "mul_add": 4}


def table(modes=((1, 0), (0, 0))) -> list[dict]:
    import oracle as O
    import sass_stats
    st = sass_stats.stats(pattern=r"k_arith")
    rows = []
    for (e, s) in FORMATS:
        for rn, ftz in modes:
            for op, code in OPS.items():
                ref = O.ref_gate_count(op, (e, s, rn, ftz))["total"] if O.ref_available() else None
                key = (f"k_arith<bfpg::Format<{e}, {s}, {'true' if rn else 'false'}, "
                       f"{'true' if ftz else 'false'}>, {code}>")
                ent = next((r for n, r in st.items() if key in n), None)
                # mul_add kernels hold two covers (sass_stats.cover_paths): one row per path
                variants = ([(op, ent["LOP3"])] if not ent.get("paths") else
                            [(op + " (general cover)", ent["paths"]["general"]),
                             (op + " (fast-domain cover)", ent["paths"]["fast"])]) if ent else [(op, None)]
                for name, ours in variants:
                    rows.append({"fmt": f"1/{e}/{s}", "mode": ("rn" if rn else "rz") + ("+ftz" if ftz else ""),
                                 "op": name, "ref_gates_per_elem": None if ref is None else ref / 32,
                                 "ours_lop3_per_elem": None if ours is None else ours / 32,
                                 "ratio": None if (ref is None or not ours) else ref / ours})
    return rows


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--md", default=None)
    a = ap.parse_args()
    rows = table()
    lines = ["| format | mode | op | reference gates/elem | ours LOP3/elem | ratio |", "|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r['fmt']} | {r['mode']} | {r['op']} | {r['ref_gates_per_elem']:.2f} | "
                     f"{r['ours_lop3_per_elem']:.2f} | {r['ratio']:.2f} |")
    out = "\n".join(lines)
    print(out)
    if a.md:
        Path(a.md).write_text("# Gate counts: reference counted_lane vs our SASS LOP3 (regenerated from the shipped libbfpgpu.so by tools/gate_table.py)\n\n" + out + "\n")


if __name__ == "__main__":
    main()
