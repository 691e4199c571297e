"""Per-kernel evidence table (markdown) from bench.py JSON lines.

    python tools/kernel_table.py profiles/a.jsonl [profiles/b.jsonl ...] > profiles/r02_kernel_table.md

One row per timed kernel of every line: throughput, both roofline legs, the
binding one, SASS LOP3 per element, executed ALU instructions per element and
DRAM traffic over algorithmic bytes (both measured by the in-run ncu pass).
"""
from __future__ import annotations

import json
import sys


def rows(path: str):
    for text in open(path):
        text = text.strip()
        if not text.startswith("{"):
            continue
        d = json.loads(text)
        cfg = d["config"]["workload"].split(":")[0].split(" ")[0]
        mhz = d.get("clocks", {}).get("sm_mhz")
        for label, e in d["roofline"].get("per_op", {}).items():
            yield cfg, label, e, mhz
        for fmt, ops in d.get("per_format", {}).items():  # variants timed beside the step
            for op, e in ops.items():
                if "(" in op:
                    yield cfg, f"{op} {fmt}", e, None


def fmt(v, spec="{:.3f}"):
    return "—" if v is None else spec.format(v)


def main() -> None:
    print("| config:kernel | Gelem/s | HBM frac (copy peak) | LOP3/elem (SASS) | ALU inst/elem (ncu) | logic frac "
          "(burst / at load clock) | binding leg | DRAM bytes / algorithmic (ncu) | SM MHz under load |")
    print("|---|---|---|---|---|---|---|---|---|")
    for path in sys.argv[1:]:
        for cfg, label, e, mhz in rows(path):
            lf = e.get("logic_frac")
            lfc = e.get("logic_frac_at_load_clock")
            logic = "—" if lf is None else f"{lf:.2f} / {fmt(lfc, '{:.2f}')}"
            print(f"| {cfg}:{label} | {e.get('gelem_s', 0):.0f} | {fmt(e.get('hbm_frac'))} | "
                  f"{fmt(e.get('lop3_per_elem'), '{:.2f}')} | {fmt(e.get('alu_inst_per_elem_measured'), '{:.2f}')} | "
                  f"{logic} | {e.get('bound', '—')} {fmt(e.get('frac'), '{:.2f}')} | "
                  f"{fmt(e.get('traffic_over_algorithmic'), '{:.2f}')} | {fmt(mhz, '{:.0f}')} |")


if __name__ == "__main__":
    main()
