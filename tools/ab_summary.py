"""Median per-kernel throughput of A/B runs (tools/gpu_ab_libs.sh output):
    python tools/ab_summary.py gpurun_out/ab_<tag>.jsonl ..."""
from __future__ import annotations

import json
import statistics
import sys
from pathlib import Path

rows: dict = {}
for f in sys.argv[1:]:
    tag = Path(f).stem.removeprefix("ab_")
    for line in open(f):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        mhz = d.get("clocks", {}).get("sm_mhz")
        for k, v in d["roofline"]["per_op"].items():
            rows.setdefault(k, {}).setdefault(tag, []).append((v["gelem_s"], mhz, v.get("logic_frac_at_load_clock")))
tags = sorted({t for r in rows.values() for t in r})
print(f"{'kernel':16s} " + " ".join(f"{t:>24s}" for t in tags))
for k, r in rows.items():
    cells = []
    for t in tags:
        v = r.get(t, [])
        if v:
            cells.append(f"{statistics.median(x[0] for x in v):9.1f} @{statistics.median(x[1] or 0 for x in v):5.0f}MHz n={len(v)}")
        else:
            cells.append(" " * 24)
    print(f"{k:16s} " + " ".join(f"{c:>24s}" for c in cells))
