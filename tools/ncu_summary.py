"""Summarise ncu reports (raw page) into JSON for profiles/ and print a table.

    python tools/ncu_summary.py out.json rep1.ncu-rep [rep2 ...]
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second", "lts__t_bytes.sum",
    # where the warps wait (PC sampling; issue-stall reasons)
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_not_selected", "smsp__pcsamp_warps_issue_stalled_selected",
    "smsp__pcsamp_warps_issue_stalled_wait", "smsp__pcsamp_warps_issue_stalled_dispatch_stall",
    "smsp__pcsamp_warps_issue_stalled_lg_throttle", "smsp__pcsamp_warps_issue_stalled_branch_resolving",
    "smsp__pcsamp_warps_issue_stalled_no_instructions",
]


def summarise(rep: str) -> list[dict]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:110]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        out.append(d)
    return out


def main() -> None:
    out, reps = sys.argv[1], sys.argv[2:]
    res = {rep: summarise(rep) for rep in reps}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    for rep, ks in res.items():
        print(rep)
        for d in ks:
            print("  ", d["kernel"][:80])
            for k in KEYS[:12]:
                if k in d:
                    print(f"      {k:62s} {d[k]}")


if __name__ == "__main__":
    main()
