"""Per-launch DRAM traffic of every timed kernel, from `ncu --set full` captures,
into profiles/ncu_traffic.json (the `roofline.traffic` source of bench.py), with
the same capture's ALU-pipe utilisation and DRAM throughput (% of peak).

    python tools/ncu_traffic.py OUT.json CFG=report.ncu-rep [CFG=report ...]

Each report is one config's kernels run by tools/profile_kernels.py with
--iters 1 (setup launches of the same kernel come first, so the LAST launch
of each kernel name is the timed one).  Keys follow bench.py: "C3:mul",
"C4:mul_1/8/15", with ":<mode>" appended for non-default modes (CFG may be
given as "C2:rz-gradual" for that).
"""
from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys

OPS = {0: "add", 1: "sub", 2: "mul", 3: "div", 4: "mul_add"}
C4 = {(3, 2), (5, 3), (5, 7), (8, 7), (8, 15)}


def rows(rep: str) -> list[dict]:
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rs = list(csv.reader(io.StringIO(txt)))
    hdr, units = rs[0], rs[1]
    out = []
    for r in rs[2:]:
        d = dict(zip(hdr, r))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        rd = float(d["dram__bytes_read.sum"]) * scale[units[hdr.index("dram__bytes_read.sum")]]
        wr = float(d["dram__bytes_write.sum"]) * scale[units[hdr.index("dram__bytes_write.sum")]]
        pct = lambda k: round(float(d[k]), 2) if k in d and d[k] not in ("", "n/a") else None
        out.append({"kernel": d["Kernel Name"], "read": rd, "write": wr,
                    "alu": pct("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
                    "dram": pct("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                    "us": float(d["gpu__time_duration.sum"]) *
                    {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3, "ms": 1e3}
                    [units[hdr.index("gpu__time_duration.sum")]]})
    return out


def label(cfg: str, kernel: str) -> str | None:
    if kernel.startswith("bfp_chain_k"):
        return "a*b+c*d" if cfg.startswith("X3") else None
    m = re.search(r"k_(arith_f32|arith|pack_f32|unpack_f32)<\S*Format<(\d+), (\d+)[^>]*>(?:, (\d+))?",
                  kernel)
    if not m:
        return None
    kind, e, s = m.group(1), int(m.group(2)), int(m.group(3))
    if kind == "arith_f32":
        return f"{OPS[int(m.group(4))]}_f32"
    if kind != "arith":
        return kind
    op = OPS[int(m.group(4))]
    return f"{op}_1/{e}/{s}" if cfg.startswith(("C4", "X1")) else op


def main() -> None:
    out = sys.argv[1]
    try:
        res = json.load(open(out))
    except (OSError, ValueError):
        res = {}
    for arg in sys.argv[2:]:
        cfg, rep = arg.split("=", 1)
        last = {}
        for r in rows(rep):
            lb = label(cfg, r["kernel"])
            if lb:
                last[lb] = r
        base, _, mode = cfg.partition(":")
        for lb, r in last.items():
            key = f"{base}:{lb}" + (f":{mode}" if mode else "")
            res[key] = {"bytes": int(r["read"] + r["write"]), "ncu_us": round(r["us"], 2),
                        "alu_pipe_pct": r["alu"], "dram_throughput_pct": r["dram"]}
            print(f"{key:24s} read {r['read'] / 1e6:10.2f} MB  write {r['write'] / 1e6:10.2f} MB  "
                  f"{r['us']:9.1f} us")
    with open(out, "w") as f:
        json.dump(dict(sorted(res.items())), f, indent=1)


if __name__ == "__main__":
    main()
