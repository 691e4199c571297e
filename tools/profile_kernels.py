"""Minimal driver for ncu: builds one config's resident operands (exactly as
bench.py does) and runs a few steps of its kernels, nothing else, so launch
lists and --set full captures see only the hot path.

    python tools/profile_kernels.py [--config C5] [--iters 1] [--ops add_1/8/15,...]
                                    [--rounding rn|rz] [--subnormals gradual|ftz] [--marker] [--aux]

--marker prints "TIMED <k>" before the timed launches (k = kernels per
iteration x iters): bench.py's in-run traffic measurement takes the last k
profiled launches as the timed ones (operand setup comes first).
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--ops", default=None, help="comma list of job labels to keep")
    ap.add_argument("--rounding", choices=["rn", "rz"], default="rn")
    ap.add_argument("--subnormals", choices=["gradual", "ftz"], default="gradual")
    ap.add_argument("--marker", action="store_true")
    ap.add_argument("--aux", action="store_true",
                    help="run the kernels' timed variants instead (mul_add forced onto its general cover)")
    ap.add_argument("--rank", type=int, default=0, help="build rank r's shard of a --world run (bench's sizes)")
    ap.add_argument("--world", type=int, default=1)
    a = ap.parse_args()
    import torch
    dev = torch.device("cuda", 0)
    import bench
    bench.MODE = (int(a.rounding == "rn"), int(a.subnormals == "ftz"))
    made = bench.make_jobs(a.config, a.rank, a.world, dev)
    jobs = ([(f"{j.label}:{name}", fn) for j in made for name, fn in j.aux.items()] if a.aux
            else [(j.label, j.launch) for j in made])
    if a.ops:
        keep = set(a.ops.split(","))
        jobs = [j for j in jobs if j[0] in keep]
    torch.cuda.synchronize()
    if a.marker:
        print(f"TIMED {len(jobs) * a.iters}", flush=True)
    st = torch.cuda.current_stream().cuda_stream
    for i in range(a.iters):
        for _, fn in jobs:
            fn(i, st)
    torch.cuda.synchronize()
    print("ok", [j[0] for j in jobs])


if __name__ == "__main__":
    main()
