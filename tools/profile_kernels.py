"""Minimal driver for ncu: builds one config's resident operands and runs a
few steps of its kernels, nothing else (so launch lists and --set full
captures see only the hot path).

    python tools/profile_kernels.py [--config C2] [--iters 5]
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--ops", default=None, help="comma list (C3/C4: which kernels)")
    a = ap.parse_args()
    import torch
    dev = torch.device("cuda", 0)
    import bench
    jobs = [(j.label, j.launch) for j in bench.make_jobs(a.config, 0, 1, dev)]
    if a.ops:
        keep = set(a.ops.split(","))
        jobs = [j for j in jobs if j[0] in keep]
    torch.cuda.synchronize()
    st = torch.cuda.current_stream().cuda_stream
    for i in range(a.iters):
        for _, fn in jobs:
            fn(i, st)
    torch.cuda.synchronize()
    print("ok", [j[0] for j in jobs])


if __name__ == "__main__":
    main()
