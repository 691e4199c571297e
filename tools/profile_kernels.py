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
    import paper_1602_04716_b200 as bfp
    from paper_1602_04716_b200 import workloads as W

    dev = torch.device("cuda", 0)
    jobs = []  # (label, callable)
    if a.config in ("C1", "C2", "C5"):
        import bench
        spec, n, ops = bench.make_inputs(a.config, 0, 1, dev)
        for op, x, y, c in ops:
            z = bfp.empty(spec, n)
            fn = {"add": bfp.bfp_add, "sub": bfp.bfp_sub, "mul": bfp.bfp_mul}.get(op)
            if op == "mul_add":
                jobs.append((op, lambda x=x, y=y, c=c, z=z: bfp.bfp_mul_add(x, y, c, out=z)))
            else:
                jobs.append((op, lambda fn=fn, x=x, y=y, z=z: fn(x, y, out=z)))
    elif a.config == "C3":
        spec = bfp.make_spec(5, 10)
        n = 1 << 28
        xa = W.c3_floats(0, n, W.SEED_A, dev)
        va = bfp.pack_f32(xa, spec)
        vb = bfp.pack_f32(W.c3_floats(0, n, W.SEED_B, dev), spec)
        z = bfp.empty(spec, n)
        out = torch.empty(n, dtype=torch.float32, device=dev)
        jobs = [("pack_f32", lambda: bfp.pack_f32(xa, spec)),
                ("add", lambda: bfp.bfp_add(va, vb, out=z)),
                ("mul", lambda: bfp.bfp_mul(va, vb, out=z)),
                ("unpack_f32", lambda: bfp.lib().bfp_unpack_f32(spec.c, z.planes.data_ptr(),
                                                                out.data_ptr(), n, None))]
    elif a.config == "C4":
        n = 1 << 28
        for (e, s) in [(3, 2), (5, 3), (5, 7), (8, 7), (8, 15)]:
            spec = bfp.make_spec(e, s)
            va = bfp.pack(W.c4_encodings(e, s, 0, n, W.SEED_A, dev), spec)
            vb = bfp.pack(W.c4_encodings(e, s, 0, n, W.SEED_B, dev), spec)
            z = bfp.empty(spec, n)
            jobs.append((f"add_{e}_{s}", lambda va=va, vb=vb, z=z: bfp.bfp_add(va, vb, out=z)))
            jobs.append((f"mul_{e}_{s}", lambda va=va, vb=vb, z=z: bfp.bfp_mul(va, vb, out=z)))
    if a.ops:
        keep = set(a.ops.split(","))
        jobs = [j for j in jobs if j[0] in keep]
    torch.cuda.synchronize()
    for _ in range(a.iters):
        for _, fn in jobs:
            fn()
    torch.cuda.synchronize()
    print("ok", [j[0] for j in jobs])


if __name__ == "__main__":
    main()
