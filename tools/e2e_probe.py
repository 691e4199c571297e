"""Host-buffer pipeline probe: one C1-sized add (2^24 fp8 elements) through
bfp_arith_host_batch at several context chunk sizes, against the raw pinned
copy time of the same bytes.

    python tools/e2e_probe.py [--n 16777216]
"""
from __future__ import annotations

import argparse
import ctypes as C
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 24)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    import torch
    import paper_1602_04716_b200 as bfp
    L = bfp.lib()
    spec = bfp.make_spec(4, 3)
    n = a.n
    pb = spec.plane_bytes(n)
    hx, hy, hz = (L.bfp_host_alloc(pb) for _ in range(3))
    C.memset(hx, 0x3c, pb)
    C.memset(hy, 0x5a, pb)
    ops = (C.c_int * 1)(0)
    outs = (C.c_void_p * 1)(hz)

    def timed(fn):
        fn()
        best = []
        for _ in range(a.reps):
            t = time.perf_counter()
            fn()
            best.append(time.perf_counter() - t)
        best.sort()
        return best[0] * 1e3, best[len(best) // 2] * 1e3

    for chunk in (1 << 20, 1 << 21, 1 << 22, 1 << 23, 1 << 24):
        ctx = L.bfp_host_ctx_create(chunk)
        f = lambda: L.bfp_arith_host_batch(ctx, 1, ops, spec.c, hx, hy, None, outs, n)
        b, m = timed(f)
        print(f"ctx chunk 2^{chunk.bit_length() - 1}: best {b:.3f} ms  median {m:.3f} ms  "
              f"-> {n / b / 1e6:.2f} Gelem/s", flush=True)
        L.bfp_host_ctx_destroy(ctx)

    dx = torch.empty(2 * pb, dtype=torch.uint8, device="cuda")
    dz = torch.empty(pb, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    hin = torch.empty(2 * pb, dtype=torch.uint8).pin_memory()
    hout = torch.empty(pb, dtype=torch.uint8).pin_memory()

    def copies():
        with torch.cuda.stream(s1):
            dx.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(dz, non_blocking=True)
        torch.cuda.synchronize()

    def h2d_only():
        dx.copy_(hin, non_blocking=True)
        torch.cuda.synchronize()

    print(f"raw H2D {2 * pb >> 20} MiB: best {timed(h2d_only)[0]:.3f} ms; "
          f"H2D || D2H {pb >> 20} MiB: best {timed(copies)[0]:.3f} ms")
    for p in (hx, hy, hz):
        L.bfp_host_free(p)


if __name__ == "__main__":
    main()
