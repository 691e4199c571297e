"""PCIe pipeline probe: where the host-buffer path's time goes at C2 size
(2 x 64 MiB in, 2 x 64 MiB out per step), copies only, pinned memory.

    python tools/pcie_probe.py [--mib 64] [--reps 5]

Patterns (each best of reps, wall clock around a synchronize):
  bulk_in      : the 2 inputs H2D, one copy each
  bulk_both    : 2 inputs H2D || 2 outputs D2H on two streams
  chunked_in C : the inputs in C chunks, one stream (in order)
  chunked_both C: C chunks in order per direction, H2D and D2H on two streams,
                 chunk k's D2H after chunk k's H2D (event), like the pipeline
  zero-copy    : bfp_mul / bfp_sub launched directly on pinned host planes
                 (the kernels read and write host memory over PCIe)
"""
from __future__ import annotations

import argparse
import time


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=64)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch
    nb = a.mib << 20
    hin = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(2)]
    hout = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(2)]
    din = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(2)]
    dout = [torch.empty(nb, dtype=torch.uint8, device="cuda") for _ in range(2)]
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(a.reps):
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t)
        return best * 1e3

    def bulk_in():
        with torch.cuda.stream(s_in):
            for i in range(2):
                din[i].copy_(hin[i], non_blocking=True)

    def bulk_both():
        with torch.cuda.stream(s_in):
            for i in range(2):
                din[i].copy_(hin[i], non_blocking=True)
        with torch.cuda.stream(s_out):
            for i in range(2):
                hout[i].copy_(dout[i], non_blocking=True)

    def chunked(c, both):
        def fn():
            step = nb // c
            for k in range(c):
                sl = slice(k * step, (k + 1) * step)
                with torch.cuda.stream(s_in):
                    for i in range(2):
                        din[i][sl].copy_(hin[i][sl], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(s_in)
                if both:
                    s_out.wait_event(ev)
                    with torch.cuda.stream(s_out):
                        for i in range(2):
                            hout[i][sl].copy_(dout[i][sl], non_blocking=True)
        return fn

    gb = 2 * nb / 1e9
    t = timed(bulk_in)
    print(f"bulk_in        {t:8.3f} ms  {gb / t * 1e3:6.1f} GB/s")
    t = timed(bulk_both)
    print(f"bulk_both      {t:8.3f} ms  {2 * gb / t * 1e3:6.1f} GB/s (both directions)")
    for c in (4, 8, 16, 32, 64):
        t1 = timed(chunked(c, False))
        t2 = timed(chunked(c, True))
        print(f"chunks {c:3d}: in {t1:8.3f} ms ({gb / t1 * 1e3:5.1f} GB/s)  both {t2:8.3f} ms "
              f"({2 * gb / t2 * 1e3:5.1f} GB/s)", flush=True)
    zero_copy(a.mib, a.reps)


def zero_copy(mib: int, reps: int) -> None:
    import ctypes as C
    import sys
    from pathlib import Path
    import torch
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    import paper_1602_04716_b200 as bfp
    L = bfp.lib()
    spec = bfp.make_spec(4, 3)
    n = (mib << 20)  # 1 byte per element
    pb = spec.plane_bytes(n)
    hx, hy, hz1, hz2 = (L.bfp_host_alloc(pb) for _ in range(4))
    C.memset(hx, 0x3c, pb)
    C.memset(hy, 0x5a, pb)
    st = torch.cuda.current_stream().cuda_stream

    def one():
        assert L.bfp_mul(spec.c, hx, hy, hz1, n, st) == 0

    def two():
        assert L.bfp_mul(spec.c, hx, hy, hz1, n, st) == 0
        assert L.bfp_sub(spec.c, hx, hy, hz2, n, st) == 0

    for name, fn, bi, bo in (("mul", one, 2 * pb, pb), ("mul+sub", two, 4 * pb, 2 * pb)):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t)
        print(f"zero-copy {name:8s} {best * 1e3:8.3f} ms  in {bi / best / 1e9:5.1f} GB/s  "
              f"out {bo / best / 1e9:5.1f} GB/s  -> {n / best / 1e9:6.2f} Gelem/s per op", flush=True)
    for p in (hx, hy, hz1, hz2):
        L.bfp_host_free(p)
    # write-only / read-only zero copy: unpack_f32 device planes -> pinned host
    # floats, pack_f32 pinned host floats -> device planes, vs plain copies
    n = 1 << 26
    spec = bfp.make_spec(5, 10)
    dpl = torch.zeros(spec.plane_bytes(n) // 4, dtype=torch.int32, device="cuda")
    dfl = torch.zeros(n, dtype=torch.float32, device="cuda")
    hfl = L.bfp_host_alloc(4 * n)
    hflt = torch.empty(n, dtype=torch.float32).pin_memory()

    def tm(fn):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t)
        return best

    t = tm(lambda: L.bfp_unpack_f32(spec.c, dpl.data_ptr(), hfl, n, st))
    print(f"kernel writes host  {4 * n / t / 1e9:6.1f} GB/s (unpack_f32 -> pinned floats)")
    t = tm(lambda: hflt.copy_(dfl, non_blocking=True))
    print(f"D2H copy            {4 * n / t / 1e9:6.1f} GB/s")
    t = tm(lambda: L.bfp_pack_f32(spec.c, hfl, dpl.data_ptr(), n, st))
    print(f"kernel reads host   {4 * n / t / 1e9:6.1f} GB/s (pack_f32 <- pinned floats)")
    t = tm(lambda: dfl.copy_(hflt, non_blocking=True))
    print(f"H2D copy            {4 * n / t / 1e9:6.1f} GB/s")
    L.bfp_host_free(hfl)


if __name__ == "__main__":
    main()
