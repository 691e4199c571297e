"""Small runs of every kernel family for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck), checked bit-exactly against the oracle so
a sanitizer-clean run is also a correct one:

    compute-sanitizer --tool memcheck  --error-exitcode 9 python tools/sanitize_kernels.py
    compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_kernels.py
    BFP_BULK=2 compute-sanitizer --tool racecheck ... python tools/sanitize_kernels.py --bulk

Covers the shared-memory tile layout kernels (k_pack_enc / k_unpack_enc /
k_pack_f32 / k_unpack_f32: warp_load_elems / warp_store_elems), the fused
float32 kernel (k_arith_f32), the arithmetic kernel (k_arith) and -- with
BFP_BULK=2 -- the cp.async.bulk + mbarrier ring (k_arith_bulk), on ragged
counts and unaligned element buffers.  Log: profiles/r02_sanitizer.log.
"""
from __future__ import annotations

import argparse
import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--bulk", action="store_true", help="expect BFP_BULK=2 (the bulk-copy ring)")
    a = ap.parse_args()
    import torch
    import oracle as O  # the checker
    import paper_1602_04716_b200 as bfp
    from paper_1602_04716_b200 import _lib

    L = _lib.lib()
    st = torch.cuda.current_stream().cuda_stream
    rng = np.random.default_rng(1)
    checked = 0
    for (e, s) in ((4, 3), (5, 10), (8, 15)):
        nb = 1 + e + s
        fmt = (e, s, 1, 0)
        spec = bfp.make_spec(e, s)
        for n in (1, 33, 1000, 5 * 1024 + 77, 148 * 1024 * 3 + 5):
            # raw encodings through unaligned buffers (one element past an aligned base)
            enc = rng.integers(0, 1 << nb, size=n, dtype=np.uint64)
            t = torch.from_numpy(enc.astype(np.int64)).cuda()
            v = bfp.pack(t, spec)
            assert np.array_equal(v.planes.cpu().numpy().view(np.uint32), O.pack_planes(enc, nb)), (fmt, n)
            assert np.array_equal(bfp.to_u64(bfp.unpack(v), spec).cpu().numpy().view(np.uint64), enc)
            eb = spec.enc_bytes()
            dt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[eb]
            buf = torch.zeros(n + 4, dtype=dt, device="cuda")
            buf[1:n + 1] = bfp.unpack(v).to(dt)
            vu = bfp.empty(spec, n)
            assert L.bfp_pack_enc(spec.c, buf[1:].data_ptr(), vu.planes.data_ptr(), n, st) == 0
            assert torch.equal(vu.planes, v.planes)
            # float32 codec
            xs = (rng.standard_normal(n) * 50).astype(np.float32)
            vf = bfp.pack_f32(torch.from_numpy(xs).cuda(), spec)
            want = O.encode_f32(fmt, xs)
            assert np.array_equal(vf.planes.cpu().numpy().view(np.uint32), O.pack_planes(want, nb))
            back = bfp.unpack_f32(vf).cpu().numpy().view(np.uint32)
            assert np.array_equal(back, O.decode_f32(fmt, want).view(np.uint32))
            # arithmetic (k_arith, or k_arith_bulk under BFP_BULK=2) and the fused float32 kernel
            ys = (rng.standard_normal(n) * 50).astype(np.float32)
            vy = bfp.pack_f32(torch.from_numpy(ys).cuda(), spec)
            wy = O.encode_f32(fmt, ys)
            for op in ("add", "mul", "mul_add"):
                z = bfp.arith({"add": 0, "mul": 2, "mul_add": 4}[op], vf, vy, vy if op == "mul_add" else None)
                got = O.unpack_planes(z.planes.cpu().numpy().view(np.uint32), n, nb)
                assert np.array_equal(got, O.binop(op, fmt, want, wy, wy if op == "mul_add" else None)), (op, n)
            zf = bfp.arith_f32(2, spec, torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda())
            assert np.array_equal(zf.cpu().numpy().view(np.uint32),
                                  O.decode_f32(fmt, O.binop("mul", fmt, want, wy)).view(np.uint32))
            checked += 1
    torch.cuda.synchronize()
    print(f"sanitize_kernels ok: {checked} (format, count) cases, bulk={a.bulk}, "
          f"{L.bfp_launch_count()} kernel launches")


if __name__ == "__main__":
    main()
