"""Guard-page ("electric fence") run of every kernel family -- TEST HARNESS,
run as a subprocess by tests/test_gpu_guard.py (compute-sanitizer is closed
on the GPU pool, so out-of-bounds accesses are caught by the MMU instead).

Every input and output buffer of a call is mapped with the CUDA virtual
memory API (cuMemAddressReserve / cuMemCreate / cuMemMap) so that it ends
exactly at the end of its mapped pages ("end" placement) or starts exactly at
their beginning ("start" placement), with unmapped guard pages on both sides:
any load or store past either end of the buffer the call was given faults
(illegal address), whatever the offset.  Each call's result is also compared
byte for byte with the same call on ordinary torch buffers.

    python tests/fence_kernels.py [--quick]        (exit 0 = no fault, all equal)
"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    import torch
    from cuda.bindings import driver as cu
    import paper_1602_04716_b200 as bfp
    from paper_1602_04716_b200 import _lib

    torch.cuda.init()
    torch.zeros(1, device="cuda")  # primary context current
    L = _lib.lib()

    def ck(r):
        err = r[0] if isinstance(r, tuple) else r
        if err != cu.CUresult.CUDA_SUCCESS:
            raise RuntimeError(f"CUDA driver error {err}")
        return r[1] if isinstance(r, tuple) and len(r) > 1 else None

    prop = cu.CUmemAllocationProp()
    prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = torch.cuda.current_device()
    G = ck(cu.cuMemGetAllocationGranularity(
        prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_MINIMUM))
    acc = cu.CUmemAccessDesc()
    acc.location = prop.location
    acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE

    class Fenced:
        """nbytes of device memory with unmapped guard pages on both sides."""

        def __init__(self, nbytes: int, place: str):
            self.n = max(nbytes, 1)
            self.m = -(-self.n // G) * G
            self.va = int(ck(cu.cuMemAddressReserve(self.m + 2 * G, 0, 0, 0)))
            self.h = ck(cu.cuMemCreate(self.m, prop, 0))
            ck(cu.cuMemMap(self.va + G, self.m, 0, self.h, 0))
            ck(cu.cuMemSetAccess(self.va + G, self.m, [acc], 1))
            self.ptr = self.va + G + (self.m - self.n if place == "end" else 0)

        def put(self, arr: np.ndarray):
            arr = np.ascontiguousarray(arr)
            assert arr.nbytes == self.n or (arr.nbytes == 0 and self.n == 1)
            if arr.nbytes:
                ck(cu.cuMemcpyHtoD(self.ptr, arr.ctypes.data, arr.nbytes))
            return self

        def get(self) -> np.ndarray:
            out = np.zeros(self.n, dtype=np.uint8)
            ck(cu.cuMemcpyDtoH(out.ctypes.data, self.ptr, self.n))
            return out

        def free(self):
            ck(cu.cuMemUnmap(self.va + G, self.m))
            ck(cu.cuMemRelease(self.h))
            ck(cu.cuMemAddressFree(self.va, self.m + 2 * G))

    rng = np.random.default_rng(0xFE7CE)
    sizes = [1, 33, 1000, 1024, 5 * 1024 + 77] + ([] if a.quick else [148 * 1024 * 2 + 3])
    fmts = [(4, 3), (5, 10), (8, 15), (11, 52)]
    checked = 0

    def run(name, fn, ins: list[np.ndarray], out_bytes: list[int]):
        """fn(in_ptrs, out_ptrs) -> status, on fenced buffers (both placements)
        and on torch buffers; outputs must agree byte for byte."""
        nonlocal checked
        tin = [torch.from_numpy(x.view(np.uint8).copy()).cuda() for x in ins]
        tout = [torch.zeros(max(nb, 1), dtype=torch.uint8, device="cuda") for nb in out_bytes]
        rc = fn([t.data_ptr() for t in tin], [t.data_ptr() for t in tout])
        assert rc == 0, (name, rc, L.bfp_last_error())
        torch.cuda.synchronize()
        want = [t.cpu().numpy()[:nb] for t, nb in zip(tout, out_bytes)]
        for place in ("end", "start"):
            fi = [Fenced(x.nbytes, place).put(x.view(np.uint8)) for x in ins]
            fo = [Fenced(nb, place) for nb in out_bytes]
            rc = fn([f.ptr for f in fi], [f.ptr for f in fo])
            assert rc == 0, (name, place, rc, L.bfp_last_error())
            ck(cu.cuCtxSynchronize())  # an out-of-bounds access faults here
            for f, w, nb in zip(fo, want, out_bytes):
                got = f.get()[:nb]
                assert np.array_equal(got, w), f"{name} ({place}): result differs"
            for f in fi + fo:
                f.free()
        checked += 1

    for (e, s) in fmts:
        nb = 1 + e + s
        spec = bfp.make_spec(e, s)
        f = spec.c
        eb = spec.enc_bytes()
        stride = int(L.bfp_bfpraw_stride(f))
        for n in sizes:
            pb = int(L.bfp_plane_bytes(f, n))
            enc = rng.integers(0, 1 << min(nb, 63), size=n, dtype=np.uint64)
            enc_b = enc.view(np.uint8).reshape(n, 8)[:, :eb].copy().reshape(-1)
            planes = np.zeros(pb, dtype=np.uint8)
            # planes of enc via the plain path (the fenced pack must reproduce them)
            t_enc = torch.from_numpy(enc_b).cuda()
            t_pl = torch.zeros(pb, dtype=torch.uint8, device="cuda")
            assert L.bfp_pack_enc(f, t_enc.data_ptr(), t_pl.data_ptr(), n, None) == 0
            planes = t_pl.cpu().numpy()
            tag = f"1/{e}/{s} n={n}"
            run(f"pack_enc {tag}", lambda i, o: L.bfp_pack_enc(f, i[0], o[0], n, None), [enc_b], [pb])
            run(f"unpack_enc {tag}", lambda i, o: L.bfp_unpack_enc(f, i[0], o[0], n, None), [planes], [n * eb])
            raw = np.zeros(n * stride, dtype=np.uint8)
            raw[:] = rng.integers(0, 256, size=n * stride, dtype=np.uint8)
            if nb % 8:  # the unused top bits of each record are zero
                rr = raw.reshape(n, stride)
                rr[:, -1] &= (1 << (nb % 8)) - 1
            run(f"pack_bfpraw {tag}", lambda i, o: L.bfp_pack_bfpraw(f, i[0], n * stride, o[0], None), [raw], [pb])
            run(f"unpack_bfpraw {tag}", lambda i, o: L.bfp_unpack_bfpraw(f, i[0], n, o[0], None), [planes],
                [n * stride])
            xs64 = rng.standard_normal(n) * 30
            run(f"pack_f64 {tag}", lambda i, o: L.bfp_pack_f64(f, i[0], o[0], n, None), [xs64], [pb])
            run(f"unpack_f64 {tag}", lambda i, o: L.bfp_unpack_f64(f, i[0], o[0], n, None), [planes], [8 * n])
            ys = rng.integers(0, 1 << min(nb, 63), size=n, dtype=np.uint64)
            t2 = torch.from_numpy(ys.view(np.uint8).reshape(n, 8)[:, :eb].copy().reshape(-1)).cuda()
            t_pl2 = torch.zeros(pb, dtype=torch.uint8, device="cuda")
            assert L.bfp_pack_enc(f, t2.data_ptr(), t_pl2.data_ptr(), n, None) == 0
            planes2 = t_pl2.cpu().numpy()
            for op in range(5):
                run(f"arith op{op} {tag}",
                    lambda i, o, op=op: L.bfp_arith(op, f, i[0], i[1], i[2] if op == 4 else None, o[0], n, None),
                    [planes, planes2] + ([planes] if op == 4 else []), [pb])
            if e <= 8 and s <= 23:
                xs = (rng.standard_normal(n) * 30).astype(np.float32)
                ys32 = (rng.standard_normal(n) * 30).astype(np.float32)
                run(f"pack_f32 {tag}", lambda i, o: L.bfp_pack_f32(f, i[0], o[0], n, None), [xs], [pb])
                run(f"unpack_f32 {tag}", lambda i, o: L.bfp_unpack_f32(f, i[0], o[0], n, None), [planes], [4 * n])
                for op in (0, 2, 4):
                    run(f"arith_f32 op{op} {tag}",
                        lambda i, o, op=op: L.bfp_arith_f32(op, f, i[0], i[1], i[2] if op == 4 else None, o[0], n,
                                                            None),
                        [xs, ys32] + ([xs] if op == 4 else []), [4 * n])
            if not a.quick and nb <= 24:
                def chain(i, o):
                    arr = (C.c_void_p * 3)(*i)
                    return L.bfp_chain(f, b"ab*c+", 3, arr, o[0], n, None)
                run(f"chain {tag}", chain, [planes, planes2, planes], [pb])
    torch.cuda.synchronize()
    print(f"fence ok: {checked} calls x 2 placements, no out-of-bounds access, results equal "
          f"(granularity {G} B, BFP_BULK={os.environ.get('BFP_BULK', '0')})")


if __name__ == "__main__":
    main()
