"""Exhaustive parity over ALL 2^32 operand pairs of 16-bit formats, through
the C ABI, against the oracle (the C restatement, itself pinned to the
reference in tests/test_oracle.py).

About 16 s per case on a 16-core GPU host.  Five RN + gradual cases run by
default (BFP_EXHAUSTIVE16=0 skips them); BFP_EXHAUSTIVE16=all runs every
16-bit format x add/sub/mul/div x rounding x subnormal mode (48 cases).  Log of a run: profiles/r01_exhaustive16.log.
The device side generates the pairs in place (x = block of 256 values, y =
all 65536) and compares the result planes' encodings against oracle chunks
computed on a thread pool (ctypes releases the GIL).
"""
from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

import paper_1602_04716_b200 as bfp

MODE = os.environ.get("BFP_EXHAUSTIVE16", "1")
pytestmark = [pytest.mark.gpu, pytest.mark.slow,
              pytest.mark.skipif(MODE == "0", reason="BFP_EXHAUSTIVE16=0")]

CASES = [("mul", (5, 10, 1, 0)), ("add", (5, 10, 1, 0)), ("mul", (6, 9, 1, 0)),
         ("mul", (8, 7, 1, 0)), ("div", (5, 10, 1, 0))]
if MODE == "all":  # every 16-bit format x add/sub/mul/div x RN/RZ x gradual/FTZ (48 cases)
    CASES = [(op, (e, s, rn, ftz)) for (e, s) in ((5, 10), (6, 9), (8, 7)) for op in ("add", "sub", "mul", "div")
             for (rn, ftz) in ((1, 0), (0, 0), (1, 1), (0, 1))]
XB = 256  # x values per chunk -> 2^24 pairs


@pytest.mark.parametrize("op,fmt", CASES,
                         ids=[f"{o}_{f[0]}_{f[1]}_{'rn' if f[2] else 'rz'}{'_ftz' if f[3] else ''}" for o, f in CASES])
def test_all_pairs_16bit(oracle, op, fmt):
    e, s, rn, ftz = fmt
    assert 1 + e + s == 16
    spec = bfp.make_spec(e, s, rn, ftz)
    fn = {"add": bfp.bfp_add, "sub": bfp.bfp_sub, "mul": bfp.bfp_mul, "div": bfp.bfp_div}[op]
    ys = np.arange(1 << 16, dtype=np.uint64)
    yd = torch.arange(1 << 16, dtype=torch.int64, device="cuda").repeat(XB)
    vy = bfp.pack(yd, spec)

    def want(x0: int) -> np.ndarray:
        x = np.repeat(np.arange(x0, x0 + XB, dtype=np.uint64), 1 << 16)
        return oracle.binop(op, fmt, x, np.tile(ys, XB)).astype(np.uint16)

    t0 = time.time()
    bad = 0
    # bounded: <= 16 oracle threads (~256 MB of operands each while running)
    # and a window of workers + 2 chunks of results in flight
    workers = max(1, min(16, (os.cpu_count() or 2) - 1))
    win = workers + 2
    starts = list(range(0, 1 << 16, XB))
    with ThreadPoolExecutor(max_workers=workers) as ex:
        futs = {x0: ex.submit(want, x0) for x0 in starts[:win]}
        for k, x0 in enumerate(starts):
            if k + win < len(starts):
                futs[starts[k + win]] = ex.submit(want, starts[k + win])
            fut = futs.pop(x0)
            xd = torch.arange(x0, x0 + XB, dtype=torch.int64, device="cuda").repeat_interleave(1 << 16)
            got = bfp.unpack(fn(bfp.pack(xd, spec), vy)).cpu().numpy().view(np.uint16)
            w = fut.result()
            if not np.array_equal(got, w):
                idx = np.nonzero(got != w)[0][:5]
                bad += int((got != w).sum())
                print(f"{op} {fmt}: mismatches at x={x0 + idx // 65536} y={idx % 65536}: "
                      f"got {got[idx]} want {w[idx]}")
    print(f"{op} 1/{e}/{s} rn={rn} ftz={ftz}: all 2^32 pairs, {bad} mismatches, {time.time() - t0:.1f} s")
    assert bad == 0
