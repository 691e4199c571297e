"""Multi-GPU host logic on CPU: world_size-2 `gloo` processes each own a
contiguous, block-aligned shard (workloads.shard), evaluate
the C5 chain on it with the same networks the kernels use (host build), and
the concatenation of shards equals the unsharded result -- there is no
exchange step.  Also checks the max-over-ranks timing reduction bench.py
uses."""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT

sys.path.insert(0, str(ROOT))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, n: int, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, str(ROOT / "tests"))
    sys.path.insert(0, str(ROOT / "oracle"))
    from conftest import HostCircuits
    import oracle as O
    from paper_1602_04716_b200 import workloads as W

    host = HostCircuits()
    fmt = (6, 9, 1, 0)
    lo, hi = W.shard(n, rank, world)
    ops = [O.encode_f32(fmt, W.c5_floats(lo, hi, sd, "cpu").numpy())
           for sd in (W.SEED_A, W.SEED_B, W.SEED_C)]
    planes = [O.pack_planes(v, 16) for v in ops]
    z = host.binop("mul_add", fmt, *planes)
    # gather shard results (sizes differ only in the last shard)
    t = torch.from_numpy(z.view(np.int32).copy())
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([t.numel()]))
    mx = int(max(s.item() for s in sizes))
    padded = torch.zeros(mx, dtype=torch.int32)
    padded[: t.numel()] = t
    got = [torch.zeros(mx, dtype=torch.int32) for _ in range(world)]
    dist.all_gather(got, padded)
    # max-over-ranks timing reduction used by bench.py
    tm = torch.tensor([float(rank + 1)])
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    if rank == 0:
        cat = np.concatenate([g[: int(s.item())].numpy() for g, s in zip(got, sizes)]).view(np.uint32)
        out_q.put((cat, float(tm.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_concatenate(oracle, host):
    n = 5 * 1024 + 300
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    cat, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert tmax == float(world)
    from paper_1602_04716_b200 import workloads as W
    fmt = (6, 9, 1, 0)
    full = [oracle.encode_f32(fmt, W.c5_floats(0, n, sd, "cpu").numpy())
            for sd in (W.SEED_A, W.SEED_B, W.SEED_C)]
    want = host.binop("mul_add", fmt, *[oracle.pack_planes(v, 16) for v in full])
    assert np.array_equal(cat, want)
    # and against the oracle's own chain
    z = oracle.unpack_planes(cat, n, 16)
    assert np.array_equal(z, oracle.binop("mul_add", fmt, *full))


def test_shard_ranges_cover_and_align():
    from paper_1602_04716_b200 import workloads as W
    for n in (1, 1023, 1024, 5000, 1 << 20, (1 << 32)):
        for world in (1, 2, 3, 4, 8):
            rs = [W.shard(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            for (a, b), (c, d) in zip(rs, rs[1:]):
                assert b == c and a % 1024 == 0
