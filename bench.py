#!/usr/bin/env python3
"""Benchmark of the B200 bitslice FP hot path (BASELINE.json metric:
"bitslice FP ops/sec (Gelem/s) per format vs LOP3/HBM roofline, 1/2/4/8 B200").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config default|C1..C5|X1..X3u|all] [--dry-run]

Default workload (`--config default`): the headline is configs[4] = C5, the
largest configuration that fits one GPU -- z = round(round(a*b) + c) in 1/6/9
(the reference chain bfp_add(bfp_mul(a, b), c), arith.hpp:235-373) over a
FIXED N = 2^32 elements split evenly over the GPUs (strong scaling, no
collective on the data path: SURVEY.md §8e); one step = one fused mul_add
launch per GPU over resident planes.  value = 2^32 / step time (max over
ranks), Gelem/s.  The same line carries C4's per-format sweep (add and mul
for 1/3/2, 1/5/3, 1/5/7, 1/8/7, 1/8/15 at 2^28 elements per GPU) and C5 in
`per_format`, each kernel with its binding roofline leg.

--gpus N with no torchrun environment re-launches itself through
torch.distributed.run with N ranks (one per GPU, NCCL for the barrier and
the max-over-ranks times only).  --dry-run does the same with gloo on the
CPU and a stand-in step: it checks the launcher, the shard ranges, the
max-over-ranks reduction and the rank-0-only output without a GPU.

JSON line (rank 0): value (device, inputs resident in HBM), e2e (the same
step through the C ABI with pinned host buffers: H2D + kernel + D2H inside
the timed region), roofline (the dominant kernel on its BINDING leg: the
LOP3 issue rate against the measured probe peak, or HBM bytes against the
measured copy peak; DRAM traffic measured by an ncu subprocess in this run),
cpu_baseline (the reference itself -- oracle/_ref, the unmodified headers
compiled in place -- on the host cores, ~10 s, best and median), clocks
(nvidia-smi during a sustained window of the same step), gpu_launches.

--impl reference times the reference's own CPU implementation (oracle/_ref)
on this host's cores for the same config / metric; rank 0 only.
"""
from __future__ import annotations

import argparse
import csv
import ctypes as C
import faulthandler
import io
import json
import os
import re
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "bitslice FP ops/sec (Gelem/s) per format vs LOP3/HBM roofline"
UNIT = "Gelem/s"
OPNAMES = {"add": 0, "sub": 1, "mul": 2, "div": 3, "mul_add": 4}
L2_BYTES = 126 * 1024 * 1024

# (rn, ftz) of every config: the reference default RN + gradual
# (format.hpp:26-27); --rounding / --subnormals select the secondary rows.
MODE = (1, 0)


def log(msg: str) -> None:
    print(f"[bench r{os.environ.get('RANK', '0')}] {msg}", file=sys.stderr, flush=True)


def mode_text() -> str:
    return ("rn" if MODE[0] else "rz") + ("+ftz" if MODE[1] else "")


# ------------------------------------------------------- distributed plumbing
def env_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def maybe_relaunch(args) -> None:
    """--gpus N > 1 without a torchrun environment: run this script under
    torch.distributed.run with N ranks on this node and exit with its code."""
    if "WORLD_SIZE" in os.environ or args.gpus <= 1:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve())] + sys.argv[1:]
    log(f"launching {args.gpus} ranks: {' '.join(cmd[1:6])} ...")
    sys.exit(subprocess.run(cmd).returncode)


class Dist:
    """One process per GPU (gloo on the CPU for --dry-run).  Collectives are
    used only for the barrier around timed regions, the max-over-ranks times
    and the per-rank report -- never on the data path."""

    def __init__(self, backend: str):
        import torch
        import torch.distributed as dist
        self.world, self.rank, self.local = env_dist()
        self.backend = backend
        self.dist = dist if self.world > 1 else None
        self.dev = torch.device("cuda", self.local) if backend == "nccl" else torch.device("cpu")
        if self.world > 1:
            if backend == "nccl":
                os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator init on stderr
                os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
                torch.cuda.set_device(self.dev)
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group("gloo")
            assert dist.get_world_size() == self.world and dist.get_rank() == self.rank
            log(f"{backend} process group up: rank {self.rank}/{self.world}, device {self.dev}")

    def barrier(self) -> None:
        if self.dist:
            self.dist.barrier()

    def reduce(self, vals: list[float], op: str = "max") -> list[float]:
        if not self.dist:
            return list(vals)
        import torch
        t = torch.tensor(vals, dtype=torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return [float(v) for v in t.cpu()]

    def gather(self, obj) -> list:
        if not self.dist:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def close(self) -> None:
        if self.dist:
            self.dist.barrier()
            self.dist.destroy_process_group()


def measured_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
              "power.limit")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.rows: list[list[str]] = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.dev), "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) < 8:
                continue
            for nm, v in zip(names, r[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        num = lambda v: float(v) if v.replace(".", "", 1).isdigit() else None  # noqa: E731
        pw = [num(r[2]) for r in self.rows if len(r) >= 8 and num(r[2]) is not None]
        lim = [num(r[8]) for r in self.rows if len(r) >= 9 and num(r[8]) is not None]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons),
                "power_w": round(statistics.median(pw), 1) if pw else None,
                "power_limit_w": max(lim) if lim else None}


def clocks_rejected(c: dict) -> bool:
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    if bad & set(c.get("reasons", [])):
        return True
    if c.get("sm_mhz") and c.get("sm_max_mhz") and c["sm_mhz"] < 0.5 * c["sm_max_mhz"] \
            and not c.get("reasons"):
        return True
    return False


_SASS = None


def sass_lop3(fmt, rn, ftz, op: int, path: str = "fast") -> int | None:
    """Static LOP3 count of the shipped arithmetic kernel (one 32-element unit
    per loop iteration) from cuobjdump of the loaded library.  mul_add kernels
    hold two covers behind a warp-uniform branch; `path` picks the count of
    the instructions a unit executes on that side ("fast": the fast-domain
    cover, "general": the general one) -- tools/sass_stats.py, `paths`."""
    global _SASS
    try:
        if _SASS is None:
            sys.path.insert(0, str(ROOT / "tools"))
            import sass_stats
            _SASS = sass_stats.stats(pattern=r"k_arith")
        e, s = fmt
        key = f"k_arith<bfpg::Format<{e}, {s}, {'true' if rn else 'false'}, " \
              f"{'true' if ftz else 'false'}>, {op}>"
        for name, r in _SASS.items():
            if key in name:
                return r["paths"][path] if r.get("paths") else r["LOP3"]
    except (OSError, subprocess.SubprocessError, ValueError, KeyError):  # no cuobjdump / odd SASS
        return None
    return None


# ------------------------------------------------------------ the workloads
class Job:
    """One timed kernel of a step: `launch(i, stream)` issues it (i = step
    index: operand sets / outputs rotate with it).  `touch(i)` = (set id,
    bytes read from that set, bytes written) for the L2 reuse accounting."""

    def __init__(self, label, op, spec, n, launch, algo_bytes, host=None, touch=None, aux=None, info=None):
        self.label, self.op, self.spec, self.n = label, op, spec, n
        self.launch, self.algo_bytes, self.host = launch, algo_bytes, host
        # aux: {name: launch}: variants of this kernel timed on their own after the
        # step (same operands, never part of the step or of `value`)
        self.aux = aux or {}
        self.info = info or {}  # facts about the operands, copied into the kernel's per_format entry
        self.touch = touch or (lambda i, lb=label, b=algo_bytes: (lb, b, 0))  # fixed operands

    @property
    def fmt(self) -> str:
        return f"1/{self.spec.exp_bits}/{self.spec.sig_bits}"


class JobMeta:
    """What the report needs of a Job once its device operands are freed."""

    def __init__(self, j: Job):
        self.label, self.op, self.spec, self.n, self.algo_bytes = j.label, j.op, j.spec, j.n, j.algo_bytes
        self.fmt, self.info = j.fmt, dict(j.info)


def _chunked_pack_f32(gen, n, spec, device, chunk=1 << 27):
    """pack_f32 of gen(lo, hi) in block-aligned chunks (bounded temporaries)."""
    import torch
    import paper_1602_04716_b200 as bfp
    v = bfp.empty(spec, n, device)
    nb = spec.total_bits()
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        x = gen(lo, hi)
        w0 = (lo // 1024) * nb * 32
        sub = v.planes[w0:w0 + ((hi - lo + 1023) // 1024) * nb * 32]
        rc = bfp.lib().bfp_pack_f32(spec.c, x.data_ptr(), sub.data_ptr(), hi - lo,
                                    torch.cuda.current_stream().cuda_stream)
        if rc != 0:
            raise RuntimeError(bfp.lib().bfp_last_error())
        del x
    return v


def spec_of(e: int, s: int):
    import paper_1602_04716_b200 as bfp
    return bfp.make_spec(e, s, bfp.rounding_mode(MODE[0]), bfp.subnormal_policy(MODE[1]))


def rotation_sets(spec, n, n_inputs: int, launches_per_step: int = 1) -> int:
    """Operand sets rotated launch by launch so that a set is re-read only
    after >= 2x L2 of traffic: with k sets and one launch streaming (n_inputs
    + 1) planes of n elements, a set's first line comes back after k launches'
    reads and writes (its own launch's included)."""
    launch = (n_inputs + 1) * spec.plane_bytes(n)
    k = max(1, -(-2 * L2_BYTES // launch))
    # every launch of a step uses a different set, so k >= launches per step
    return max(k, launches_per_step)


def _arith_job(label, op, spec, n, sets, device, slot=0, stride=1):
    """sets: list of (a, b, c) operand tuples; launch i of this job uses set
    (stride * i + slot) mod len(sets) -- jobs of one step take different slots
    so no launch re-reads the set its predecessor just read."""
    import paper_1602_04716_b200 as bfp
    L = bfp.lib()
    outs = [bfp.empty(spec, n, device) for _ in range(2)]  # rotating outputs
    nin = 3 if sets[0][2] is not None else 2
    pb = spec.plane_bytes(n)

    def idx(i):
        return (stride * i + slot) % len(sets)

    def launch(i, st, flags=1):
        # resident operands that nothing in the step writes: BFP_INPUTS_READY
        # lets each kernel's first loads overlap its predecessor's tail
        a, b, c = sets[idx(i)]
        rc = L.bfp_arith_ex(OPNAMES[op], spec.c, a.planes.data_ptr(), b.planes.data_ptr(),
                            c.planes.data_ptr() if c is not None else None,
                            outs[i & 1].planes.data_ptr(), n, st, flags)
        if rc != 0:
            raise RuntimeError(L.bfp_last_error())

    # mul_add kernels pick one of two covers per warp (the fast-domain one when
    # the whole block is inside it: include/bfpgpu.h, BFP_GENERAL_NETWORK); the
    # general cover is timed on the same operands beside the step
    aux = {"general_network": lambda i, st: launch(i, st, 1 | 2)} if op == "mul_add" else None
    info = {}
    if op == "mul_add":  # which cover the launch's warps take: the library's own predicate + vote
        info["fast_cover_blocks_frac"] = round(bfp.mul_add_fast_blocks(*sets[0]) / max(1, -(-n // 1024)), 6)

    nbits = spec.total_bits()
    a, b, c = sets[0]
    return Job(label, op, spec, n, launch, (nin + 1) * nbits / 8 * n,
               host={"kind": "arith", "op": op, "inputs": [a, b] + ([c] if c is not None else []),
                     "sets": len(sets)},
               touch=lambda i: ((id(sets), idx(i)), nin * pb, pb), aux=aux, info=info)


def _clone_sets(first, k):
    return [first] + [tuple(v.clone() if v is not None else None for v in first) for _ in range(k - 1)]


X1_FMTS = [(3, 2), (4, 3), (5, 3), (5, 7), (5, 10), (8, 7), (8, 15)]
C4_FMTS = [(3, 2), (5, 3), (5, 7), (8, 7), (8, 15)]


def config_n(cfg: str, rank: int, world: int) -> tuple[int, int]:
    """Element range [lo, hi) of this rank: C5 splits a fixed 2^32 total over
    the ranks (strong scaling); every other config gives each rank its own
    block of the per-GPU N (weak scaling).  Both block-aligned, contiguous."""
    from paper_1602_04716_b200 import workloads as W
    if cfg == "C5":
        return W.shard(1 << 32, rank, world)
    n = CONFIG_TEXT[cfg][2]
    return rank * n, (rank + 1) * n


def make_jobs(cfg: str, rank: int, world: int, device) -> list:
    """Per-rank resident operands and the timed kernels of config `cfg`."""
    import torch
    import paper_1602_04716_b200 as bfp
    from paper_1602_04716_b200 import workloads as W

    L = bfp.lib()
    lo, hi = config_n(cfg, rank, world)
    n = hi - lo
    if cfg == "C1":
        spec = spec_of(4, 3)
        a = bfp.pack_f32(W.c1_floats(lo, hi, W.SEED_A, device), spec)
        b = bfp.pack_f32(W.c1_floats(lo, hi, W.SEED_B, device), spec)
        sets = _clone_sets((a, b, None), rotation_sets(spec, n, 2))  # same data, distinct buffers
        return [_arith_job("add", "add", spec, n, sets, device)]
    if cfg == "C2":
        spec = spec_of(4, 3)
        a = bfp.pack(W.c2_encodings(lo, hi, W.SEED_A, device), spec)
        b = bfp.pack(W.c2_encodings(lo, hi, W.SEED_B, device), spec)
        sets = _clone_sets((a, b, None), rotation_sets(spec, n, 2, launches_per_step=2))
        # mul takes even launches' sets, sub odd ones: the sub never re-reads
        # the operands the mul just streamed through L2
        return [_arith_job("mul", "mul", spec, n, sets, device, slot=0, stride=2),
                _arith_job("sub", "sub", spec, n, sets, device, slot=1, stride=2)]
    if cfg == "C3":
        spec = spec_of(5, 10)
        xa = W.c3_floats(lo, hi, W.SEED_A, device)
        xb = W.c3_floats(lo, hi, W.SEED_B, device)
        a, b = bfp.pack_f32(xa, spec), bfp.pack_f32(xb, spec)
        del xb
        torch.cuda.empty_cache()
        pk_out = [bfp.empty(spec, n, device) for _ in range(2)]
        up_out = [torch.empty(n, dtype=torch.float32, device=device) for _ in range(2)]

        def pack_launch(i, st):
            rc = L.bfp_pack_f32(spec.c, xa.data_ptr(), pk_out[i & 1].planes.data_ptr(), n, st)
            if rc != 0:
                raise RuntimeError(L.bfp_last_error())

        def unpack_launch(i, st):
            rc = L.bfp_unpack_f32(spec.c, a.planes.data_ptr(), up_out[i & 1].data_ptr(), n, st)
            if rc != 0:
                raise RuntimeError(L.bfp_last_error())

        nb = spec.total_bits()
        pb = spec.plane_bytes(n)
        return [Job("pack_f32", "pack_f32", spec, n, pack_launch, (4 + nb / 8) * n,
                    host={"kind": "pack_f32", "x": xa}, touch=lambda i: ("xa", 4 * n, pb)),
                _arith_job("add", "add", spec, n, [(a, b, None)], device),
                _arith_job("mul", "mul", spec, n, [(a, b, None)], device),
                Job("unpack_f32", "unpack_f32", spec, n, unpack_launch, (nb / 8 + 4) * n,
                    host={"kind": "unpack_f32", "v": a}, touch=lambda i: ("a", pb, 4 * n))]
    if cfg in ("C4", "X1"):
        jobs = []
        fmts = C4_FMTS if cfg == "C4" else X1_FMTS
        ops = ("add", "mul") if cfg == "C4" else ("div",)
        for (e, s) in fmts:
            spec = spec_of(e, s)
            a = bfp.pack(W.c4_encodings(e, s, lo, hi, W.SEED_A, device), spec)
            b = bfp.pack(W.c4_encodings(e, s, lo, hi, W.SEED_B, device), spec)
            torch.cuda.empty_cache()
            for op in ops:
                jobs.append(_arith_job(f"{op}_1/{e}/{s}", op, spec, n, [(a, b, None)], device))
        return jobs
    if cfg == "C5":
        spec = spec_of(6, 9)
        ops = [_chunked_pack_f32(lambda a_, b_, sd=sd: W.c5_floats(lo + a_, lo + b_, sd, device), n,
                                 spec, device)
               for sd in (W.SEED_A, W.SEED_B, W.SEED_C)]
        torch.cuda.empty_cache()
        return [_arith_job("mul_add", "mul_add", spec, n, [tuple(ops)], device)]
    if cfg == "X2":  # secondary: fused float32-in/out ops, C3 operands
        spec = spec_of(5, 10)
        xa = W.c3_floats(lo, hi, W.SEED_A, device)
        xb = W.c3_floats(lo, hi, W.SEED_B, device)
        outs = [torch.empty(n, dtype=torch.float32, device=device) for _ in range(2)]
        jobs = []
        for op in ("add", "mul"):
            def launch(i, st, op=op):
                rc = L.bfp_arith_f32(OPNAMES[op], spec.c, xa.data_ptr(), xb.data_ptr(), None,
                                     outs[i & 1].data_ptr(), n, st)
                if rc != 0:
                    raise RuntimeError(L.bfp_last_error())
            jobs.append(Job(f"{op}_f32", f"{op}_f32", spec, n, launch, 12 * n,
                            host={"kind": "none"}, touch=lambda i: ("x", 8 * n, 4 * n)))
        return jobs
    if cfg in ("X3", "X3u"):  # secondary: z = a*b + c*d, fused (bfp_chain) or as 3 kernels
        spec = spec_of(5, 10)
        vs = [bfp.pack(W.c4_encodings(5, 10, lo, hi, sd, device), spec)
              for sd in (W.SEED_A, W.SEED_B, W.SEED_C, W.SEED_C + 1)]
        torch.cuda.empty_cache()
        outs = [bfp.empty(spec, n, device) for _ in range(2)]
        nb = spec.total_bits()
        if cfg == "X3":
            ptrs = (C.c_void_p * 4)(*[v.planes.data_ptr() for v in vs])

            def launch(i, st):
                rc = L.bfp_chain(spec.c, b"ab*cd*+", 4, ptrs, outs[i & 1].planes.data_ptr(), n, st)
                if rc != 0:
                    raise RuntimeError(L.bfp_last_error())
            return [Job("a*b+c*d", "chain:ab*cd*+", spec, n, launch, 5 * nb / 8 * n, host={"kind": "none"})]
        t = [bfp.empty(spec, n, device) for _ in range(2)]

        def op(code, x, y, z):
            def launch(i, st):
                rc = L.bfp_arith(code, spec.c, x.planes.data_ptr(), y.planes.data_ptr(), None,
                                 z.planes.data_ptr(), n, st)
                if rc != 0:
                    raise RuntimeError(L.bfp_last_error())
            return launch
        return [Job("mul a*b", "mul", spec, n, op(2, vs[0], vs[1], t[0]), 3 * nb / 8 * n, host={"kind": "none"}),
                Job("mul c*d", "mul", spec, n, op(2, vs[2], vs[3], t[1]), 3 * nb / 8 * n, host={"kind": "none"}),
                Job("add", "add", spec, n, op(0, t[0], t[1], outs[0]), 3 * nb / 8 * n, host={"kind": "none"})]
    raise ValueError(cfg)


def l2_reuse_distance(jobs, steps: int = 128) -> int:
    """Smallest amount of traffic (bytes) between a read of an operand set's
    first line and its next read, over `steps` consecutive steps of the launch
    sequence: everything the reading launch streams after it plus every launch
    in between (-1 if no set is read twice in that window)."""
    seq = [j.touch(i) for i in range(steps) for j in jobs]
    best = None
    for p, (sid, _, _) in enumerate(seq):
        for q in range(p + 1, len(seq)):
            if seq[q][0] == sid:
                d = sum(r + w for _, r, w in seq[p:q])
                best = d if best is None else min(best, d)
                break
    return best if best is not None else -1


# ---------------------------------------------------------- device timing
def run_device(cfg: str, steps: int, warmup: int, D: Dist, jobs=None) -> dict:
    import torch
    import paper_1602_04716_b200 as bfp

    device = D.dev
    torch.cuda.set_device(device)
    L = bfp.lib()
    if jobs is None:
        jobs = make_jobs(cfg, D.rank, D.world, device)
    stream = torch.cuda.current_stream(device)
    st = stream.cuda_stream

    def step(i):
        for j in jobs:
            j.launch(i, st)

    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()

    # The K timed steps are issued through the C ABI exactly as a caller does,
    # captured once into a CUDA graph (launch-bound small steps such as C1 --
    # a 48 MiB, ~8 us kernel -- would otherwise measure the host's per-call
    # overhead, not the device) and replayed; consecutive kernels keep their
    # programmatic-dependent-launch edges inside the graph.
    cap = torch.cuda.Stream(device)

    def capture(fn) -> tuple:
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        l0 = L.bfp_launch_count()
        with torch.cuda.graph(g, stream=cap):
            fn(cap.cuda_stream)
        torch.cuda.synchronize()
        return g, L.bfp_launch_count() - l0

    def all_steps(s):
        for i in range(steps):
            for j in jobs:
                j.launch(i, s)

    g_all, launches = capture(all_steps)
    g_all.replay()  # untimed: graph upload + one more warm pass
    torch.cuda.synchronize()

    def timed_replay(g) -> float:
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        D.barrier()
        torch.cuda.synchronize()
        t0.record(stream)  # replay() launches the graph on the current stream
        g.replay()
        t1.record(stream)
        torch.cuda.synchronize()
        D.barrier()
        return t0.elapsed_time(t1)

    # Timed region (the value): K whole steps, back to back, bracketed by a
    # barrier + synchronize on both sides; nvidia-smi samples the clocks
    # during it and during a sustained window of the same graph (~1.5 s).
    t_probe = time.perf_counter()
    g_all.replay()
    torch.cuda.synchronize()
    one = max(time.perf_counter() - t_probe, 1e-5)
    with ClockSampler(local_index(device)) as cs:
        ms_total = timed_replay(g_all)
        for _ in range(max(1, int(1.5 / one))):
            g_all.replay()
        torch.cuda.synchronize()
    clocks = cs.summary()
    ms_rank = ms_total
    ms_total = D.reduce([ms_total])[0]
    # The same K steps issued eagerly (one host call per kernel), for reference.
    te0, te1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    te0.record(stream)
    for i in range(steps):
        step(i)
    te1.record(stream)
    torch.cuda.synchronize()
    ms_total_eager = te0.elapsed_time(te1)
    # Per-kernel durations (the roofline): for each kernel of the step, a graph
    # of its K launches (same rotating operands) timed with events around the
    # replay on the launching stream -> mean launch duration, max over ranks.
    kern_ms = []
    for j in jobs:
        g, _ = capture(lambda s, j=j: [j.launch(i, s) for i in range(steps)])
        g.replay()
        torch.cuda.synchronize()
        kern_ms.append(timed_replay(g) / steps)
        del g
    kern_ms = D.reduce(kern_ms)
    # variants of a kernel (the general mul_add cover), timed the same way
    aux_ms = {}
    for j in jobs:
        for name, fn in j.aux.items():
            g, _ = capture(lambda s, fn=fn: [fn(i, s) for i in range(steps)])
            g.replay()
            torch.cuda.synchronize()
            aux_ms[f"{j.label}:{name}"] = D.reduce([timed_replay(g) / steps])[0]
            del g
    del g_all
    return {"jobs": jobs, "ms_total": ms_total, "ms_total_rank": ms_rank, "kern_ms": kern_ms,
            "clocks": clocks, "launches": int(launches), "ms_total_eager": ms_total_eager,
            "aux_ms": aux_ms}


def local_index(device) -> int:
    """nvidia-smi index of a torch device (honours CUDA_VISIBLE_DEVICES)."""
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    idx = device.index or 0
    if vis:
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        if idx < len(ids) and ids[idx].isdigit():
            return int(ids[idx])
    return idx


def run_e2e(jobs, steps: int, D: Dist) -> dict | None:
    """The same step through the C ABI with HOST buffers (pinned): every step
    copies its inputs H2D and its results D2H inside the timed region."""
    import torch
    import paper_1602_04716_b200 as bfp

    L = bfp.lib()
    ctx = L.bfp_host_ctx_create(int(os.environ.get("BFP_E2E_CHUNK", 1 << 24)))
    bufs = []

    def pinned(nbytes):
        p = L.bfp_host_alloc(nbytes)
        if not p:
            raise RuntimeError("bfp_host_alloc failed")
        bufs.append(p)
        return p

    def host_copy(t: torch.Tensor, chunk: int = 1 << 30):
        nbytes = t.numel() * t.element_size()
        p = pinned(nbytes)
        flat = t.reshape(-1).view(torch.uint8)
        for o in range(0, nbytes, chunk):  # bounded pageable temporaries
            src = flat[o:o + chunk].cpu().numpy()
            C.memmove(p + o, src.ctypes.data, src.nbytes)
        return p

    try:
        calls = []  # (fn, h2d bytes, d2h bytes, elements)
        groups = []  # arith jobs sharing the same operand tensors -> one batched call
        for j in jobs:
            if (j.host["kind"] == "arith" and groups and groups[-1][0].host["kind"] == "arith"
                    and all(a is b for a, b in zip(groups[-1][0].host["inputs"], j.host["inputs"]))
                    and len(groups[-1][0].host["inputs"]) == len(j.host["inputs"])):
                groups[-1].append(j)
            else:
                groups.append([j])
        for grp in groups:
            j = grp[0]
            spec, n = j.spec, j.n
            pb = spec.plane_bytes(n)
            if j.host["kind"] == "arith":
                hin = [host_copy(v.planes) for v in j.host["inputs"]]
                hz = [pinned(pb) for _ in grp]
                hc = hin[2] if len(hin) > 2 else None
                ops = (C.c_int * len(grp))(*[OPNAMES[g.op] for g in grp])
                outs = (C.c_void_p * len(grp))(*hz)
                calls.append((lambda spec=spec, hin=hin, hc=hc, ops=ops, outs=outs, n=n, k=len(grp):
                              L.bfp_arith_host_batch(ctx, k, ops, spec.c, hin[0], hin[1], hc, outs, n),
                              len(hin) * pb, len(grp) * pb, len(grp) * n))
            elif j.host["kind"] == "pack_f32":
                hx = host_copy(j.host["x"])
                hz = pinned(pb)
                calls.append((lambda spec=spec, hx=hx, hz=hz, n=n:
                              L.bfp_pack_f32_host(ctx, spec.c, hx, hz, n), 4 * n, pb, n))
            elif j.host["kind"] == "unpack_f32":
                hp = host_copy(j.host["v"].planes)
                hz = pinned(4 * n)
                calls.append((lambda spec=spec, hp=hp, hz=hz, n=n:
                              L.bfp_unpack_f32_host(ctx, spec.c, hp, hz, n), pb, 4 * n, n))
        torch.cuda.empty_cache()
        if not calls:  # no host-buffer entry point for these kernels (X2, X3)
            return None

        def step():
            for fn, _, _, _ in calls:
                rc = fn()
                if rc != 0:
                    raise RuntimeError(L.bfp_last_error())

        step()
        k = max(2, min(steps // 4, 10))
        D.barrier()
        t = time.perf_counter()
        for _ in range(k):
            step()
        dt = (time.perf_counter() - t) / k
        dt = D.reduce([dt])[0]
        return {"s_per_step": dt, "h2d": sum(c[1] for c in calls),
                "d2h": sum(c[2] for c in calls), "elems": sum(c[3] for c in calls), "steps": k}
    finally:
        for p in bufs:
            L.bfp_host_free(p)
        L.bfp_host_ctx_destroy(ctx)


def hbm_2r1w_probe(dev, nbytes: int = 1 << 30) -> float:
    """HBM rate of a plain 2-read : 1-write stream (torch bitwise_xor over
    1 GiB int32 operands, best of 10 by CUDA events) -- the access mix of a
    binary op.  MEASURED_PEAKS.json's copy is 1:1, which HBM serves slightly
    slower, so the binary-op kernels can exceed it; this is the context."""
    import torch
    n = nbytes // 4
    a = torch.randint(0, 1 << 30, (n,), dtype=torch.int32, device=dev)
    b = torch.randint(0, 1 << 30, (n,), dtype=torch.int32, device=dev)
    c = torch.empty_like(a)
    best = 1e9
    for _ in range(12):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.bitwise_xor(a, b, out=c)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b, c
    torch.cuda.empty_cache()
    return round(3 * nbytes / (best * 1e-3) / 1e9, 1)


def pcie_probe(dev, nbytes: int = 1 << 28) -> dict:
    """Pinned-host <-> device copy bandwidth on this box (the e2e ceiling):
    H2D alone, D2H alone, and both directions at once on two streams."""
    import torch
    h_in = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    d_b = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)

    def timed(fn, reps=3):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize(dev)
            t = time.perf_counter()
            fn()
            torch.cuda.synchronize(dev)
            best = min(best, time.perf_counter() - t)
        return best

    def h2d():
        d_a.copy_(h_in, non_blocking=True)

    def d2h():
        h_out.copy_(d_b, non_blocking=True)

    def both():
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)

    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    return {"h2d_gbs": round(nbytes / t1 / 1e9, 1), "d2h_gbs": round(nbytes / t2 / 1e9, 1),
            "bidir_gbs": round(2 * nbytes / t3 / 1e9, 1)}


def lop3_peak(dev) -> dict | None:
    """LOP3 issue rate of the probe kernel (bfp_probe_lop3: 8 independent
    chains per thread on every SM).  burst = one launch on a cool GPU (the
    clock ceiling; the roofline denominator); sustained = back-to-back
    launches for ~2 s, median of the second half, with the SM clock it
    settled at (the register-only probe is not power-capped and settles at
    the ceiling, so load-clock fractions scale it to the kernels' clock)."""
    import paper_1602_04716_b200 as bfp
    L = bfp.lib()
    ms, rate = C.c_float(), C.c_double()
    if L.bfp_probe_lop3(4000, C.byref(ms), C.byref(rate)) != 0:
        return None
    burst = rate.value
    rates = []
    with ClockSampler(local_index(dev)) as cs:
        t = time.perf_counter()
        while time.perf_counter() - t < 2.0:
            if L.bfp_probe_lop3(4000, C.byref(ms), C.byref(rate)) != 0:
                return None
            rates.append(rate.value)
    sus = statistics.median(rates[len(rates) // 2:])
    return {"burst": burst, "sustained": sus, "sustained_sm_mhz": cs.summary().get("sm_mhz")}


# ------------------------------------------- DRAM traffic, measured in-run
def _under_profiler() -> bool:
    return any(k in os.environ for k in ("CUDA_INJECTION64_PATH", "NV_TPS_LAUNCH_TOKEN", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE"))


def ncu_traffic(cfgs: list[str], local: int, world: int = 1, timeout: int = 600) -> dict:
    """DRAM bytes per launch of every timed kernel, measured in THIS run: an
    ncu subprocess (dram__bytes_read/write.sum; no timing is taken from it)
    over tools/profile_kernels.py, which builds the same resident operands as
    rank 0 of this run (same shard size) and issues each config's kernels
    once, in job order.  Returns
    {cfg: [{"kernel", "bytes", "ncu_us"} per job]} or {"error": ...}."""
    if _under_profiler():
        return {"error": "bench itself runs under a profiler"}
    exe = "ncu"
    try:
        subprocess.run([exe, "--version"], capture_output=True, check=True, timeout=60)
    except (OSError, subprocess.SubprocessError):
        return {"error": "ncu not available"}
    out = {}
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    env.pop("LOCAL_RANK", None)
    if "CUDA_VISIBLE_DEVICES" not in env:
        env["CUDA_VISIBLE_DEVICES"] = str(local)
    mode = ["--rounding", "rn" if MODE[0] else "rz", "--subnormals", "ftz" if MODE[1] else "gradual"]
    for cfg in cfgs:
        kre = {"C3": "k_arith|k_pack_f32|k_unpack_f32", "X3": "bfp_chain_k"}.get(cfg, "k_arith")
        logf = Path(os.environ.get("TMPDIR", "/tmp")) / f"bench_ncu_{os.getpid()}_{cfg}.csv"
        cmd = [exe, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                                 "sm__inst_executed_pipe_alu.sum",
               "--clock-control", "none", "-k", f"regex:{kre}", "--csv", "--print-units", "base",
               "--log-file", str(logf),
               sys.executable, str(ROOT / "tools" / "profile_kernels.py"), "--config", cfg,
               "--iters", "1", "--marker", "--rank", "0", "--world", str(world)] + mode
        # the same command line first WITHOUT ncu: ncu only ever sees a
        # program that just exited 0 with no CUDA fault (B200_PROFILING.md)
        plain = cmd[cmd.index(sys.executable):]
        try:
            p0 = subprocess.run(plain, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
        except subprocess.TimeoutExpired:
            out[cfg] = {"error": "plain run of the profiled command timed out"}
            continue
        if p0.returncode != 0 or re.search(r"CUDA error|illegal memory access|illegal address|Xid|segmentation fault",
                                           p0.stdout + p0.stderr, re.I):
            out[cfg] = {"error": f"plain run failed (rc={p0.returncode}); ncu not run"}
            continue
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
            txt = logf.read_text() if logf.exists() else ""
        except subprocess.TimeoutExpired:
            out[cfg] = {"error": "ncu timed out"}
            continue
        finally:
            logf.unlink(missing_ok=True)
        rows, order = {}, []
        for rec in csv.reader(io.StringIO(txt)):
            if len(rec) < 15 or rec[0] == "ID":
                continue
            kid, kname, metric, value = rec[0], rec[4], rec[12], rec[14]
            if kid not in rows:
                rows[kid] = {"kernel": kname}
                order.append(kid)
            try:
                rows[kid][metric] = float(value.replace(",", ""))
            except ValueError:
                pass
        # profile_kernels prints "TIMED k" before the timed launches; operand
        # setup comes first, so the timed ones are the LAST k profiled kernels
        m = re.search(r"TIMED (\d+)", r.stdout)
        if not m or r.returncode != 0:
            out[cfg] = {"error": f"ncu rc={r.returncode}: {(r.stderr or r.stdout)[-300:]}"}
            continue
        k = int(m.group(1))
        if len(order) < k:
            out[cfg] = {"error": f"ncu saw {len(order)} kernels, expected >= {k}"}
            continue
        out[cfg] = [{"kernel": rows[i]["kernel"][:160],
                     "bytes": int(rows[i].get("dram__bytes_read.sum", 0) + rows[i].get("dram__bytes_write.sum", 0)),
                     "alu_warp_inst": rows[i].get("sm__inst_executed_pipe_alu.sum"),
                     "ncu_us": round(rows[i].get("gpu__time_duration.sum", 0) / 1e3, 2)} for i in order[-k:]]
    return out


# --------------------------------------------------------- reference (CPU)
def ref_cpu_jobs(cfg: str, sample: int, threads: int):
    """The reference's CPU path for `cfg` on `sample` elements: a list of
    (label, callable) over operands prepared outside the timing.  Arithmetic
    runs the unmodified templates (oracle/_ref) on lane<1024> plane images;
    C3's pack / unpack time encode_scalar + the shipped pack and the shipped
    unpack + decode_scalar (the reference's own conversion path; its
    transpose output is wrong -- SURVEY.md §0.4 -- but its cost is what a
    reference user pays).  Labels equal the GPU jobs' labels."""
    import numpy as np
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O
    from paper_1602_04716_b200 import workloads as W

    R = O.ref()
    jobs = []

    def arith(label, op, fmt, encs):
        nb = 1 + fmt[0] + fmt[1]
        planes = [O.pack_planes(v, nb) for v in encs]
        c = planes[2] if len(planes) > 2 else None
        jobs.append((label, lambda: O.ref_binop_planes(op, fmt, planes[0], planes[1], c,
                                                        threads=threads)))

    if cfg == "C1":
        fmt = (4, 3) + MODE
        encs = [O.encode_f32(fmt, W.c1_floats(0, sample, sd, "cpu").numpy()) for sd in (1, 2)]
        arith("add", "add", fmt, encs)
    elif cfg == "C2":
        fmt = (4, 3) + MODE
        encs = [W.c2_encodings(0, sample, sd, "cpu").numpy().astype(np.uint64) for sd in (1, 2)]
        arith("mul", "mul", fmt, encs)
        arith("sub", "sub", fmt, encs)
    elif cfg == "C3":
        fmt = (5, 10) + MODE
        xs = [W.c3_floats(0, sample, sd, "cpu").numpy() for sd in (1, 2)]
        encs = [O.encode_f32(fmt, x) for x in xs]
        planes_out = np.zeros(O.nblocks(sample) * 16 * 32, dtype=np.uint32)
        fl_out = np.zeros(sample, dtype=np.float32)
        pa = O.pack_planes(encs[0], 16)
        x0 = np.ascontiguousarray(xs[0])
        jobs.append(("pack_f32", lambda: R.ref_pack_f32_path(
            x0.ctypes.data_as(O._f32p), sample, planes_out.ctypes.data_as(O._u32p), 5, 10, MODE[0], MODE[1],
            threads)))
        arith("add", "add", fmt, encs)
        arith("mul", "mul", fmt, encs)
        jobs.append(("unpack_f32", lambda: R.ref_unpack_f32_path(
            pa.ctypes.data_as(O._u32p), sample, fl_out.ctypes.data_as(O._f32p), 5, 10, threads)))
    elif cfg in ("C4", "X1"):
        for (e, s) in (C4_FMTS if cfg == "C4" else X1_FMTS):
            fmt = (e, s) + MODE
            encs = [W.c4_encodings(e, s, 0, sample, sd, "cpu").numpy().astype(np.uint64)
                    for sd in (1, 2)]
            for op in (("add", "mul") if cfg == "C4" else ("div",)):
                arith(f"{op}_1/{e}/{s}", op, fmt, encs)
    elif cfg == "C5":
        fmt = (6, 9) + MODE
        encs = [O.encode_f32(fmt, W.c5_floats(0, sample, sd, "cpu").numpy()) for sd in (1, 2, 3)]
        arith("mul_add", "mul_add", fmt, encs)
    elif cfg in ("X3", "X3u"):
        fmt = (5, 10) + MODE
        planes = [O.pack_planes(W.c4_encodings(5, 10, 0, sample, sd, "cpu").numpy().astype(np.uint64), 16)
                  for sd in (1, 2, 3, 4)]

        def expr():
            p = O.ref_binop_planes("mul", fmt, planes[0], planes[1], threads=threads)
            q = O.ref_binop_planes("mul", fmt, planes[2], planes[3], threads=threads)
            O.ref_binop_planes("add", fmt, p, q, threads=threads)
        if cfg == "X3":
            jobs.append(("a*b+c*d", expr))
        else:  # three op results per expression, as the X3u line counts them
            jobs += [("mul a*b", lambda: O.ref_binop_planes("mul", fmt, planes[0], planes[1], threads=threads)),
                     ("mul c*d", lambda: O.ref_binop_planes("mul", fmt, planes[2], planes[3], threads=threads)),
                     ("add", lambda: O.ref_binop_planes("add", fmt, planes[0], planes[1], threads=threads))]
    elif cfg == "X2":
        # the reference user's float32 path: encode_scalar + pack of both
        # operands, the op, unpack + decode_scalar of the result
        fmt = (5, 10) + MODE
        xs = [np.ascontiguousarray(W.c3_floats(0, sample, sd, "cpu").numpy()) for sd in (1, 2)]
        pl = [np.zeros(O.nblocks(sample) * 16 * 32, dtype=np.uint32) for _ in range(2)]
        fl_out = np.zeros(sample, dtype=np.float32)
        encs = [O.encode_f32(fmt, x) for x in xs]
        planes = [O.pack_planes(v, 16) for v in encs]
        for op in ("add", "mul"):
            def chain(op=op):
                for x, p in zip(xs, pl):
                    R.ref_pack_f32_path(x.ctypes.data_as(O._f32p), sample, p.ctypes.data_as(O._u32p),
                                        5, 10, MODE[0], MODE[1], threads)
                z = O.ref_binop_planes(op, fmt, planes[0], planes[1], None, threads=threads)
                R.ref_unpack_f32_path(np.ascontiguousarray(z).ctypes.data_as(O._u32p), sample,
                                      fl_out.ctypes.data_as(O._f32p), 5, 10, threads)
            jobs.append((f"{op}_f32", chain))
    else:
        raise ValueError(cfg)
    return jobs, O.ref_lib_path().name


# CPU sample per config (elements per op per timed step).  C5 follows
# a 2^26 slice of the 2^32 workload gives the rate; C2 runs
# the GPU's full N; C4 a quarter of it (2^26 per format: 48-192 MiB per
# operand, past the host's last-level cache, so the rate is the streaming
# one); the others a bounded slice so one step stays near a second on ~16
# host threads.
REF_SAMPLE = {"C1": 1 << 24, "C2": 1 << 26, "C3": 1 << 24, "C4": 1 << 26, "C5": 1 << 26,
              "X1": 1 << 22, "X2": 1 << 22, "X3": 1 << 22, "X3u": 1 << 22}


def ref_cpu_run(cfg: str, sample: int, seconds: float = 10.0, min_reps: int = 1,
                warmup: int = 1, threads: int | None = None, jobs=None) -> dict:
    """Time the reference's CPU path: whole steps (every job once), `warmup`
    untimed, then repeated for at least `seconds` and `min_reps` steps; the
    rate comes from the best step, the median alongside.  Both arms call this
    same function with the same sample, so their CPU figures agree."""
    threads = threads or os.cpu_count() or 1
    if jobs is None:
        jobs = ref_cpu_jobs(cfg, sample, threads)
    jobs, libname = jobs
    for _ in range(warmup):
        for _, fn in jobs:
            fn()
    times, per_job = [], {lbl: [] for lbl, _ in jobs}
    t_start = time.perf_counter()
    while True:
        t = time.perf_counter()
        for lbl, fn in jobs:
            tj = time.perf_counter()
            fn()
            per_job[lbl].append(time.perf_counter() - tj)
        times.append(time.perf_counter() - t)
        if len(times) >= min_reps and time.perf_counter() - t_start >= seconds:
            break
    best, med = min(times), statistics.median(times)
    return {"value": len(jobs) * sample / best / 1e9, "value_median": len(jobs) * sample / med / 1e9,
            "cores": threads, "reps": len(times), "best_s": best, "median_s": med, "lib": libname,
            "seconds": round(time.perf_counter() - t_start, 2),
            "ops": [lbl for lbl, _ in jobs], "sample": sample,
            "per_op_gelems": {lbl: round(sample / min(v) / 1e9, 5) for lbl, v in per_job.items()},
            "per_op_gelems_median": {lbl: round(sample / statistics.median(v) / 1e9, 5)
                                     for lbl, v in per_job.items()}}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_block(cfg: str, seconds: float, min_reps: int = 1, warmup: int = 1) -> dict:
    """cpu_baseline of `cfg`: all host threads for >= `seconds` (best and
    median), plus a 1-thread run of the same sample for the scaling check."""
    sample = REF_SAMPLE[cfg]
    cb = ref_cpu_run(cfg, sample, seconds=seconds, min_reps=min_reps, warmup=warmup)
    c1 = ref_cpu_run(cfg, sample, seconds=0.0, min_reps=2, warmup=0, threads=1)
    return {"value": round(cb["value"], 4), "unit": UNIT, "cores": cb["cores"], "kind": "reference",
            "value_median": round(cb["value_median"], 4),
            "sample": f"{sample} elements x {cb['ops']} per step, {cb['reps']} steps over "
                      f"{cb['seconds']} s (value = best step, value_median = median step), "
                      f"lane<1024>, {cb['cores']} threads, {cpu_model()}, {cb['lib']}",
            "per_op": cb["per_op_gelems"], "per_op_median": cb["per_op_gelems_median"],
            "nproc": os.cpu_count(), "value_1_thread": round(c1["value"], 4),
            "thread_scaling": round(cb["value"] / c1["value"], 2)}


CONFIG_TEXT = {
    "C1": ("C1: fp8 1/4/3 elementwise add, N=2^24 per GPU; float32 U[-16,16] -> encode_scalar "
           "-> planes", "1/4/3", 1 << 24),
    "C2": ("C2: fp8 1/4/3 elementwise mul + sub, N=2^26 per GPU; raw encodings (random sign, all "
           "16 exponent codes incl. subnormal/Inf/NaN, 1% zeros)", "1/4/3", 1 << 26),
    "C3": ("C3: 1/5/10 float32->bitslice pack, add, mul, bitslice->float32 unpack, N=2^28 per GPU, "
           "each timed separately; float32 normal(0,100) clamped to +-65504", "1/5/10", 1 << 28),
    "C4": ("C4: add + mul sweep over 1/3/2, 1/5/3, 1/5/7, 1/8/7, 1/8/15, N=2^28 per GPU per "
           "format; uniform finite bit patterns", "sweep", 1 << 28),
    "C5": ("C5: 1/6/9 z=round(round(a*b)+c) fused (one mul_add kernel), N=2^32 total split evenly "
           "over the GPUs; float32 sign x 2^U[-10,9] x U[1,2) -> encode_scalar", "1/6/9", None),
    "X1": ("X1 (secondary, not a BASELINE config): div sweep over 1/3/2, 1/4/3, 1/5/3, 1/5/7, 1/5/10, "
           "1/8/7, 1/8/15, N=2^28 per GPU per format; C4 operand distribution", "sweep", 1 << 28),
    "X2": ("X2 (secondary, not a BASELINE config): 1/5/10 add and mul with float32 in / float32 out "
           "in one kernel each (pack -> op -> unpack in registers), N=2^28 per GPU; C3 operands",
           "1/5/10", 1 << 28),
    "X3": ("X3 (secondary, not a BASELINE config): z = a*b + c*d in 1/5/10 as ONE bfp_chain kernel "
           "(intermediates in registers), N=2^28 per GPU; uniform finite operands", "1/5/10", 1 << 28),
    "X3u": ("X3u (secondary, not a BASELINE config): z = a*b + c*d in 1/5/10 as three kernels "
            "(mul, mul, add through HBM), N=2^28 per GPU; uniform finite operands", "1/5/10", 1 << 28),
}

OPS_OF = {
    "C1": ["add"], "C2": ["mul", "sub"], "C3": ["pack_f32", "add", "mul", "unpack_f32"],
    "C4": [f"{op}_1/{e}/{s}" for (e, s) in C4_FMTS for op in ("add", "mul")],
    "C5": ["mul_add"], "X1": [f"div_1/{e}/{s}" for (e, s) in X1_FMTS],
    "X2": ["add_f32", "mul_f32"], "X3": ["a*b+c*d"], "X3u": ["mul a*b", "mul c*d", "add"],
}


def label_fmt_op(cfg: str, lbl: str) -> tuple[str, str]:
    """("1/8/15", "mul") of a job label such as "mul_1/8/15" or C5's "mul_add"."""
    if "_1/" in lbl:
        op, fmt = lbl.split("_1/")
        return "1/" + fmt, op
    return CONFIG_TEXT[cfg][1], lbl


def scaling_of(cfg: str) -> str:
    """C5 splits a fixed 2^32 elements over the GPUs (strong); every other
    config fixes the per-GPU N (weak)."""
    return "strong" if cfg == "C5" else "weak"


def config_block(cfg: str, world: int, sweep: list[str] | None = None) -> dict:
    """Identical for both arms (same workload, ops and sizes)."""
    text, fmt, n = CONFIG_TEXT[cfg]
    d = {"workload": text, "format": fmt, "rounding": "rn" if MODE[0] else "rz",
         "subnormals": "ftz" if MODE[1] else "gradual",
         "parallelism": f"dp{world} (independent block-aligned shards, no collective)",
         "ops_per_step": OPS_OF[cfg],
         "l2": "inputs larger than L2 (no flush): no operand set is re-read before >= 2x L2 (252 MiB) "
               "of other reads and writes -- sets rotate launch by launch where one set is smaller "
               "(measured distance: roofline.step.l2_reuse_distance_bytes); outputs rotate over two "
               "buffers"}
    if n:
        d["n_per_gpu"] = n
    else:
        d["n_total"] = 1 << 32
        d["n_per_gpu"] = (1 << 32) // world
    if sweep:
        d["per_format_configs"] = sweep
    return d


# ------------------------------------------------------------------- arms
def op_entry(j, ms: float, n_total: int, peaks: dict, peak_lop3: dict | None, clocks: dict,
             path: str = "fast") -> dict:
    """One kernel on both roofline legs (per GPU) and which one binds."""
    dur = ms * 1e-3
    ach = j.algo_bytes / dur / 1e9
    ent = {"ms": round(ms, 4), "gelem_s": round(n_total / dur / 1e9, 2),
           "gelem_s_per_gpu": round(j.n / dur / 1e9, 2),
           "hbm_gbs": round(ach, 1), "hbm_frac": round(ach / peaks["hbm_gbs"], 4),
           "algorithmic_bytes": int(j.algo_bytes), "bound": "hbm",
           "frac": round(ach / peaks["hbm_gbs"], 4)}
    e, s = j.spec.exp_bits, j.spec.sig_bits
    chain_ops = ([{"+": "add", "-": "sub", "*": "mul", "/": "div"}[ch]
                  for ch in j.op.split(":", 1)[1] if ch in "+-*/"]
                 if j.op.startswith("chain:") else None)
    if j.op in OPNAMES or chain_ops:
        rn, ftz = int(j.spec.rounding), int(j.spec.subnormals)
        if chain_ops:
            parts = [sass_lop3((e, s), rn, ftz, OPNAMES[o]) for o in chain_ops]
            lop3 = None if None in parts else sum(parts)
        else:
            lop3 = sass_lop3((e, s), rn, ftz, OPNAMES[j.op], path)
        if lop3 is not None and peak_lop3:
            pe = lop3 / 32.0
            hbm_t = j.algo_bytes / (peaks["hbm_gbs"] * 1e9)
            logic_t = pe * j.n / peak_lop3["burst"]
            lf = logic_t / dur
            ent.update({"lop3_per_elem": round(pe, 3),
                        "tlop3_s": round(pe * j.n / dur / 1e12, 3),
                        "logic_frac": round(lf, 4)})
            mhz, pmhz = clocks.get("sm_mhz"), peak_lop3.get("sustained_sm_mhz")
            if mhz and pmhz:  # against the LOP3 rate of the clock the step ran at
                ent["logic_frac_at_load_clock"] = round(pe * j.n / (peak_lop3["sustained"] * mhz / pmhz) / dur, 4)
            if logic_t > hbm_t:
                ent["bound"], ent["frac"] = "logic", round(lf, 4)
    return ent


def roofline_block(jd, ent: dict, peaks: dict, peak_lop3: dict | None, traffic) -> dict:
    """The dominant kernel on its binding leg: bound / achieved / peak / unit /
    frac recomputable from the line (logic: LOP3 per element x elements per
    launch / launch time vs the probe's measured LOP3 rate)."""
    dur = ent["ms"] * 1e-3
    hbm = {"achieved": ent["hbm_gbs"], "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": ent["hbm_frac"],
           "peak_source": peaks["source"], "algorithmic_bytes_per_launch": ent["algorithmic_bytes"]}
    r = {"kernel": f"{jd.label} ({jd.fmt} {mode_text()})", "launch_ms": ent["ms"],
         "elements_per_launch": jd.n}
    logic = None
    per_elem = ent.get("lop3_per_elem", ent.get("alu_inst_per_elem_measured"))
    if per_elem is not None and "logic_frac" in ent and peak_lop3:
        src = ("SASS LOP3 count of the shipped kernel (cuobjdump of the loaded libbfpgpu.so) / 32 "
               "elements per unit" if "lop3_per_elem" in ent else
               "executed ALU-pipe instructions per element (ncu sm__inst_executed_pipe_alu in this run)")
        logic = {"achieved": round(per_elem * jd.n / dur / 1e12, 4),
                 "peak": round(peak_lop3["burst"] / 1e12, 4), "unit": "TLOP3/s", "frac": ent["logic_frac"],
                 "lop3_per_elem": per_elem,
                 "lop3_source": src,
                 "peak_source": "bfp_probe_lop3 measured in this run (burst; 148 SM x 64/clk x f_SM)",
                 "peak_sustained": round(peak_lop3["sustained"] / 1e12, 4),
                 "peak_sustained_sm_mhz": peak_lop3["sustained_sm_mhz"]}
        if "logic_frac_at_load_clock" in ent:
            logic["frac_at_load_clock"] = ent["logic_frac_at_load_clock"]
    lead = logic if ent["bound"] == "logic" and logic else hbm
    r.update({"bound": ent["bound"], "achieved": lead["achieved"], "peak": lead["peak"],
              "unit": lead["unit"], "frac": lead["frac"]})
    r["traffic"] = traffic.get("bytes") if isinstance(traffic, dict) else None
    if isinstance(traffic, dict):
        r["traffic_over_algorithmic"] = round(traffic["bytes"] / ent["algorithmic_bytes"], 4) \
            if traffic.get("bytes") else None
        r["traffic_source"] = traffic.get("source")
    r["legs"] = {"hbm": hbm}
    if logic:
        r["legs"]["logic"] = logic
    return r


def measure_config(cfg: str, args, D: Dist, probes: dict) -> dict:
    """Device timing (+ e2e, + probes once) of one config on this rank."""
    import torch
    log(f"device timing {cfg}")
    res = run_device(cfg, args.steps, args.warmup, D)
    if clocks_rejected(res["clocks"]):  # re-measure once
        log("clocks rejected; re-measuring")
        res = run_device(cfg, args.steps, args.warmup, D, jobs=res["jobs"])
    jobs = res["jobs"]
    log(f"device done: {res['ms_total'] / args.steps:.4f} ms/step (max over ranks)")
    res["n_total"] = [int(v) for v in D.reduce([float(j.n) for j in jobs], op="sum")]
    res["l2_reuse"] = l2_reuse_distance(jobs)
    e2e = None
    if not args.no_e2e and (cfg == args.configs[0] or args.e2e_all):
        log("e2e (host buffers through the C ABI)")
        e2e = run_e2e(jobs, args.steps, D)
    if "lop3" not in probes:
        log("lop3 / hbm probes")
        probes["lop3"] = lop3_peak(D.dev)
        probes["hbm_2r1w"] = hbm_2r1w_probe(D.dev)
    if e2e is not None and "pcie" not in probes:
        probes["pcie"] = pcie_probe(D.dev)
    res["e2e"] = e2e
    res["jobs"] = None
    res["job_meta"] = [JobMeta(j) for j in jobs]  # the operands are released here
    del jobs
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return res


def build_line(cfg: str, res: dict, args, D: Dist, probes: dict, traffic: dict) -> dict:
    peaks = measured_peaks()
    jobs = res["job_meta"]
    ms_step = res["ms_total"] / args.steps
    value = sum(res["n_total"]) / (ms_step * 1e-3) / 1e9
    per_op, per_format = {}, {}
    tr = traffic.get(cfg)
    for k, (j, ms, nt) in enumerate(zip(jobs, res["kern_ms"], res["n_total"])):
        ent = op_entry(j, ms, nt, peaks, probes.get("lop3"), res["clocks"])
        if isinstance(tr, list) and k < len(tr):
            ent["traffic"] = tr[k]["bytes"]
            ent["traffic_over_algorithmic"] = round(tr[k]["bytes"] / j.algo_bytes, 4)
            if tr[k].get("alu_warp_inst"):
                # executed ALU-pipe instructions per element (one warp instruction
                # = 32 threads x one 32-element unit each), measured by ncu in this run
                ape = tr[k]["alu_warp_inst"] * 32 / j.n
                ent["alu_inst_per_elem_measured"] = round(ape, 3)
                lop3 = probes.get("lop3")
                if "lop3_per_elem" not in ent and lop3:
                    # kernels without a static LOP3 count (fused float32 codec, chains):
                    # the logic leg from the executed ALU-pipe instructions
                    lf = ape * j.n / lop3["burst"] / (ms * 1e-3)
                    ent.update({"logic_frac": round(lf, 4), "logic_leg": "executed ALU-pipe instructions (ncu)",
                                "tlop3_s": round(ape * j.n / (ms * 1e-3) / 1e12, 3)})
                    if lf > ent["hbm_frac"]:
                        ent["bound"], ent["frac"] = "logic", round(lf, 4)
        per_op[j.label] = ent
        per_format.setdefault(j.fmt, {})[j.op] = {
            key: ent[key] for key in ("gelem_s", "bound", "frac", "ms", "hbm_frac", "logic_frac",
                                      "logic_frac_at_load_clock", "lop3_per_elem", "alu_inst_per_elem_measured",
                                      "traffic_over_algorithmic")
            if key in ent}
        per_format[j.fmt][j.op]["config"] = cfg
        per_format[j.fmt][j.op].update(j.info)
        for name, ams in res.get("aux_ms", {}).items():
            if name.split(":")[0] != j.label:
                continue
            # the same kernel forced onto its general cover (BFP_GENERAL_NETWORK), same operands
            aent = op_entry(j, ams, nt, peaks, probes.get("lop3"), res["clocks"], path="general")
            per_format[j.fmt][f"{j.op} ({name.split(':')[1]})"] = dict(
                # (no load-clock fraction: the clocks were sampled during the step, not this launch)
                {key: aent[key] for key in ("gelem_s", "bound", "frac", "ms", "hbm_frac", "logic_frac",
                                            "lop3_per_elem") if key in aent},
                config=cfg, note="same launch with BFP_GENERAL_NETWORK: every warp runs the general cover "
                                 "(the one taken when a block holds a zero, subnormal, Inf, NaN, huge or tiny operand); not part "
                                 "of the step")
            per_format[j.fmt][j.op]["cover"] = (
                "fast_cover_blocks_frac of this launch's 1024-element blocks pass the kernel's per-block test "
                "(bfp_mul_add_fast_blocks: finite normals with 1 <= ea, eb < 48, 32 <= ea + eb <= 91, "
                "16 <= ec < 48 for 1/6/9; C5's exponent fields are 21..41) and run the fast-domain cover, "
                "the rest the general one")
    k_dom = max(range(len(jobs)), key=lambda k: res["kern_ms"][k])
    jd = jobs[k_dom]
    t_dom = None
    if isinstance(tr, list) and k_dom < len(tr):
        t_dom = {"bytes": tr[k_dom]["bytes"], "source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum "
                 f"of this kernel, measured by an ncu subprocess in this run ({tr[k_dom]['kernel'][:60]}...)"}
    elif isinstance(tr, dict):
        t_dom = {"bytes": None, "source": f"not measured: {tr.get('error')}"}
    roof = roofline_block(jd, per_op[jd.label], peaks, probes.get("lop3"), t_dom)
    roof["hbm_2r1w_probe_gbs"] = probes.get("hbm_2r1w")
    roof["per_op"] = per_op
    step_bytes = sum(j.algo_bytes for j in jobs)
    step_gbs = step_bytes / (ms_step * 1e-3) / 1e9
    # self-check: inputs never stay in L2 between uses, so no step or kernel
    # can beat the HBM copy peak by much; a faster figure means broken timing
    for j, ms in zip(jobs, res["kern_ms"]):
        if j.algo_bytes / (ms * 1e-3) / 1e9 > 1.15 * peaks["hbm_gbs"]:
            raise RuntimeError(f"{cfg}:{j.label}: {ms} ms per launch is faster than HBM allows")
    if step_gbs > 1.15 * peaks["hbm_gbs"]:
        raise RuntimeError(f"{cfg}: step time {ms_step} ms is faster than HBM allows")
    roof["step"] = {"algorithmic_bytes_per_gpu": int(step_bytes), "ms": round(ms_step, 5),
                    "achieved_gbs_per_gpu": round(step_gbs, 1),
                    "hbm_frac": round(step_gbs / peaks["hbm_gbs"], 4),
                    "note": "whole step: K steps captured once into a CUDA graph through the C ABI and "
                            "replayed (consecutive kernels overlap through programmatic dependent "
                            "launch); per-kernel figures come from one graph per kernel holding its K "
                            "launches; all times max over ranks",
                    "ms_per_step_eager": round(res["ms_total_eager"] / args.steps, 5)}
    pw = res["clocks"].get("power_w")
    if pw:  # board energy per result element at the sampled draw (logic kernels run power-capped)
        roof["step"]["pj_per_elem"] = round(pw * ms_step * 1e-3 / (sum(res["n_total"]) / D.world) * 1e12, 1)
    cfgb = config_block(cfg, D.world)
    reuse = res["l2_reuse"]
    roof["step"]["l2_reuse_distance_bytes"] = reuse
    if 0 <= reuse < 2 * L2_BYTES:
        raise RuntimeError(f"{cfg}: L2 reuse distance {reuse} B < 2x L2")
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": D.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
        "higher_is_better": True, "scaling": scaling_of(cfg), "vs_baseline": None,
        "dtype": "u32 (bitslice words)",
        "data": "synthetic (seeded SplitMix64 operands; BASELINE.json configs)",
        "config": cfgb, "roofline": roof, "per_format": per_format,
        "clocks": res["clocks"], "gpu_launches": res["launches"],
    }
    e2e = res.get("e2e")
    if e2e is not None:
        pcie = probes["pcie"]
        bound_s = max(e2e["h2d"] / (pcie["h2d_gbs"] * 1e9), e2e["d2h"] / (pcie["d2h_gbs"] * 1e9),
                      (e2e["h2d"] + e2e["d2h"]) / (pcie["bidir_gbs"] * 1e9))
        line["e2e"] = {"value": round(e2e["elems"] * D.world / e2e["s_per_step"] / 1e9, 3),
                       "unit": UNIT, "h2d_bytes_per_step": int(e2e["h2d"]),
                       "d2h_bytes_per_step": int(e2e["d2h"]),
                       "pcie_measured": pcie, "frac_of_pcie_bound": round(bound_s / e2e["s_per_step"], 4),
                       "path": "C ABI host entry points (bfp_arith_host_batch / bfp_pack_f32_host / "
                               "bfp_unpack_f32_host) on pinned host buffers: inputs copied H2D in chunk "
                               "order on one stream, kernels on a second, results copied back (or "
                               "written in place over PCIe for small calls); per-GPU bytes",
                       "steps": e2e["steps"]}
    return line


def main_ours(args) -> None:
    import torch
    D = Dist("nccl")
    torch.cuda.set_device(D.dev)
    info = {"rank": D.rank, "local_rank": D.local, "host": socket.gethostname(),
            "device": torch.cuda.get_device_name(D.dev),
            "pci_bus_id": getattr(torch.cuda.get_device_properties(D.dev), "pci_bus_id", None)}
    probes: dict = {}
    results = []
    for cfg in args.configs:
        res = measure_config(cfg, args, D, probes)
        lo, hi = config_n(cfg, D.rank, D.world)
        res["rank_info"] = D.gather(dict(info, shard=[lo, hi], ms_per_step=round(
            res["ms_total_rank"] / args.steps, 5)))
        results.append((cfg, res))
        torch.cuda.empty_cache()
    traffic = {}
    if not args.no_ncu:
        if D.rank == 0:
            log("DRAM traffic: ncu subprocess over tools/profile_kernels.py")
            traffic = ncu_traffic(list(args.configs), D.local, D.world)
        D.barrier()
    lines = [build_line(cfg, res, args, D, probes, traffic) for cfg, res in results]
    for line, (cfg, res) in zip(lines, results):
        line["ranks"] = res["rank_info"]
    if D.rank == 0 and D.world == 1 and not args.no_cpu_baseline:
        for line, (cfg, _) in zip(lines, results):
            if cfg in REF_SAMPLE:
                log(f"cpu baseline {cfg}")
                cb = line["cpu_baseline"] = cpu_block(cfg, args.cpu_seconds)
                for lbl, v in cb["per_op"].items():
                    fmt, op = label_fmt_op(cfg, lbl)
                    if op in line["per_format"].get(fmt, {}):
                        line["per_format"][fmt][op]["cpu_gelem_s"] = v
    if args.headline:  # one line: the first config, the others folded into per_format
        head = lines[0]
        for line, (cfg, _) in zip(lines[1:], results[1:]):
            for fmt, ops in line["per_format"].items():
                head["per_format"].setdefault(fmt, {}).update(ops)
            head.setdefault("secondary", {})[cfg] = {
                "value": line["value"], "ms_per_step": line["ms_per_step"], "clocks": line["clocks"],
                "roofline": {k: line["roofline"][k] for k in ("kernel", "bound", "achieved", "peak", "unit",
                                                             "frac", "traffic")},
                "config": line["config"]}
        head["config"]["per_format_configs"] = [cfg for cfg, _ in results]
        lines = [head]
    if D.rank == 0:
        for line in lines:
            print(json.dumps(line), flush=True)
    D.close()


def main_reference(args) -> None:
    """The reference's own CPU implementation (oracle/_ref) on this host's
    cores, same config / metric / unit; rank 0 only (other ranks exit 0)."""
    world, rank, _ = env_dist()
    if rank != 0:
        return
    lines = []
    for cfg in args.configs:
        sample = REF_SAMPLE[cfg]
        log(f"reference {cfg}: {sample} elements per op per step")
        cb = cpu_block(cfg, args.cpu_seconds, min_reps=args.steps, warmup=args.warmup)
        value = cb["value"]
        per_format = {}
        for lbl, v in cb["per_op"].items():
            fmt, op = label_fmt_op(cfg, lbl)
            per_format.setdefault(fmt, {})[op] = {"gelem_s": v, "gelem_s_median": cb["per_op_median"][lbl],
                                                  "config": cfg}
        lines.append({
            "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(len(cb["per_op"]) * sample / (value * 1e9) * 1e3, 3),
            "higher_is_better": True, "scaling": scaling_of(cfg), "vs_baseline": None,
            "dtype": "u64 lanes (lane<1024> bitslice)",
            "data": "synthetic (seeded SplitMix64 operands; BASELINE.json configs)",
            "config": config_block(cfg, world), "per_format": per_format,
            "cpu_baseline": cb,
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        })
    if args.headline:
        head = lines[0]
        for line in lines[1:]:
            for fmt, ops in line["per_format"].items():
                head["per_format"].setdefault(fmt, {}).update(ops)
        head["config"]["per_format_configs"] = list(args.configs)
        lines = [head]
    for line in lines:
        print(json.dumps(line), flush=True)


def main_dry_run(args) -> None:
    """gloo on the CPU: the launcher, shard ranges, barrier + max-over-ranks
    reduction and rank-0-only output of the real path, with a stand-in step
    (a SplitMix64 pass over a slice of the rank's shard plus a rank-dependent
    delay, so the maximum is the slowest rank)."""
    import torch
    from paper_1602_04716_b200 import workloads as W
    D = Dist("gloo")
    cfg = args.configs[0]
    lo, hi = config_n(cfg, D.rank, D.world)
    ts = []
    for i in range(args.warmup + args.steps):
        D.barrier()
        t = time.perf_counter()
        W.splitmix64(torch.arange(lo, min(hi, lo + (1 << 16)), dtype=torch.int64), W.SEED_A).sum()
        time.sleep(0.002 * (D.rank + 1))
        D.barrier()
        if i >= args.warmup:
            ts.append((time.perf_counter() - t) * 1e3)
    ms_rank = sum(ts)
    ms_max = D.reduce([ms_rank])[0]
    n_total = int(D.reduce([float(hi - lo)], op="sum")[0])
    ranks = D.gather({"rank": D.rank, "local_rank": D.local, "shard": [lo, hi], "ms_total": ms_rank,
                      "host": socket.gethostname()})
    if D.rank == 0:
        print(json.dumps({"dry_run": True, "metric": METRIC, "n_gpus": D.world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "ms_total_max": ms_max,
                          "n_total": n_total, "scaling": scaling_of(cfg), "config": config_block(cfg, D.world),
                          "ranks": ranks}), flush=True)
    D.close()


def main() -> None:
    faulthandler.enable()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="default",
                    help="default (C5 headline + C4 per-format sweep in one line), C1..C5, X1..X3u, "
                         "a comma list (one line each), or 'all'")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-all", action="store_true", help="e2e for every config, not just the first")
    ap.add_argument("--no-ncu", action="store_true", help="skip the in-run ncu traffic measurement")
    ap.add_argument("--dry-run", action="store_true", help="gloo on the CPU with a stand-in step")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--rounding", choices=["rn", "rz"], default="rn")
    ap.add_argument("--subnormals", choices=["gradual", "ftz"], default="gradual")
    args = ap.parse_args()
    global MODE
    MODE = (int(args.rounding == "rn"), int(args.subnormals == "ftz"))
    args.headline = args.config == "default"
    args.configs = (["C5", "C4"] if args.config == "default" else
                    ["C1", "C2", "C3", "C4", "C5"] if args.config == "all" else args.config.split(","))
    for c in args.configs:
        if c not in CONFIG_TEXT:
            ap.error(f"unknown config {c}")
    if args.warmup < 3:
        args.warmup = 3
    maybe_relaunch(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if "WORLD_SIZE" in os.environ and args.gpus not in (1, world):
        ap.error(f"--gpus {args.gpus} but the launcher started WORLD_SIZE={world} ranks")
    args.gpus = world
    if args.dry_run:
        main_dry_run(args)
    elif args.impl == "reference":
        main_reference(args)
    else:
        main_ours(args)


if __name__ == "__main__":
    main()
