#!/usr/bin/env python3
"""Benchmark of the B200 bitslice FP hot path (BASELINE.json metric:
"bitslice FP ops/sec (Gelem/s) per format vs LOP3/HBM roofline").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2|C1|C3|C4|C5|all]

Default workload: configs[1] = C2 -- 1/4/3 (fp8, RN, gradual) elementwise
multiply AND subtract over N = 2^26 elements per GPU; one step = one mul
launch + one sub launch over resident planes.  The metric counts result
elements: value = 2 * N * world / step time (Gelem/s).  Under torchrun each
rank owns its own 2^26-element shard (weak scaling, no collective on the data
path).

JSON line (rank 0): value (device, inputs resident in HBM), e2e (the same
step through the C ABI with host planes: H2D + kernels + D2H), roofline
(dominant kernel, HBM leg + measured LOP3 leg), cpu_baseline (the reference
itself -- oracle/_ref, the unmodified headers compiled in place -- on the
host cores, bounded sample), clocks (nvidia-smi during a sustained window of
the same step), gpu_launches.

--impl reference times the reference's own CPU implementation (oracle/_ref)
on this host's cores on the same config/metric; rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import faulthandler
import json
import os
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


# ---------------------------------------------------------------- utilities
def env_dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


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
        num = lambda v: float(v) if v.replace(".", "", 1).isdigit() else None
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


def sass_lop3(fmt, rn, ftz, op: int) -> int | None:
    """Static LOP3 count of the arithmetic kernel (one 32-element unit per
    loop iteration) from cuobjdump of the loaded library."""
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
                return r["LOP3"]
    except (OSError, subprocess.SubprocessError, ValueError, KeyError):  # no cuobjdump / odd SASS
        return None
    return None


# ------------------------------------------------------------ the workloads
class Job:
    """One timed kernel of a step: `launch(i)` issues it on the current
    stream (i = step index, for rotating outputs)."""

    def __init__(self, label, op, spec, n, launch, algo_bytes, host=None):
        self.label, self.op, self.spec, self.n = label, op, spec, n
        self.launch, self.algo_bytes, self.host = launch, algo_bytes, host


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


L2_BYTES = 126 * 1024 * 1024

# (rn, ftz) of every config: the reference default RN + gradual
# (format.hpp:26-27); --rounding / --subnormals select the secondary rows.
MODE = (1, 0)


def mode_text() -> str:
    return ("rn" if MODE[0] else "rz") + ("+ftz" if MODE[1] else "")


def spec_of(e: int, s: int):
    import paper_1602_04716_b200 as bfp
    return bfp.make_spec(e, s, bfp.rounding_mode(MODE[0]), bfp.subnormal_policy(MODE[1]))


def input_sets(spec, n, n_inputs: int) -> int:
    """Rotating input sets so that consecutive uses of one set are separated
    by >= 2x L2 of other traffic (inputs always come from HBM)."""
    set_bytes = n_inputs * spec.plane_bytes(n)
    return max(1, -(-2 * L2_BYTES // set_bytes))


def _arith_job(label, op, spec, n, sets, device):
    """sets: list of (a, b, c) operand tuples rotated step by step."""
    import torch
    import paper_1602_04716_b200 as bfp
    L = bfp.lib()
    outs = [bfp.empty(spec, n, device) for _ in range(2)]  # rotating outputs

    def launch(i, st):
        # resident operands that nothing in the step writes: BFP_INPUTS_READY
        # lets each kernel's first loads overlap its predecessor's tail
        a, b, c = sets[i % len(sets)]
        rc = L.bfp_arith_ex(OPNAMES[op], spec.c, a.planes.data_ptr(), b.planes.data_ptr(),
                            c.planes.data_ptr() if c is not None else None,
                            outs[i & 1].planes.data_ptr(), n, st, 1)
        if rc != 0:
            raise RuntimeError(L.bfp_last_error())

    nbits = spec.total_bits()
    a, b, c = sets[0]
    nin = 3 if c is not None else 2
    return Job(label, op, spec, n, launch, (nin + 1) * nbits / 8 * n,
               host={"kind": "arith", "op": op, "inputs": [a, b] + ([c] if c is not None else []),
                     "sets": len(sets)})


X1_FMTS = [(3, 2), (4, 3), (5, 3), (5, 7), (5, 10), (8, 7), (8, 15)]


def make_jobs(cfg: str, rank: int, world: int, device) -> list:
    """Per-rank resident operands and the timed kernels of config `cfg`."""
    import torch
    import paper_1602_04716_b200 as bfp
    from paper_1602_04716_b200 import workloads as W

    L = bfp.lib()
    if cfg == "C1":
        n = 1 << 24
        spec = spec_of(4, 3)
        lo = rank * n
        sets = []
        for r in range(input_sets(spec, n, 2)):  # same data, distinct buffers
            if r == 0:
                a = bfp.pack_f32(W.c1_floats(lo, lo + n, W.SEED_A, device), spec)
                b = bfp.pack_f32(W.c1_floats(lo, lo + n, W.SEED_B, device), spec)
            sets.append((a, b, None) if r == 0 else (a.clone(), b.clone(), None))
        return [_arith_job("add", "add", spec, n, sets, device)]
    if cfg == "C2":
        n = 1 << 26
        spec = spec_of(4, 3)
        lo = rank * n
        a = bfp.pack(W.c2_encodings(lo, lo + n, W.SEED_A, device), spec)
        b = bfp.pack(W.c2_encodings(lo, lo + n, W.SEED_B, device), spec)
        sets = [(a, b, None)] + [(a.clone(), b.clone(), None)
                                 for _ in range(input_sets(spec, n, 2) - 1)]
        return [_arith_job("mul", "mul", spec, n, sets, device),
                _arith_job("sub", "sub", spec, n, sets, device)]
    if cfg == "C3":
        n = 1 << 28
        spec = spec_of(5, 10)
        lo = rank * n
        xa = W.c3_floats(lo, lo + n, W.SEED_A, device)
        xb = W.c3_floats(lo, lo + n, W.SEED_B, device)
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
        return [Job("pack_f32", "pack_f32", spec, n, pack_launch, (4 + nb / 8) * n,
                    host={"kind": "pack_f32", "x": xa}),
                _arith_job("add", "add", spec, n, [(a, b, None)], device),
                _arith_job("mul", "mul", spec, n, [(a, b, None)], device),
                Job("unpack_f32", "unpack_f32", spec, n, unpack_launch, (nb / 8 + 4) * n,
                    host={"kind": "unpack_f32", "v": a})]
    if cfg == "C4":
        n = 1 << 28
        lo = rank * n
        jobs = []
        for (e, s) in W.CONFIGS["C4"]["fmts"]:
            spec = spec_of(e, s)
            a = bfp.pack(W.c4_encodings(e, s, lo, lo + n, W.SEED_A, device), spec)
            b = bfp.pack(W.c4_encodings(e, s, lo, lo + n, W.SEED_B, device), spec)
            torch.cuda.empty_cache()
            jobs.append(_arith_job(f"add_1/{e}/{s}", "add", spec, n, [(a, b, None)], device))
            jobs.append(_arith_job(f"mul_1/{e}/{s}", "mul", spec, n, [(a, b, None)], device))
        return jobs
    if cfg == "C5":
        total = 1 << 32
        lo, hi = W.shard(total, rank, world)
        n = hi - lo
        spec = spec_of(6, 9)
        ops = [_chunked_pack_f32(lambda a_, b_, sd=sd: W.c5_floats(lo + a_, lo + b_, sd, device), n,
                                 spec, device)
               for sd in (W.SEED_A, W.SEED_B, W.SEED_C)]
        torch.cuda.empty_cache()
        return [_arith_job("mul_add", "mul_add", spec, n, [tuple(ops)], device)]
    if cfg == "X1":  # secondary: bfp_div over the C4 formats + 1/4/3, 1/5/10
        n = 1 << 28
        lo = rank * n
        jobs = []
        for (e, s) in X1_FMTS:
            spec = spec_of(e, s)
            a = bfp.pack(W.c4_encodings(e, s, lo, lo + n, W.SEED_A, device), spec)
            b = bfp.pack(W.c4_encodings(e, s, lo, lo + n, W.SEED_B, device), spec)
            torch.cuda.empty_cache()
            jobs.append(_arith_job(f"div_1/{e}/{s}", "div", spec, n, [(a, b, None)], device))
        return jobs
    if cfg == "X2":  # secondary: fused float32-in/out ops, C3 operands
        n = 1 << 28
        spec = spec_of(5, 10)
        lo = rank * n
        xa = W.c3_floats(lo, lo + n, W.SEED_A, device)
        xb = W.c3_floats(lo, lo + n, W.SEED_B, device)
        outs = [torch.empty(n, dtype=torch.float32, device=device) for _ in range(2)]
        jobs = []
        for op in ("add", "mul"):
            def launch(i, st, op=op):
                rc = L.bfp_arith_f32(OPNAMES[op], spec.c, xa.data_ptr(), xb.data_ptr(), None,
                                     outs[i & 1].data_ptr(), n, st)
                if rc != 0:
                    raise RuntimeError(L.bfp_last_error())
            jobs.append(Job(f"{op}_f32", f"{op}_f32", spec, n, launch, 12 * n,
                            host={"kind": "none"}))
        return jobs
    if cfg in ("X3", "X3u"):  # secondary: z = a*b + c*d, fused (bfp_chain) or as 3 kernels
        n = 1 << 28
        spec = spec_of(5, 10)
        lo = rank * n
        vs = [bfp.pack(W.c4_encodings(5, 10, lo, lo + n, sd, device), spec)
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


def run_device(cfg: str, steps: int, warmup: int, world: int, rank: int, local: int,
               jobs=None) -> dict:
    import torch
    import torch.distributed as dist
    import paper_1602_04716_b200 as bfp

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    L = bfp.lib()
    if jobs is None:
        jobs = make_jobs(cfg, rank, world, device)
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

    # sustained window of the same graph for the clock record (~1.5 s)
    t_probe = time.perf_counter()
    g_all.replay()
    torch.cuda.synchronize()
    one = max(time.perf_counter() - t_probe, 1e-5)
    with ClockSampler(local) as cs:
        for _ in range(max(1, int(1.5 / one))):
            g_all.replay()
        torch.cuda.synchronize()
    clocks = cs.summary()

    def timed_replay(g) -> float:
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0.record(stream)  # replay() launches the graph on the current stream
        g.replay()
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        return t0.elapsed_time(t1)

    # Timed region (the value): K whole steps, back to back.
    ms_total = timed_replay(g_all)
    if world > 1:
        t = torch.tensor([ms_total], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
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
    # replay on the launching stream -> mean launch duration.
    kern_ms = []
    for k, j in enumerate(jobs):
        g, _ = capture(lambda s, j=j: [j.launch(i, s) for i in range(steps)])
        g.replay()
        torch.cuda.synchronize()
        kern_ms.append(timed_replay(g) / steps)
        del g
    del g_all
    return {"jobs": jobs, "ms_total": ms_total, "kern_ms": kern_ms, "clocks": clocks,
            "launches": int(launches), "ms_total_eager": ms_total_eager}


def run_e2e(cfg: str, jobs, steps: int, world: int, rank: int, local: int) -> dict:
    """The same step through the C ABI with HOST buffers (pinned): every step
    copies its inputs H2D and its results D2H inside the timed region."""
    import torch
    import torch.distributed as dist
    import paper_1602_04716_b200 as bfp

    device = torch.device("cuda", local)
    L = bfp.lib()
    ctx = L.bfp_host_ctx_create(int(os.environ.get("BFP_E2E_CHUNK", 1 << 24)))
    bufs = []

    def pinned(nbytes):
        p = L.bfp_host_alloc(nbytes)
        if not p:
            raise RuntimeError("bfp_host_alloc failed")
        bufs.append(p)
        return p

    def host_copy(t: torch.Tensor):
        nbytes = t.numel() * t.element_size()
        p = pinned(nbytes)
        src = t.cpu().numpy()  # keep alive across the copy
        C.memmove(p, src.ctypes.data, nbytes)
        del src
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
        if not calls:  # no host-buffer entry point for these kernels (X2)
            return None

        def step():
            for fn, _, _, _ in calls:
                rc = fn()
                if rc != 0:
                    raise RuntimeError(L.bfp_last_error())

        step()
        if world > 1:
            dist.barrier()
        k = max(2, min(steps // 4, 10))
        t = time.perf_counter()
        for _ in range(k):
            step()
        dt = (time.perf_counter() - t) / k
        if world > 1:
            tt = torch.tensor([dt], device=device)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        return {"s_per_step": dt, "h2d": sum(c[1] for c in calls),
                "d2h": sum(c[2] for c in calls), "elems": sum(c[3] for c in calls), "steps": k}
    finally:
        for p in bufs:
            L.bfp_host_free(p)
        L.bfp_host_ctx_destroy(ctx)


def hbm_2r1w_probe(local: int, nbytes: int = 1 << 30) -> float:
    """HBM rate of a plain 2-read : 1-write stream (torch bitwise_xor over
    1 GiB int32 operands, best of 10 by CUDA events) -- the access mix of a
    binary op.  MEASURED_PEAKS.json's copy is 1:1, which HBM serves slightly
    slower, so the binary-op kernels can exceed it; this is the context."""
    import torch
    dev = torch.device("cuda", local)
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


def pcie_probe(local: int, nbytes: int = 1 << 28) -> dict:
    """Pinned-host <-> device copy bandwidth on this box (the e2e ceiling):
    H2D alone, D2H alone, and both directions at once on two streams."""
    import torch
    dev = torch.device("cuda", local)
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


def load_clock_frac(lop3: float, dur: float, peak: dict, clocks: dict) -> float | None:
    """Logic fraction against the probe's LOP3 rate scaled to the SM clock the
    step ran at (sampled during the timed graph replays): logic-heavy kernels
    run power-capped below the probe's clock, which the burst figure ignores."""
    mhz, pmhz = clocks.get("sm_mhz"), peak.get("sustained_sm_mhz")
    if not mhz or not pmhz:
        return None
    return round(lop3 / (peak["sustained"] * mhz / pmhz) / dur, 4)


def lop3_peak(local: int = 0) -> dict | None:
    """LOP3 issue rate of the probe kernel (bfp_probe_lop3: 8 independent
    chains per thread on every SM).  burst = one launch on a cool GPU (the
    clock ceiling); sustained = back-to-back launches for ~2 s, median of the
    second half, with the SM clock it settled at (the denominator for kernels
    timed inside long steps; in practice the register-only probe is not
    power-capped and settles at the clock ceiling, so load_clock_frac scales
    it to the clock the kernels actually ran at)."""
    import paper_1602_04716_b200 as bfp
    L = bfp.lib()
    ms, rate = C.c_float(), C.c_double()
    if L.bfp_probe_lop3(4000, C.byref(ms), C.byref(rate)) != 0:
        return None
    burst = rate.value
    rates = []
    with ClockSampler(local) as cs:
        t = time.perf_counter()
        while time.perf_counter() - t < 2.0:
            if L.bfp_probe_lop3(4000, C.byref(ms), C.byref(rate)) != 0:
                return None
            rates.append(rate.value)
    sus = statistics.median(rates[len(rates) // 2:])
    return {"burst": burst, "sustained": sus, "sustained_sm_mhz": cs.summary().get("sm_mhz")}


# --------------------------------------------------------- reference (CPU)
def ref_cpu_jobs(cfg: str, sample: int, threads: int):
    """The reference's CPU path for `cfg` on `sample` elements: a list of
    (label, callable) over operands prepared outside the timing.  Arithmetic
    runs the unmodified templates (oracle/_ref) on lane<1024> plane images;
    C3's pack / unpack time encode_scalar + the shipped pack and the shipped
    unpack + decode_scalar (the reference's own conversion path; its
    transpose output is wrong -- SURVEY.md §0.4 -- but its cost is what a
    reference user pays)."""
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
    elif cfg == "C4":
        for (e, s) in W.CONFIGS["C4"]["fmts"]:
            fmt = (e, s) + MODE
            encs = [W.c4_encodings(e, s, 0, sample, sd, "cpu").numpy().astype(np.uint64)
                    for sd in (1, 2)]
            arith(f"add_1/{e}/{s}", "add", fmt, encs)
            arith(f"mul_1/{e}/{s}", "mul", fmt, encs)
    elif cfg == "C5":
        fmt = (6, 9) + MODE
        encs = [O.encode_f32(fmt, W.c5_floats(0, sample, sd, "cpu").numpy()) for sd in (1, 2, 3)]
        arith("mul_add", "mul_add", fmt, encs)
    elif cfg == "X1":
        for (e, s) in X1_FMTS:
            fmt = (e, s) + MODE
            encs = [W.c4_encodings(e, s, 0, sample, sd, "cpu").numpy().astype(np.uint64)
                    for sd in (1, 2)]
            arith(f"div_1/{e}/{s}", "div", fmt, encs)
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


REF_SAMPLE = {"C1": 1 << 22, "C2": 1 << 22, "C3": 1 << 20, "C4": 1 << 20, "C5": 1 << 20,
              "X1": 1 << 20, "X2": 1 << 20, "X3": 1 << 20, "X3u": 1 << 20}


def ref_cpu_run(cfg: str, sample: int, reps: int | None = None, seconds: float = 10.0,
                threads: int | None = None) -> dict:
    """Time the reference's CPU path: whole steps (every job once) repeated
    `reps` times or for ~`seconds`; rate from the best step."""
    threads = threads or os.cpu_count() or 1
    jobs, libname = ref_cpu_jobs(cfg, sample, threads)
    times, per_job = [], {lbl: [] for lbl, _ in jobs}
    t_start = time.perf_counter()
    while True:
        t = time.perf_counter()
        for lbl, fn in jobs:
            tj = time.perf_counter()
            fn()
            per_job[lbl].append(time.perf_counter() - tj)
        times.append(time.perf_counter() - t)
        if reps is not None and len(times) >= reps:
            break
        if reps is None and time.perf_counter() - t_start >= seconds:
            break
    best = min(times)
    return {"value": len(jobs) * sample / best / 1e9, "cores": threads, "reps": len(times),
            "best_s": best, "median_s": statistics.median(times), "lib": libname,
            "ops": [lbl for lbl, _ in jobs], "sample": sample,
            "per_op_gelems": {lbl: round(sample / min(v) / 1e9, 5) for lbl, v in per_job.items()}}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


CONFIG_TEXT = {
    "C1": ("C1: fp8 1/4/3 elementwise add, N=2^24 per GPU; float32 U[-16,16] -> encode_scalar "
           "-> planes", "1/4/3", 1 << 24),
    "C2": ("C2: fp8 1/4/3 elementwise mul + sub, N=2^26 per GPU; raw encodings (random sign, all "
           "16 exponent codes incl. subnormal/Inf/NaN, 1% zeros)", "1/4/3", 1 << 26),
    "C3": ("C3: 1/5/10 float32->bitslice pack, add, mul, bitslice->float32 unpack, N=2^28 per GPU, "
           "each timed separately; float32 normal(0,100) clamped to +-65504", "1/5/10", 1 << 28),
    "C4": ("C4: add + mul sweep over 1/3/2, 1/5/3, 1/5/7, 1/8/7, 1/8/15, N=2^28 per GPU per "
           "format; uniform finite bit patterns", "sweep", 1 << 28),
    "C5": ("C5: 1/6/9 z=round(round(a*b)+c) fused, N=2^32 total split evenly over the GPUs; "
           "float32 sign x 2^U[-10,9] x U[1,2) -> encode_scalar", "1/6/9", None),
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


def scaling_of(cfg: str) -> str:
    """C5 splits a fixed 2^32 elements over the GPUs (strong); every other
    config fixes the per-GPU N (weak)."""
    return "strong" if cfg == "C5" else "weak"


def config_block(cfg: str, world: int, jobs=None) -> dict:
    text, fmt, n = CONFIG_TEXT[cfg]
    d = {"workload": text, "format": fmt, "rounding": "rn" if MODE[0] else "rz",
         "subnormals": "ftz" if MODE[1] else "gradual",
         "parallelism": f"dp{world} (independent block-aligned shards, no collective)",
         "l2": "inputs larger than L2: operand sets rotate step by step so each set is reused "
               "only after >= 2x L2 (126 MB) of other traffic; outputs rotate over two buffers"}
    if n:
        d["n_per_gpu"] = n
    else:
        d["n_total"] = 1 << 32
    if jobs is not None:
        d["ops_per_step"] = [j.label for j in jobs]
    return d


# ------------------------------------------------------------------- arms
def main_reference(args) -> None:
    world, rank, local = env_dist()
    if rank != 0:
        return
    for cfg in args.configs:
        sample = REF_SAMPLE[cfg]
        r = ref_cpu_run(cfg, sample, reps=args.warmup)  # warm-up steps
        r = ref_cpu_run(cfg, sample, reps=args.steps)
        r1 = ref_cpu_run(cfg, sample, reps=3, threads=1)  # thread-scaling check
        value = r["value"]
        line = {
            "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(r["median_s"] * 1e3, 3), "higher_is_better": True,
            "scaling": scaling_of(cfg), "vs_baseline": None, "dtype": "u64 lanes (lane<1024> bitslice)",
            "data": "synthetic (seeded SplitMix64 operands; BASELINE.json configs)",
            "config": config_block(cfg, world),
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": r["cores"],
                             "kind": "reference",
                             "sample": f"{r['sample']} elements x {r['ops']} per step, "
                                       f"lane<1024>, {r['cores']} threads, {cpu_model()}, "
                                       f"{r['lib']}",
                             "per_op": r["per_op_gelems"], "nproc": os.cpu_count(),
                             "value_1_thread": round(r1["value"], 4),
                             "thread_scaling": round(value / r1["value"], 2)},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)


def main_ours(args) -> None:
    import torch
    import torch.distributed as dist

    world, rank, local = env_dist()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    log = (lambda m: print(f"[bench r{rank}] {m}", file=sys.stderr, flush=True))
    peak_lop3 = None
    hbm_2r1w = None
    for cfg in args.configs:
        log(f"device timing {cfg}")
        res = run_device(cfg, args.steps, args.warmup, world, rank, local)
        if clocks_rejected(res["clocks"]):  # re-measure once
            log("clocks rejected; re-measuring")
            res = run_device(cfg, args.steps, args.warmup, world, rank, local, jobs=res["jobs"])
        jobs = res["jobs"]
        log(f"device done: {res['ms_total'] / args.steps:.4f} ms/step; e2e")
        e2e = run_e2e(cfg, jobs, args.steps, world, rank, local) if not args.no_e2e else None
        if peak_lop3 is None and rank == 0:
            log("lop3 probe")
            peak_lop3 = lop3_peak(local)
            hbm_2r1w = hbm_2r1w_probe(local)

        total_elems = sum(j.n for j in jobs) * world
        ms_step = res["ms_total"] / args.steps
        value = total_elems / (ms_step * 1e-3) / 1e9
        peaks = measured_peaks()
        per_op = {}
        roofs = []
        tfile = ROOT / "profiles" / "ncu_traffic.json"
        tmap = json.loads(tfile.read_text()) if tfile.exists() else {}
        tsuf = "" if MODE == (1, 0) else f":{mode_text()}"
        for j, ms in zip(jobs, res["kern_ms"]):
            dur = ms * 1e-3
            ach = j.algo_bytes / dur / 1e9
            e, s = j.spec.exp_bits, j.spec.sig_bits
            ent = {"ms": round(ms, 4), "gelem_s": round(j.n / dur / 1e9, 2),
                   "hbm_gbs": round(ach, 1), "hbm_frac": round(ach / peaks["hbm_gbs"], 4)}
            chain_ops = ([{"+": "add", "-": "sub", "*": "mul", "/": "div"}[ch]
                          for ch in j.op.split(":", 1)[1] if ch in "+-*/"]
                         if j.op.startswith("chain:") else None)
            if j.op in OPNAMES or chain_ops:
                if chain_ops:
                    parts = [sass_lop3((e, s), int(j.spec.rounding), int(j.spec.subnormals), OPNAMES[o])
                             for o in chain_ops]
                    lop3 = None if None in parts else sum(parts)
                else:
                    lop3 = sass_lop3((e, s), int(j.spec.rounding), int(j.spec.subnormals), OPNAMES[j.op])
                if lop3 is not None and peak_lop3:
                    pe = lop3 / 32.0
                    hbm_t = j.algo_bytes / (peaks["hbm_gbs"] * 1e9)
                    logic_t = pe * j.n / peak_lop3["burst"]
                    ent.update({"lop3_per_elem": round(pe, 3),
                                "logic_frac": round(logic_t / dur, 4),
                                "logic_frac_at_load_clock": load_clock_frac(pe * j.n, dur, peak_lop3,
                                                                            res["clocks"]),
                                "binding": "logic" if logic_t > hbm_t else "hbm",
                                "frac_of_binding": round(max(hbm_t, logic_t) / dur, 4)})
            tr = tmap.get(f"{cfg}:{j.label}{tsuf}")
            if isinstance(tr, dict):
                ent["ncu"] = {k: v for k, v in tr.items() if k != "bytes"}
                tr = tr.get("bytes")
            if tr is not None:
                ent["traffic"] = tr
                ent["traffic_over_algorithmic"] = round(tr / j.algo_bytes, 3)
            per_op[j.label] = ent
            roofs.append((ms, j, ach))
        ms_dom, jd, ach = max(roofs, key=lambda r: r[0])
        traffic = tmap.get(f"{cfg}:{jd.label}{tsuf}")
        if isinstance(traffic, dict):
            traffic = traffic.get("bytes")
        roof = {"bound": "hbm", "kernel": f"{jd.label} (1/{jd.spec.exp_bits}/{jd.spec.sig_bits} {mode_text()})",
                "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(ach / peaks["hbm_gbs"], 4), "traffic": traffic,
                "peak_source": peaks["source"],
                "hbm_2r1w_probe_gbs": hbm_2r1w,
                "algorithmic_bytes_per_launch": int(jd.algo_bytes),
                "launch_ms": round(ms_dom, 4), "per_op": per_op}
        if peak_lop3:
            roof["peak_lop3_per_s_measured"] = peak_lop3["burst"]
            roof["peak_lop3_per_s_sustained"] = peak_lop3["sustained"]
            roof["peak_lop3_sustained_sm_mhz"] = peak_lop3["sustained_sm_mhz"]
        step_bytes = sum(j.algo_bytes for j in jobs)
        step_gbs = step_bytes / (ms_step * 1e-3) / 1e9
        # self-check: inputs rotate through > 2x L2, so no step or kernel can
        # beat the HBM copy peak; a faster figure means the timing is broken
        for j, ms in zip(jobs, res["kern_ms"]):
            if j.algo_bytes / (ms * 1e-3) / 1e9 > 1.1 * peaks["hbm_gbs"] * world:
                raise RuntimeError(f"{cfg}:{j.label}: {ms} ms per launch is faster than HBM allows")
        if step_gbs > 1.1 * peaks["hbm_gbs"] * world:
            raise RuntimeError(f"{cfg}: step time {ms_step} ms is faster than HBM allows")
        roof["step"] = {"algorithmic_bytes": int(step_bytes), "ms": round(ms_step, 5),
                        "achieved_gbs": round(step_gbs, 1),
                        "frac": round(step_gbs / peaks["hbm_gbs"], 4),
                        "note": "whole step: K steps captured once into a CUDA graph through the "
                                "C ABI and replayed (consecutive kernels overlap through "
                                "programmatic dependent launch); per-kernel figures above come "
                                "from one graph per kernel holding its K launches",
                        "ms_per_step_eager": round(res["ms_total_eager"] / args.steps, 5)}
        pw = res["clocks"].get("power_w")
        if pw:  # board energy per result element at the sampled draw (the logic kernels run power-capped)
            roof["step"]["pj_per_elem"] = round(pw * ms_step * 1e-3 / (total_elems / world) * 1e12, 1)
        dd = per_op[jd.label]
        if "binding" in dd:
            roof["binding_leg"] = dd["binding"]
            roof["frac_of_binding"] = dd["frac_of_binding"]
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
            "higher_is_better": True, "scaling": scaling_of(cfg), "vs_baseline": None,
            "dtype": "u32 (bitslice words)",
            "data": "synthetic (seeded SplitMix64 operands; BASELINE.json configs)",
            "config": config_block(cfg, world, jobs),
            "roofline": roof,
            "clocks": res["clocks"],
            "gpu_launches": res["launches"],
        }
        if e2e is not None:
            pcie = pcie_probe(local)
            # copy-only time of the step's traffic at the measured link rates
            bound_s = max(e2e["h2d"] / (pcie["h2d_gbs"] * 1e9), e2e["d2h"] / (pcie["d2h_gbs"] * 1e9),
                          (e2e["h2d"] + e2e["d2h"]) / (pcie["bidir_gbs"] * 1e9))
            line["e2e"] = {"value": round(e2e["elems"] * world / e2e["s_per_step"] / 1e9, 3),
                           "pcie_measured": pcie,
                           "frac_of_pcie_bound": round(bound_s / e2e["s_per_step"], 4),
                           "unit": UNIT, "h2d_bytes_per_step": int(e2e["h2d"]),
                           "d2h_bytes_per_step": int(e2e["d2h"]),
                           "path": "C ABI host entry points (bfp_arith_host_batch / "
                                   "bfp_pack_f32_host / bfp_unpack_f32_host: pinned host buffers; "
                                   "inputs copied H2D in chunk order on one stream, kernels on a "
                                   "second write each chunk's results in place into the pinned "
                                   "host outputs over PCIe; ops sharing operands copy them once)",
                           "steps": e2e["steps"]}
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            log("cpu baseline")
            cb = ref_cpu_run(cfg, REF_SAMPLE[cfg], seconds=args.cpu_seconds)
            c1 = ref_cpu_run(cfg, REF_SAMPLE[cfg], reps=3, threads=1)  # thread-scaling check
            line["cpu_baseline"] = {
                "value": round(cb["value"], 4), "unit": UNIT, "cores": cb["cores"],
                "kind": "reference",
                "sample": f"{cb['sample']} elements x {cb['ops']} per step, best of {cb['reps']} "
                          f"steps (~{args.cpu_seconds:.0f} s), lane<1024>, {cb['cores']} threads, "
                          f"{cpu_model()}, {cb['lib']}",
                "per_op": cb["per_op_gelems"], "nproc": os.cpu_count(),
                "value_1_thread": round(c1["value"], 4),
                "thread_scaling": round(cb["value"] / c1["value"], 2)}
        del jobs, res
        torch.cuda.empty_cache()
        if rank == 0:
            print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    faulthandler.enable()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C2", help="C1..C5, comma list, or 'all'")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--rounding", choices=["rn", "rz"], default="rn")
    ap.add_argument("--subnormals", choices=["gradual", "ftz"], default="gradual")
    args = ap.parse_args()
    global MODE
    MODE = (int(args.rounding == "rn"), int(args.subnormals == "ftz"))
    args.configs = (["C1", "C2", "C3", "C4", "C5"] if args.config == "all"
                    else args.config.split(","))
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        main_reference(args)
    else:
        main_ours(args)


if __name__ == "__main__":
    main()
