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
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

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
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


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
    except Exception:
        return None
    return None


# ------------------------------------------------------------ the workloads
def make_inputs(cfg: str, rank: int, world: int, device):
    """Per-rank operands of config `cfg` as resident planes."""
    import torch
    import paper_1602_04716_b200 as bfp
    from paper_1602_04716_b200 import workloads as W

    if cfg == "C1":
        n = 1 << 24
        spec = bfp.make_spec(4, 3)
        lo = rank * n
        a = bfp.pack_f32(W.c1_floats(lo, lo + n, W.SEED_A, device), spec)
        b = bfp.pack_f32(W.c1_floats(lo, lo + n, W.SEED_B, device), spec)
        return spec, n, [("add", a, b, None)]
    if cfg == "C2":
        n = 1 << 26
        spec = bfp.make_spec(4, 3)
        lo = rank * n
        a = bfp.pack(W.c2_encodings(lo, lo + n, W.SEED_A, device), spec)
        b = bfp.pack(W.c2_encodings(lo, lo + n, W.SEED_B, device), spec)
        return spec, n, [("mul", a, b, None), ("sub", a, b, None)]
    if cfg == "C5":
        total = 1 << 32
        lo, hi = W.shard(total, rank, world)
        spec = bfp.make_spec(6, 9)
        ops = [bfp.pack_f32(W.c5_floats(lo, hi, sd, device), spec)
               for sd in (W.SEED_A, W.SEED_B, W.SEED_C)]
        torch.cuda.empty_cache()
        return spec, hi - lo, [("mul_add", ops[0], ops[1], ops[2])]
    raise ValueError(cfg)


def algorithmic_bytes(op: str, nbits: int, n: int) -> float:
    if op == "mul_add":
        return 4 * nbits / 8 * n
    if op == "pack_f32":
        return (4 + nbits / 8) * n
    if op == "unpack_f32":
        return (nbits / 8 + 4) * n
    return 3 * nbits / 8 * n


def run_device(cfg: str, steps: int, warmup: int, world: int, rank: int, local: int) -> dict:
    import torch
    import torch.distributed as dist
    import paper_1602_04716_b200 as bfp

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    L = bfp.lib()
    spec, n, ops = make_inputs(cfg, rank, world, device)
    nbits = spec.total_bits()
    # two rotating output sets; inputs (2 x n*nbits/8 B) + outputs exceed L2
    outs = [[bfp.empty(spec, n, device) for _ in ops] for _ in range(2)]
    stream = torch.cuda.current_stream(device)

    def step(i, evs=None):
        for k, (op, a, b, c) in enumerate(ops):
            if evs is not None:
                evs[k][0].record(stream)
            z = outs[i & 1][k]
            rc = L.bfp_arith(OPNAMES[op], spec.c, a.planes.data_ptr(), b.planes.data_ptr(),
                             c.planes.data_ptr() if c is not None else None, z.planes.data_ptr(),
                             n, stream.cuda_stream)
            if rc != 0:
                raise RuntimeError(L.bfp_last_error())
            if evs is not None:
                evs[k][1].record(stream)

    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()

    # sustained window of the same step for the clock record (~1.5 s)
    t_probe = time.perf_counter()
    step(0)
    torch.cuda.synchronize()
    one = max(time.perf_counter() - t_probe, 1e-5)
    reps = max(1, int(1.5 / one))
    with ClockSampler(local) as cs:
        for i in range(reps):
            step(i)
        torch.cuda.synchronize()
    clocks = cs.summary()

    # timed region
    per_kernel = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                   for _ in range(steps)] for _ in ops]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = L.bfp_launch_count()
    t0.record(stream)
    for i in range(steps):
        step(i, [[per_kernel[k][i][0], per_kernel[k][i][1]] for k in range(len(ops))])
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = L.bfp_launch_count() - launches0
    ms_total = t0.elapsed_time(t1)
    kern_ms = [sum(per_kernel[k][i][0].elapsed_time(per_kernel[k][i][1]) for i in range(steps)) / steps
               for k in range(len(ops))]
    if world > 1:
        t = torch.tensor([ms_total], device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    return {"spec": spec, "n": n, "ops": [o[0] for o in ops], "ms_total": ms_total,
            "kern_ms": kern_ms, "clocks": clocks, "launches": int(launches), "nbits": nbits}


def run_e2e(cfg: str, steps: int, world: int, rank: int, local: int) -> dict:
    """The same step through the C ABI with HOST planes (pinned): every step
    copies its inputs H2D and its results D2H inside the timed region."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1602_04716_b200 as bfp

    device = torch.device("cuda", local)
    L = bfp.lib()
    spec, n, ops = make_inputs(cfg, rank, world, device)
    pb = spec.plane_bytes(n)
    ctx = L.bfp_host_ctx_create(1 << 22)
    bufs = []

    def host_copy(t):
        p = L.bfp_host_alloc(pb)
        if not p:
            raise RuntimeError("bfp_host_alloc failed")
        bufs.append(p)
        src = t.planes.cpu().numpy()  # keep alive across the copy
        C.memmove(p, src.ctypes.data, pb)
        del src
        return p

    try:
        hops = []
        for op, a, b, c in ops:
            hops.append((op, host_copy(a), host_copy(b), host_copy(c) if c is not None else None,
                         L.bfp_host_alloc(pb)))
            bufs.append(hops[-1][4])
        del ops
        torch.cuda.empty_cache()

        def step():
            for op, ha, hb, hc, hz in hops:
                rc = L.bfp_arith_host(ctx, OPNAMES[op], spec.c, ha, hb, hc, hz, n)
                if rc != 0:
                    raise RuntimeError(L.bfp_last_error())

        step()
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        k = max(2, steps // 4)
        for _ in range(k):
            step()
        dt = (time.perf_counter() - t) / k
        if world > 1:
            tt = torch.tensor([dt], device=device)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
        n_in = sum(3 if o[3] is not None else 2 for o in hops)
        return {"s_per_step": dt, "h2d": n_in * pb, "d2h": len(hops) * pb, "elems": len(hops) * n}
    finally:
        for p in bufs:
            L.bfp_host_free(p)
        L.bfp_host_ctx_destroy(ctx)


def lop3_peak() -> float | None:
    import paper_1602_04716_b200 as bfp
    ms, rate = C.c_float(), C.c_double()
    if bfp.lib().bfp_probe_lop3(4000, C.byref(ms), C.byref(rate)) != 0:
        return None
    return rate.value


# --------------------------------------------------------- reference (CPU)
def ref_cpu_run(cfg: str, sample: int, reps: int | None = None, seconds: float = 10.0,
                threads: int | None = None) -> dict:
    """The reference templates (oracle/_ref: unmodified headers + shim) over
    `sample` elements of the config's operands, lane<1024>, all host cores."""
    import numpy as np
    import torch
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as O
    from paper_1602_04716_b200 import workloads as W

    threads = threads or os.cpu_count() or 1
    if cfg == "C2":
        fmt, opl = (4, 3, 1, 0), ["mul", "sub"]
        a = W.c2_encodings(0, sample, W.SEED_A, "cpu").numpy().astype(np.uint64)
        b = W.c2_encodings(0, sample, W.SEED_B, "cpu").numpy().astype(np.uint64)
        c = None
    elif cfg == "C1":
        fmt, opl = (4, 3, 1, 0), ["add"]
        a = O.encode_f32(fmt, W.c1_floats(0, sample, W.SEED_A, "cpu").numpy())
        b = O.encode_f32(fmt, W.c1_floats(0, sample, W.SEED_B, "cpu").numpy())
        c = None
    elif cfg == "C5":
        fmt, opl = (6, 9, 1, 0), ["mul_add"]
        a, b, c = (O.encode_f32(fmt, W.c5_floats(0, sample, sd, "cpu").numpy())
                   for sd in (W.SEED_A, W.SEED_B, W.SEED_C))
    else:
        raise ValueError(cfg)
    nb = 1 + fmt[0] + fmt[1]
    pa, pb = O.pack_planes(a, nb), O.pack_planes(b, nb)
    pc = O.pack_planes(c, nb) if c is not None else None
    times = []
    t_start = time.perf_counter()
    while True:
        t = time.perf_counter()
        for op in opl:
            O.ref_binop_planes(op, fmt, pa, pb, pc, threads=threads)
        times.append(time.perf_counter() - t)
        if reps is not None and len(times) >= reps:
            break
        if reps is None and time.perf_counter() - t_start >= seconds:
            break
    best = min(times)
    return {"value": len(opl) * sample / best / 1e9, "cores": threads, "reps": len(times),
            "best_s": best, "median_s": statistics.median(times), "lib": O.ref_lib_path().name,
            "ops": opl, "sample": sample}


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def config_block(cfg: str, world: int) -> dict:
    base = {"l2": "inputs + outputs > L2 (126 MB); two rotating output sets",
            "parallelism": f"dp{world} (independent shards, no collective)",
            "rounding": "rn", "subnormals": "gradual"}
    if cfg == "C2":
        return {"workload": "C2: fp8 1/4/3 elementwise mul + sub, N=2^26 per GPU, raw encodings "
                            "(random sign, all 16 exponent codes, 1% zeros)",
                "format": "1/4/3", "n_per_gpu": 1 << 26, "ops_per_step": ["mul", "sub"], **base}
    if cfg == "C1":
        return {"workload": "C1: fp8 1/4/3 elementwise add, N=2^24 per GPU, float32 U[-16,16] "
                            "-> encode_scalar", "format": "1/4/3", "n_per_gpu": 1 << 24,
                "ops_per_step": ["add"], **base}
    if cfg == "C5":
        return {"workload": "C5: 1/6/9 z=round(round(a*b)+c), N=2^32 total split over GPUs",
                "format": "1/6/9", "n_total": 1 << 32, "ops_per_step": ["mul_add"], **base}
    return {"workload": cfg, **base}


# ------------------------------------------------------------------- arms
def main_reference(args) -> None:
    world, rank, local = env_dist()
    if rank != 0:
        return
    cfg = args.config
    sample = {"C2": 1 << 24, "C1": 1 << 24, "C5": 1 << 22}[cfg]
    for _ in range(args.warmup):
        ref_cpu_run(cfg, sample, reps=1)
    r = ref_cpu_run(cfg, sample, reps=args.steps)
    ms = r["median_s"] * 1e3
    value = r["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32 (bitslice)",
        "data": "synthetic (seeded SplitMix64 operands; BASELINE.json configs)",
        "config": config_block(cfg, world),
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": r["cores"],
                         "kind": "reference",
                         "sample": f"{r['sample']} elements x {r['ops']} per step, lane<1024>, "
                                   f"{r['cores']} threads, {cpu_model()}, {r['lib']}"},
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
    cfg = args.config
    log = (lambda m: print(f"[bench r{rank}] {m}", file=sys.stderr, flush=True))
    log(f"device timing {cfg}")
    res = run_device(cfg, args.steps, args.warmup, world, rank, local)
    if clocks_rejected(res["clocks"]):  # re-measure once
        res = run_device(cfg, args.steps, args.warmup, world, rank, local)
    log(f"device done: {res['ms_total'] / args.steps:.4f} ms/step; e2e")
    e2e = run_e2e(cfg, args.steps, world, rank, local)
    log("lop3 probe")
    peak_lop3 = lop3_peak() if rank == 0 else None

    spec, n, nbits = res["spec"], res["n"], res["nbits"]
    total_elems = n * len(res["ops"]) * world
    ms_step = res["ms_total"] / args.steps
    value = total_elems / (ms_step * 1e-3) / 1e9
    k_dom = max(range(len(res["ops"])), key=lambda k: res["kern_ms"][k])
    op_dom = res["ops"][k_dom]
    dur = res["kern_ms"][k_dom] * 1e-3
    algo = algorithmic_bytes(op_dom, nbits, n)
    peaks = measured_peaks()
    achieved = algo / dur / 1e9
    e, s = spec.exp_bits, spec.sig_bits
    lop3 = sass_lop3((e, s), int(spec.rounding), int(spec.subnormals), OPNAMES[op_dom])
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        tj = json.loads(tfile.read_text())
        traffic = tj.get(f"{cfg}:{op_dom}")
    roof = {
        "bound": "hbm", "kernel": f"k_arith<{e},{s},rn>:{op_dom}",
        "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
        "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": traffic,
        "peak_source": peaks["source"], "algorithmic_bytes_per_launch": int(algo),
        "launch_ms": round(dur * 1e3, 4),
        "per_op_ms": {o: round(t, 4) for o, t in zip(res["ops"], res["kern_ms"])},
    }
    if lop3 is not None and peak_lop3:
        per_elem = lop3 / 32.0
        ach = per_elem * n / dur
        roof["logic"] = {"lop3_per_elem_sass": round(per_elem, 3), "achieved_lop3_per_s": ach,
                         "peak_lop3_per_s_measured": peak_lop3, "frac": round(ach / peak_lop3, 4)}
        hbm_t = algo / (peaks["hbm_gbs"] * 1e9)
        logic_t = per_elem * n / peak_lop3
        roof["binding_leg"] = "logic" if logic_t > hbm_t else "hbm"
        roof["frac_of_binding"] = round(max(hbm_t, logic_t) / dur, 4)

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u32 (bitslice words; 1/4/3 custom FP)",
        "data": "synthetic (seeded SplitMix64 operands; BASELINE.json configs)",
        "config": config_block(cfg, world),
        "roofline": roof,
        "e2e": {"value": round(e2e["elems"] * world / e2e["s_per_step"] / 1e9, 3), "unit": UNIT,
                "h2d_bytes_per_step": int(e2e["h2d"]), "d2h_bytes_per_step": int(e2e["d2h"]),
                "path": "bfp_arith_host (C ABI, pinned host planes, chunked H2D/kernel/D2H)"},
        "clocks": res["clocks"],
        "gpu_launches": res["launches"],
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        log("cpu baseline")
        cb = ref_cpu_run(cfg, 1 << 22, seconds=args.cpu_seconds)
        line["cpu_baseline"] = {
            "value": round(cb["value"], 4), "unit": UNIT, "cores": cb["cores"], "kind": "reference",
            "sample": f"{cb['sample']} elements x {cb['ops']}, best of {cb['reps']} reps "
                      f"(~{args.cpu_seconds:.0f} s), lane<1024>, {cb['cores']} threads, "
                      f"{cpu_model()}, {cb['lib']}"}
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
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C5"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        main_reference(args)
    else:
        main_ours(args)


if __name__ == "__main__":
    main()
