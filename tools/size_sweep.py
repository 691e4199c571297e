"""Per-launch time and throughput of one op against the vector size, with and
without BFP_INPUTS_READY -- where launch latency and the load ramp stop
mattering.  Each point: K launches captured in one CUDA graph over operand
sets rotated so every set is re-read only after >= 2x L2 of other traffic.

    python tools/size_sweep.py [--fmt 4,3] [--op add] [--k 200]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--fmt", default="4,3")
    ap.add_argument("--op", default="add")
    ap.add_argument("--k", type=int, default=200)
    a = ap.parse_args()
    import torch
    import paper_1602_04716_b200 as bfp
    L = bfp.lib()
    e, s = map(int, a.fmt.split(","))
    spec = bfp.make_spec(e, s)
    op = {"add": 0, "sub": 1, "mul": 2, "div": 3}[a.op]
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6551.4) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else 6551.4
    l2 = 126 << 20
    rows = []
    for lg in range(14, 29, 2):
        n = 1 << lg
        pb = spec.plane_bytes(n)
        sets = max(2, -(-2 * l2 // (2 * pb)))
        g = torch.Generator(device="cuda").manual_seed(lg)
        ops = [torch.randint(-2**31, 2**31 - 1, (pb // 4,), dtype=torch.int32, device="cuda", generator=g)
               for _ in range(2 * sets)]
        outs = [torch.empty(pb // 4, dtype=torch.int32, device="cuda") for _ in range(2)]
        res = {"n": n}
        for flag in (0, 1):
            st = torch.cuda.Stream()

            def run(k0, k1):
                for i in range(k0, k1):
                    x, y = ops[2 * (i % sets)], ops[2 * (i % sets) + 1]
                    rc = L.bfp_arith_ex(op, spec.c, x.data_ptr(), y.data_ptr(), None, outs[i & 1].data_ptr(), n,
                                        st.cuda_stream, flag)
                    assert rc == 0
            run(0, 8)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=st):
                run(0, a.k)
            graph.replay()
            torch.cuda.synchronize()
            best = 1e9
            for _ in range(3):
                t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                t0.record()
                graph.replay()
                t1.record()
                torch.cuda.synchronize()
                best = min(best, t0.elapsed_time(t1) / a.k)
            gbs = 3 * pb / (best * 1e-3) / 1e9
            res[f"flag{flag}"] = {"us": round(best * 1e3, 2), "gelem_s": round(n / (best * 1e-3) / 1e9, 1),
                                  "hbm_frac": round(gbs / peak, 3)}
            del graph
        rows.append(res)
        print(json.dumps(res), flush=True)
        del ops, outs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
