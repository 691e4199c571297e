"""bench.py keeps the driver's JSON-line contract (both arms): the default
headline line (C5 + the C4 per-format sweep) and a short C1 line."""
from __future__ import annotations

import json
import subprocess
import sys

import pytest

from conftest import ROOT, full_suite_only

pytestmark = pytest.mark.gpu


def _run(*args: str) -> dict:
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                       timeout=1500, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


BASE_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "gpu_launches",
             "e2e", "cpu_baseline")


def _check_roofline(r: dict):
    assert r["bound"] in ("hbm", "logic")
    assert r["unit"] == ("GB/s" if r["bound"] == "hbm" else "TLOP3/s")
    assert 0 < r["frac"] <= 1.5 and abs(r["achieved"] / r["peak"] - r["frac"]) < 2e-3
    lead = r["legs"][r["bound"]]
    assert lead["achieved"] == r["achieved"] and lead["peak"] == r["peak"]
    if r["bound"] == "logic":  # recomputable: LOP3/elem x elements per launch / launch time
        lg = r["legs"]["logic"]
        ach = lg["lop3_per_elem"] * r["elements_per_launch"] / (r["launch_ms"] * 1e-3) / 1e12
        assert ach == pytest.approx(r["achieved"], rel=2e-3)


def test_default_headline_line():
    d = _run("--steps", "5", "--warmup", "3", "--cpu-seconds", "2")
    for k in BASE_KEYS + ("per_format", "ranks"):
        assert k in d, k
    assert d["config"]["workload"].startswith("C5") and d["scaling"] == "strong"
    assert d["config"]["n_total"] == 1 << 32 and d["config"]["per_format_configs"] == ["C5", "C4"]
    assert d["gpu_launches"] == 5 and d["n_gpus"] == 1
    r = d["roofline"]
    _check_roofline(r)
    # C5's operands lie in mul_add's fast domain: the smaller cover runs and the
    # kernel sits between its two legs (either may bind, box by box)
    assert r["bound"] in ("hbm", "logic") and r["kernel"].startswith("mul_add")
    assert {"hbm", "logic"} <= set(r["legs"])
    assert r["traffic"] and 0.8 < r["traffic_over_algorithmic"] < 1.3, r.get("traffic_source")
    pf = d["per_format"]
    assert set(pf) == {"1/6/9", "1/3/2", "1/5/3", "1/5/7", "1/8/7", "1/8/15"}
    assert set(pf["1/6/9"]) == {"mul_add", "mul_add (general_network)"}
    fast, gen = pf["1/6/9"]["mul_add"], pf["1/6/9"]["mul_add (general_network)"]
    assert fast["lop3_per_elem"] < gen["lop3_per_elem"] and gen["gelem_s"] > 0
    assert fast["fast_cover_blocks_frac"] == 1.0  # C5's operands: every block inside the fast domain
    # which cover ran, measured: executed ALU instructions per element (ncu, this run)
    assert fast["alu_inst_per_elem_measured"] < gen["lop3_per_elem"]
    for fmt in ("1/3/2", "1/5/3", "1/5/7", "1/8/7", "1/8/15"):
        for op in ("add", "mul"):
            ent = pf[fmt][op]
            assert ent["gelem_s"] > 0 and ent["bound"] in ("hbm", "logic") and 0 < ent["frac"] <= 1.5
            assert ent["cpu_gelem_s"] > 0
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] == 3 * (1 << 33) and e["d2h_bytes_per_step"] == 1 << 33
    c = d["cpu_baseline"]
    assert c["value"] > 0 and c["value_median"] > 0 and c["kind"] == "reference" and c["cores"] >= 1


@full_suite_only
def test_c1_line():
    d = _run("--config", "C1", "--steps", "4", "--warmup", "3", "--cpu-seconds", "2")
    for k in BASE_KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] >= 4
    assert d["config"]["workload"].startswith("C1")
    _check_roofline(d["roofline"])
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 2 * (1 << 24) and e["d2h_bytes_per_step"] == 1 << 24
    c = d["cpu_baseline"]
    assert c["value"] > 0 and c["cores"] >= 1 and c["kind"] in ("reference", "port") and c["sample"]
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@full_suite_only
def test_reference_line():
    d = _run("--impl", "reference", "--steps", "2", "--warmup", "1", "--cpu-seconds", "2")
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("C5")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["value"] == d["value"]
    assert set(d["per_format"]) == {"1/6/9", "1/3/2", "1/5/3", "1/5/7", "1/8/7", "1/8/15"}
    # same config block as our arm's line
    from bench import config_block  # noqa: E402
    import bench
    want = config_block("C5", 1)
    want["per_format_configs"] = ["C5", "C4"]
    assert d["config"] == want
