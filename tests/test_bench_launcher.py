"""bench.py's multi-rank path on the CPU: `--gpus N` re-launches itself under
torch.distributed.run with N ranks; --dry-run runs them on gloo with a
stand-in step.  Checks the shard ranges (contiguous,
block-aligned, covering N), the max-over-ranks time reduction, and that
rank 0 alone prints the JSON line.  Also the L2 reuse accounting of the
operand rotation (no GPU needed)."""
from __future__ import annotations

import json
import subprocess
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, str(ROOT))


def _dry(*args: str) -> tuple[list[dict], str]:
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--dry-run", *args], capture_output=True,
                       text=True, timeout=300, cwd=ROOT, env={**__import__("os").environ, "OMP_NUM_THREADS": "1"})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    return lines, r.stderr


@pytest.mark.parametrize("gpus,cfg", [(2, "default"), (4, "C5"), (2, "C4")])
def test_dry_run_world(gpus, cfg):
    lines, err = _dry("--gpus", str(gpus), "--config", cfg, "--steps", "3", "--warmup", "3")
    assert len(lines) == 1, lines  # rank 0 alone prints
    d = lines[0]
    assert d["dry_run"] is True and d["n_gpus"] == gpus and d["steps"] == 3
    ranks = sorted(d["ranks"], key=lambda r: r["rank"])
    assert [r["rank"] for r in ranks] == list(range(gpus))
    assert sorted(r["local_rank"] for r in ranks) == list(range(gpus))
    # max over ranks: the slowest rank's total (the stand-in delay grows with rank)
    assert d["ms_total_max"] == pytest.approx(max(r["ms_total"] for r in ranks))
    assert d["ms_per_step"] == pytest.approx(d["ms_total_max"] / 3)
    assert d["ms_total_max"] >= ranks[-1]["ms_total"] - 1e-9
    shards = [r["shard"] for r in ranks]
    if cfg in ("default", "C5"):  # strong scaling: a fixed 2^32 split over the ranks
        assert d["scaling"] == "strong" and d["n_total"] == 1 << 32
        assert shards[0][0] == 0 and shards[-1][1] == 1 << 32
        for (a, b), (c, _) in zip(shards, shards[1:]):
            assert b == c
        assert all(lo % 1024 == 0 and hi - lo == (1 << 32) // gpus for lo, hi in shards)
    else:  # weak scaling: every rank its own 2^28 block
        assert d["scaling"] == "weak" and d["n_total"] == gpus << 28
        assert shards == [[r << 28, (r + 1) << 28] for r in range(gpus)]
    assert f"gloo process group up: rank {gpus - 1}/{gpus}" in err


def test_gpus_mismatch_rejected():
    import os
    env = {**os.environ, "WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--dry-run"],
                       capture_output=True, text=True, timeout=120, cwd=ROOT, env=env)
    assert r.returncode != 0 and "WORLD_SIZE=2" in r.stderr


class _Spec:
    def __init__(self, nb):
        self.nb = nb

    def plane_bytes(self, n):
        return -(-n // 1024) * self.nb * 128


class _J:
    def __init__(self, touch):
        self.touch = touch


@pytest.mark.parametrize("nb,n,nin,per_step", [(8, 1 << 24, 2, 1), (8, 1 << 26, 2, 2), (16, 1 << 20, 3, 1)])
def test_rotation_keeps_reuse_beyond_2x_l2(nb, n, nin, per_step):
    import bench
    spec = _Spec(nb)
    k = bench.rotation_sets(spec, n, nin, per_step)
    pb = spec.plane_bytes(n)
    jobs = [_J(lambda i, s=s: (("sets", (per_step * i + s) % k), nin * pb, pb)) for s in range(per_step)]
    d = bench.l2_reuse_distance(jobs)
    assert d >= 2 * bench.L2_BYTES
    if k > per_step:  # one set fewer would break it
        k -= 1
        assert 0 <= bench.l2_reuse_distance(jobs) < 2 * bench.L2_BYTES
