"""The post-mapping optimiser of the LOP3 covers (tools/lutmap/resub.hpp):
window resubstitution with don't-cares + node elimination.

Every rewrite it makes is meant to preserve the network's function on all
reachable inputs; here the optimised networks of the small formats are compared
with the template's AND/XOR graph on EVERY input combination (up to all 2^24
(a, b, c) triples of the 1/4/3 fused mul_add), and must not be larger than the
structural mapper's cover.  The covers the kernels run are additionally checked
like any network by test_circuits_host.py (host) and the -m gpu suite.
"""
from __future__ import annotations

import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LUTMAP = ROOT / "tools" / "lutmap"
CSRC = ROOT / "paper_1602_04716_b200" / "csrc"


def test_optimised_networks_exhaustive(tmp_path):
    exe = tmp_path / "resub_check"
    subprocess.run(["g++", "-O2", "-std=c++17", f"-I{LUTMAP}", f"-I{CSRC}", str(LUTMAP / "resub_check.cpp"),
                    "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600)
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert r.returncode == 0, r.stdout + r.stderr
    assert len(lines) == 10
    saved = 0
    for l in lines:
        f = l.split()
        assert f[-1] == "ok", l
        mapped, optimised = int(f[f.index("mapped") + 1]), int(f[f.index("optimised") + 1])
        assert optimised <= mapped, l
        saved += mapped - optimised
    assert saved > 0  # the pass does something on these networks
