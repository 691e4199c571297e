"""Out-of-bounds checks of every kernel family with guard pages (compute-
sanitizer is closed on the GPU pool): tests/fence_kernels.py maps each buffer
of a call so it ends -- or starts -- exactly at a page edge with unmapped pages
around it, so any access past either end faults; results must also equal the
same call on ordinary buffers.  Run in a subprocess (a fault poisons the CUDA
context), once with the plain arithmetic kernels and once with the
cp.async.bulk + mbarrier ring variant (BFP_BULK=2).  Log:
profiles/r02_fence.log."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("bulk", ["0", "2"])
def test_no_out_of_bounds_access(bulk):
    env = {**os.environ, "BFP_BULK": bulk}
    args = [sys.executable, str(ROOT / "tests" / "fence_kernels.py")] + (["--quick"] if bulk != "0" else [])
    r = subprocess.run(args, capture_output=True, text=True, timeout=1200, env=env, cwd=ROOT)
    print(r.stdout[-2000:])
    assert r.returncode == 0, (r.stdout[-3000:] + r.stderr[-3000:])
    assert "fence ok" in r.stdout
