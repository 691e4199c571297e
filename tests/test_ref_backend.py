"""The reference-side binding (integration/bfp/gpu_backend.hpp, INTEGRATION.md
§2): the adapter a maintainer would add to the reference tree, compiled
against the UNMODIFIED reference headers (oracle/Makefile `backend`, where
/root/reference exists; the binary travels prebuilt in oracle/_ref/), run on
the B200 and byte-compared with the reference's own bfp_add / bfp_sub /
bfp_mul / bfp_div and bfp_add(bfp_mul(a, b), c) on the same
bfp_vector<lane<1024>> operands (tests/native/ref_backend_test.cpp)."""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

from conftest import ROOT

EXE = ROOT / "oracle" / "_ref" / "ref_backend_test"
REF = Path("/root/reference/proj/include/bfp/arith.hpp")


@pytest.mark.skipif(not REF.exists(), reason="reference tree not present (GPU box)")
def test_backend_builds_against_reference():
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "backend"], check=True, timeout=600)
    assert EXE.exists()
    ldd = subprocess.run(["ldd", str(EXE)], capture_output=True, text=True).stdout
    assert "libbfpgpu.so" in ldd and "not found" not in ldd.split("libbfpgpu.so", 1)[1].splitlines()[0]


@pytest.mark.gpu
def test_backend_matches_reference_operators():
    if not EXE.exists():
        pytest.skip("oracle/_ref/ref_backend_test not built (needs /root/reference at build time)")
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.startswith("ok ") and "identical to the reference" in r.stdout
    print(r.stdout.strip())
