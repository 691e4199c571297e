"""The C++ drop-in header (include/bfp/gpu.hpp) used the way a reference
user would: compiled against libbfpgpu.so, checked against the oracle."""
from __future__ import annotations

import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_cpp_api(tmp_path, oracle):
    exe = tmp_path / "cpp_api_test"
    lib = ROOT / "paper_1602_04716_b200"
    cmd = ["g++", "-std=c++20", f"-I{ROOT / 'include'}", "-I/usr/local/cuda/include",
           str(ROOT / "tests" / "native" / "cpp_api_test.cpp"), "-o", str(exe),
           f"-L{lib}", "-lbfpgpu", f"-L{ROOT / 'oracle'}", "-loracle", "-L/usr/local/cuda/lib64",
           "-lcudart", f"-Wl,-rpath,{lib}", f"-Wl,-rpath,{ROOT / 'oracle'}"]
    subprocess.run(cmd, check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ok" in r.stdout
