"""Build libbfpgpu.so (in-tree) for sm_100a with nvcc.

    python -m paper_1602_04716_b200.build [-j N] [--force]

Every .cu under csrc/ (the C ABI + one translation unit per instantiated
format) is compiled in parallel with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and linked into
``paper_1602_04716_b200/libbfpgpu.so``.  ptxas resource usage (-Xptxas -v)
is kept in ``_build/*.ptxas.log``.
"""
from __future__ import annotations

import argparse
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
# BFP_BUILD_TAG=<tag> builds an A/B variant into _build_<tag>/ and
# ab/<tag>/libbfpgpu.so (loaded with BFP_LIB=...; tools/gpu_ab_libs.sh)
_TAG = os.environ.get("BFP_BUILD_TAG", "")
BUILD = PKG / (f"_build_{_TAG}" if _TAG else "_build")
LIB = (PKG.parent / "ab" / _TAG / "libbfpgpu.so") if _TAG else PKG / "libbfpgpu.so"
INCLUDE = PKG.parent / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + os.environ.get("BFP_EXTRA_NVCC", "").split() + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-v", "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}",
]


GEN_DIR = CSRC / "gen"
LUTMAP = PKG.parent / "tools" / "lutmap"


def generate(verbose: bool = True) -> None:
    """LOP3-mapped covers of the compiled networks (tools/lutmap/gen.cpp):
    rebuilt when the circuits, the format list or the mapper change."""
    deps = [CSRC / "bfp_circuits.cuh", CSRC / "bfp_formats.h"] + sorted(LUTMAP.glob("*.[ch]pp"))
    outs = sorted(GEN_DIR.glob("gen_*.cuh"))
    if len(outs) >= 9 and not any(_stale(o, deps) for o in outs):
        return
    GEN_DIR.mkdir(exist_ok=True)
    BUILD.mkdir(exist_ok=True)
    exe = BUILD / "lutmap_gen"
    subprocess.run(["g++", "-O2", "-std=c++17", f"-I{CSRC}", str(LUTMAP / "gen.cpp"), "-o", str(exe)],
                   check=True)
    subprocess.run([str(exe), str(GEN_DIR)], check=True)
    if verbose:
        print(f"[bfp build] generated LOP3 covers in {GEN_DIR}", file=sys.stderr)


def sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu")) + sorted((CSRC / "inst").glob("*.cu"))


def headers() -> list[Path]:
    return (sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + sorted(INCLUDE.glob("*.h")))


def _deps(src: Path) -> list[Path]:
    d = [src] + headers()
    if src.parent.name == "inst":  # its generated cover
        d.append(GEN_DIR / src.name.replace("fmt_", "gen_").replace(".cu", ".cuh"))
    return d


def _obj(src: Path) -> Path:
    rel = src.relative_to(CSRC).with_suffix("")
    return BUILD / (str(rel).replace(os.sep, "__") + ".o")


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def _compile(src: Path, force: bool) -> tuple[Path, str]:
    obj = _obj(src)
    if not force and not _stale(obj, _deps(src)):
        return obj, "up-to-date"
    cmd = [NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = obj.with_suffix(".ptxas.log")
    log.write_text(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src.name}:\n{r.stderr[-4000:]}")
    return obj, "built"


def build(jobs: int | None = None, force: bool = False, verbose: bool = True) -> Path:
    BUILD.mkdir(exist_ok=True)
    generate(verbose)
    srcs = sources()
    jobs = jobs or max(1, min(len(srcs), os.cpu_count() or 4))
    with ThreadPoolExecutor(jobs) as ex:
        results = list(ex.map(lambda s: _compile(s, force), srcs))
    objs = [o for o, _ in results]
    if verbose:
        for (o, st), s in zip(results, srcs):
            if st != "up-to-date":
                print(f"[bfp build] {s.name}: {st}", file=sys.stderr)
    if force or _stale(LIB, objs):
        LIB.parent.mkdir(parents=True, exist_ok=True)
        cmd = [NVCC, *ARCH, "-shared", "--cudart", "static", "-o", str(LIB), *map(str, objs)]
        subprocess.run(cmd, check=True)
        if verbose:
            print(f"[bfp build] linked {LIB}", file=sys.stderr)
    if _TAG:  # A/B variants keep only their library (the GPU snapshot is size-capped)
        import shutil
        shutil.rmtree(BUILD, ignore_errors=True)
    return LIB


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", "--jobs", type=int, default=None)
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    build(a.jobs, a.force)


if __name__ == "__main__":
    main()
