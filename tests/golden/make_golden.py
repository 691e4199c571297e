"""Regenerate the golden fixtures in tests/golden/ from the REFERENCE itself.

    python tests/golden/make_golden.py

Runs the unmodified reference headers (compiled in place by oracle/Makefile
into oracle/_ref/) on seeded operands and stores inputs + outputs:

  arith.npz   per format x mode: x, y, c and bfp_add / bfp_sub / bfp_mul /
              bfp_div / bfp_add(bfp_mul(x, y), c) results (arith.hpp:235-444)
  codec.npz   per format x mode: encode_scalar((double)f) of float32 inputs
              (format.hpp:125-188) and (float)decode_scalar of encodings
              (format.hpp:101-123)
  layout.npz  field_from_elements plane images (bitfield.hpp:33-43) of ragged
              encoding vectors, and the SHIPPED pack() output of the same
              vector (pack.hpp:41-58, Defect B) for the record

The reference cannot run on the GPU box; these fixtures carry its answers.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))
import oracle as O  # noqa: E402
from conftest import FORMATS, MODES, operands, related  # noqa: E402

N_ARITH = 2048
N_CODEC = 1024


def special_values(e: int, s: int) -> np.ndarray:
    f = lambda sg, ex, fr: (sg << (e + s)) | (ex << s) | fr  # noqa: E731
    emax = (1 << e) - 1
    vals = []
    for sg in (0, 1):
        vals += [f(sg, 0, 0), f(sg, 0, 1), f(sg, 0, (1 << s) - 1), f(sg, 1, 0), f(sg, 1, (1 << s) - 1),
                 f(sg, emax - 1, (1 << s) - 1), f(sg, emax - 1, 0), f(sg, emax, 0),
                 f(sg, emax, 1 << (s - 1)), f(sg, emax, 1), f(sg, (1 << (e - 1)) - 1, 0)]
    return np.array(vals, dtype=np.uint64)


def float_inputs(rng: np.random.Generator) -> np.ndarray:
    bits = rng.integers(0, 1 << 32, size=N_CODEC, dtype=np.uint64).astype(np.uint32)
    # magnitudes spread over the interesting binary32 exponent range
    ex = rng.integers(100, 160, size=N_CODEC // 2, dtype=np.uint32)
    bits[: N_CODEC // 2] = (bits[: N_CODEC // 2] & np.uint32(0x807FFFFF)) | (ex << np.uint32(23))
    specials = np.array([0, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000, 0xFFFFFFFF, 1, 0x80000001,
                         0x00800000, 0x3F800000, 0x477FE000, 0x477FF000, 0x477FEFFF, 0x43700000,
                         0x43780000, 0x3FC00000, 0x44000000], dtype=np.uint32)
    bits[: len(specials)] = specials
    return bits.view(np.float32)


def main() -> None:
    if not O.ref_available():
        O.build(ref=True)
    rng = np.random.default_rng(0x160204716)
    arith = {}
    codec = {}
    for (e, s) in FORMATS:
        nb = 1 + e + s
        sp = special_values(e, s)
        x = operands(e, s, N_ARITH, rng)
        y = operands(e, s, N_ARITH, rng)
        y[: N_ARITH // 8] = related(x[: N_ARITH // 8], e, s, rng)
        k = len(sp)
        x[-k * k:] = np.repeat(sp, k)[: k * k] if k * k <= N_ARITH else x[-k * k:]
        y[-k * k:] = np.tile(sp, k)[: k * k] if k * k <= N_ARITH else y[-k * k:]
        c = operands(e, s, N_ARITH, rng)
        for (rn, ftz) in MODES:
            fmt = (e, s, rn, ftz)
            key = f"{e}_{s}_{rn}_{ftz}"
            arith[f"x_{key}"] = x.astype(np.uint32)
            arith[f"y_{key}"] = y.astype(np.uint32)
            arith[f"c_{key}"] = c.astype(np.uint32)
            for op in ("add", "sub", "mul", "div", "mul_add"):
                z = O.ref_binop_enc(op, fmt, x, y, c if op == "mul_add" else None, threads=8)
                arith[f"{op}_{key}"] = z.astype(np.uint32)
            fin = float_inputs(rng)
            codec[f"f32in_{key}"] = fin.view(np.uint32)
            codec[f"enc_{key}"] = O.ref_encode_f32(fmt, fin).astype(np.uint32)
            encs = rng.integers(0, 1 << nb, size=N_CODEC, dtype=np.uint64)
            encs[: len(sp)] = sp
            codec[f"decin_{key}"] = encs.astype(np.uint32)
            codec[f"dec_{key}"] = O.ref_decode_f32(fmt, encs).view(np.uint32)
    layout = {}
    for (e, s) in [(4, 3), (5, 10), (8, 15), (8, 23)]:
        nb = 1 + e + s
        n = 2500  # ragged: 2 full blocks + a partial one
        encs = rng.integers(0, 1 << nb, size=n, dtype=np.uint64)
        layout[f"enc_{e}_{s}"] = encs.astype(np.uint32)
        layout[f"planes_{e}_{s}"] = O.ref_pack_planes((e, s), encs)
        layout[f"shipped_{e}_{s}"] = O.ref_pack_planes((e, s), encs, shipped=True)
    np.savez_compressed(HERE / "arith.npz", **arith)
    np.savez_compressed(HERE / "codec.npz", **codec)
    np.savez_compressed(HERE / "layout.npz", **layout)
    for name in ("arith.npz", "codec.npz", "layout.npz"):
        print(name, (HERE / name).stat().st_size, "bytes")


if __name__ == "__main__":
    main()
