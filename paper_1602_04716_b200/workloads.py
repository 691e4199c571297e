"""Seeded synthetic operands for BASELINE.json's five configurations.

No public dataset is involved; these generators stand in
with the shapes, sizes and value distributions SURVEY.md §8d specifies.
Bits come from a counter-based SplitMix64 of (seed ^ index) evaluated with
torch int64 ops, so host and device produce identical values and any shard
[lo, hi) of a vector can be generated on its own GPU.

  C1  1/4/3 add, N=2^24: float32 x = (k - 2^23) * 2^-19, k uniform in
      [0, 2^24]  (uniform in [-16, 16], exact in float32) -> encode_scalar
  C2  1/4/3 mul + sub, N=2^26: raw encodings, sign ~ B(1/2), exponent field
      uniform over all 16 codes, fraction uniform; 1% replaced by +-0
  C3  1/5/10 pack/add/mul/unpack, N=2^28: float32 normal(0, 100) clamped to
      +-65504 (Box-Muller on the hashed bits)
  C4  add + mul sweep, N=2^28: uniform finite bit patterns, exponent field in
      [0, 2^e - 2]
  C5  1/6/9 z = round(round(a*b)+c), N=2^32 total: sign uniform, unbiased
      exponent uniform in [-10, 9], uniform 23-bit mantissa (float32)
"""
from __future__ import annotations

import math

import torch

BASE_SEED = 0x160204716
SEED_A, SEED_B, SEED_C = 1, 2, 3

_M64 = (1 << 64) - 1


def _s64(v: int) -> int:
    v &= _M64
    return v - (1 << 64) if v >= (1 << 63) else v


_G = _s64(0x9E3779B97F4A7C15)
_C1 = _s64(0xBF58476D1CE4E5B9)
_C2 = _s64(0x94D049BB133111EB)


def _lsr(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def splitmix64(idx: torch.Tensor, seed: int) -> torch.Tensor:
    """SplitMix64 finaliser of (seed * golden + idx): int64 bit patterns."""
    z = idx.to(torch.int64) * _G + _s64(seed * 0x9E3779B97F4A7C15 + BASE_SEED)
    z = (z ^ _lsr(z, 30)) * _C1
    z = (z ^ _lsr(z, 27)) * _C2
    return z ^ _lsr(z, 31)


def _bits(lo: int, hi: int, seed: int, device) -> torch.Tensor:
    idx = torch.arange(lo, hi, dtype=torch.int64, device=device)
    return splitmix64(idx, seed)


def _field(h: torch.Tensor, shift: int, width: int) -> torch.Tensor:
    return _lsr(h, shift) & ((1 << width) - 1)


def c1_floats(lo: int, hi: int, seed: int, device="cuda") -> torch.Tensor:
    h = _bits(lo, hi, seed, device)
    k = _lsr(h, 8) % ((1 << 24) + 1)
    return ((k - (1 << 23)).to(torch.float32) * (2.0 ** -19)).contiguous()


def c2_encodings(lo: int, hi: int, seed: int, device="cuda") -> torch.Tensor:
    """1/4/3 encodings (uint8)."""
    h = _bits(lo, hi, seed, device)
    sign = _field(h, 0, 1)
    ex = _field(h, 1, 4)
    fr = _field(h, 5, 3)
    zero = _field(h, 16, 32) % 100 == 0
    enc = (sign << 7) | (ex << 3) | fr
    enc = torch.where(zero, sign << 7, enc)
    return enc.to(torch.uint8)


def c3_floats(lo: int, hi: int, seed: int, device="cuda") -> torch.Tensor:
    h = _bits(lo, hi, seed, device)
    u1 = (_field(h, 0, 24).to(torch.float64) + 1.0) * (2.0 ** -24)
    u2 = _field(h, 24, 24).to(torch.float64) * (2.0 ** -24)
    z = torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * math.pi * u2)
    return (z * 100.0).clamp(-65504.0, 65504.0).to(torch.float32).contiguous()


def c4_encodings(e: int, s: int, lo: int, hi: int, seed: int, device="cuda") -> torch.Tensor:
    """Uniform finite bit patterns of 1/e/s (int32 bit patterns)."""
    h = _bits(lo, hi, seed, device)
    sign = _field(h, 0, 1)
    ex = _field(h, 1, 16) % ((1 << e) - 1)
    fr = _field(h, 17, s)
    return ((sign << (e + s)) | (ex << s) | fr).to(torch.int32)


def c5_floats(lo: int, hi: int, seed: int, device="cuda") -> torch.Tensor:
    h = _bits(lo, hi, seed, device)
    sign = _field(h, 0, 1)
    ex = _field(h, 1, 16) % 20 - 10 + 127
    man = _field(h, 17, 23)
    bits = (sign << 31) | (ex << 23) | man
    return bits.to(torch.int32).view(torch.float32).contiguous()


CONFIGS = {
    "C1": {"fmt": (4, 3), "n": 1 << 24, "ops": ["add"]},
    "C2": {"fmt": (4, 3), "n": 1 << 26, "ops": ["mul", "sub"]},
    "C3": {"fmt": (5, 10), "n": 1 << 28, "ops": ["pack_f32", "add", "mul", "unpack_f32"]},
    "C4": {"fmts": [(3, 2), (5, 3), (5, 7), (8, 7), (8, 15)], "n": 1 << 28, "ops": ["add", "mul"]},
    "C5": {"fmt": (6, 9), "n": 1 << 32, "ops": ["mul_add"]},
}


def shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, 1024-element-block aligned element range of `rank`
    (GPU g owns [g*N/G, (g+1)*N/G))."""
    blocks = (n + 1023) // 1024
    b0 = blocks * rank // world
    b1 = blocks * (rank + 1) // world
    return min(n, b0 * 1024), min(n, b1 * 1024)
