"""Host-side mirror of the reference operator API over device-resident planes.

Same names, argument meaning and error behaviour as the reference headers
(/root/reference/proj/include/bfp/), with the lane width replaced by
device-resident slice-major planes of any length:

  reference                                   here
  ------------------------------------------  --------------------------------------
  rounding_mode, subnormal_policy             rounding_mode, subnormal_policy
    format.hpp:16-17
  format_spec, validate, make_spec            format_spec, validate, make_spec
    format.hpp:23-73                            (ValueError == std::invalid_argument)
  bfp_vector<L>  pack.hpp:20-26               bfp_vector (spec, planes, count)
  pack / unpack  pack.hpp:41-76               pack / unpack  (documented layout)
  encode_scalar + pack, unpack + decode       pack_f32 / unpack_f32
  bfp_add / bfp_sub / bfp_mul / bfp_div       bfp_add / bfp_sub / bfp_mul / bfp_div
    arith.hpp:235-444                           (require_same_shape incl. name)
  bfp_add(bfp_mul(a, b), c)                   bfp_mul_add (one fused kernel)
  encode_scalar / decode_scalar               encode_scalar / decode_scalar (host)
    format.hpp:101-188

All device work goes through libbfpgpu.so (include/bfpgpu.h) on the current
torch CUDA stream.  Planes are stored as torch.int32 (bit patterns).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import struct
from dataclasses import dataclass, field

import torch

from ._lib import BfpFormat, check, lib


class rounding_mode(enum.IntEnum):  # format.hpp:16
    rz = 0
    rn = 1


class subnormal_policy(enum.IntEnum):  # format.hpp:17
    gradual = 0
    ftz = 1


OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_MUL_ADD = 0, 1, 2, 3, 4


@dataclass(frozen=True)
class format_spec:
    """format.hpp:23-55."""

    exp_bits: int = 0
    sig_bits: int = 0
    rounding: rounding_mode = rounding_mode.rn
    subnormals: subnormal_policy = subnormal_policy.gradual
    name: str = ""
    _c: BfpFormat = field(default=None, init=False, repr=False, compare=False, hash=False)

    def __post_init__(self):
        object.__setattr__(self, "_c", BfpFormat(self.exp_bits, self.sig_bits, int(self.rounding),
                                                 int(self.subnormals), self.name.encode()))

    def total_bits(self) -> int:
        return 1 + self.exp_bits + self.sig_bits

    def bias(self) -> int:
        return (1 << (self.exp_bits - 1)) - 1

    def emax(self) -> int:
        return self.bias()

    def emin(self) -> int:
        return 1 - self.bias()

    def exp_field_max(self) -> int:
        return (1 << self.exp_bits) - 1

    def sign_mask(self) -> int:
        return 1 << (self.exp_bits + self.sig_bits)

    def frac_mask(self) -> int:
        return (1 << self.sig_bits) - 1

    def make(self, sign: int, biased_exp: int, fraction: int) -> int:
        return ((sign & 1) << (self.exp_bits + self.sig_bits)) | (biased_exp << self.sig_bits) | fraction

    def inf(self, sign: int) -> int:
        return self.make(sign, self.exp_field_max(), 0)

    def max_finite(self, sign: int) -> int:
        return self.make(sign, self.exp_field_max() - 1, self.frac_mask())

    def canonical_nan(self) -> int:
        return self.make(0, self.exp_field_max(), 1 << (self.sig_bits - 1))

    @property
    def c(self) -> C.POINTER(BfpFormat):
        return C.byref(self._c)

    def plane_bytes(self, count: int) -> int:
        return ((count + 1023) // 1024) * self.total_bits() * 128

    def enc_bytes(self) -> int:
        n = self.total_bits()
        return 1 if n <= 8 else 2 if n <= 16 else 4 if n <= 32 else 8


class value_class(enum.IntEnum):  # format.hpp:19
    zero = 0
    subnormal = 1
    normal = 2
    infinity = 3
    nan = 4


@dataclass
class scalar_custom:  # format.hpp:75-81
    sign: int = 0
    biased_exp: int = 0
    fraction: int = 0
    cls: value_class = value_class.zero


def split(enc: int, f: format_spec) -> scalar_custom:
    """format.hpp:83-95: sign / biased exponent / fraction / class of one encoding."""
    sign = (enc >> (f.exp_bits + f.sig_bits)) & 1
    be = (enc >> f.sig_bits) & f.exp_field_max()
    fr = enc & f.frac_mask()
    if be == f.exp_field_max():
        cls = value_class.nan if fr else value_class.infinity
    elif be == 0:
        cls = value_class.subnormal if fr else value_class.zero
    else:
        cls = value_class.normal
    return scalar_custom(sign, be, fr, cls)


def classify(enc: int, f: format_spec) -> value_class:
    """format.hpp:97-99."""
    return split(enc, f).cls


def validate(f: format_spec) -> None:
    """format.hpp:57-64 (raises ValueError where the reference throws invalid_argument)."""
    if f.exp_bits < 2 or f.exp_bits > 11:
        raise ValueError("exp_bits must be in [2, 11]")
    if f.sig_bits < 1 or f.sig_bits > 52:
        raise ValueError("sig_bits must be in [1, 52]")
    if f.total_bits() > 64:
        raise ValueError("1 + exp_bits + sig_bits must not exceed 64")


def make_spec(exp_bits: int, sig_bits: int, rounding: rounding_mode = rounding_mode.rn,
              subnormals: subnormal_policy = subnormal_policy.gradual, name: str = "") -> format_spec:
    """format.hpp:66-73."""
    f = format_spec(exp_bits, sig_bits, rounding_mode(rounding), subnormal_policy(subnormals), name)
    validate(f)
    return f


def require_same_shape(a: format_spec, b: format_spec) -> None:
    """arith.hpp:228-231 -- compares the whole spec, name included."""
    check(lib().bfp_same_shape(a.c, b.c), "require_same_shape")


@dataclass
class bfp_vector:
    """pack.hpp:20-26: a format plus its bitslice field -- here `count` elements
    in device-resident planes (torch.int32, bfp_plane_bytes / 4 words)."""

    spec: format_spec
    planes: torch.Tensor
    count: int

    @property
    def width(self) -> int:
        return self.count

    def clone(self) -> "bfp_vector":
        return bfp_vector(self.spec, self.planes.clone(), self.count)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def empty(spec: format_spec, count: int, device=None) -> bfp_vector:
    words = spec.plane_bytes(count) // 4
    planes = torch.empty(words, dtype=torch.int32, device=device or "cuda")
    return bfp_vector(spec, planes, count)


def _enc_dtype(spec: format_spec) -> torch.dtype:
    return {1: torch.uint8, 2: torch.int16, 4: torch.int32, 8: torch.int64}[spec.enc_bytes()]  # bit patterns


def pack(encs: torch.Tensor, spec: format_spec) -> bfp_vector:
    """Encodings (sign:exp:frac, one integer per element, on the device) ->
    bitslice planes in the documented layout (pack.hpp:13-15, 41-58)."""
    validate(spec)
    encs = encs.to(_enc_dtype(spec)).contiguous()
    out = empty(spec, encs.numel(), encs.device)
    check(lib().bfp_pack_enc(spec.c, encs.data_ptr(), out.planes.data_ptr(), encs.numel(), _stream()),
          "pack")
    return out


def unpack(v: bfp_vector, count: int | None = None) -> torch.Tensor:
    """pack.hpp:60-76: planes -> `count` encodings (device tensor of the
    format's encoding width; bit patterns, see to_u64)."""
    count = v.count if count is None else count
    if count > v.count:
        raise ValueError("unpack: count exceeds vector width")
    out = torch.empty(count, dtype=_enc_dtype(v.spec), device=v.planes.device)
    check(lib().bfp_unpack_enc(v.spec.c, v.planes.data_ptr(), out.data_ptr(), count, _stream()),
          "unpack")
    return out


def bfpraw_stride(spec: format_spec) -> int:
    """pack.hpp:78-80."""
    return (spec.total_bits() + 7) // 8


def pack_bfpraw(raw: torch.Tensor, spec: format_spec) -> bfp_vector:
    """.bfpraw bytes (device uint8: little-endian ceil(n/8)-byte records,
    pack.hpp:78-109) -> planes.  ValueError when the length is not a multiple
    of the stride (from_bfpraw, pack.hpp:98-100)."""
    validate(spec)
    raw = raw.to(torch.uint8).contiguous()
    stride = bfpraw_stride(spec)
    if raw.numel() % stride:
        raise ValueError("bfpraw: byte count not a multiple of the encoding stride")
    out = empty(spec, raw.numel() // stride, raw.device)
    check(lib().bfp_pack_bfpraw(spec.c, raw.data_ptr(), raw.numel(), out.planes.data_ptr(),
                                _stream()), "pack_bfpraw")
    return out


def unpack_bfpraw(v: bfp_vector, count: int | None = None) -> torch.Tensor:
    """planes -> .bfpraw bytes (to_bfpraw, pack.hpp:86-95)."""
    count = v.count if count is None else count
    if count > v.count:
        raise ValueError("unpack_bfpraw: count exceeds vector width")
    out = torch.empty(count * bfpraw_stride(v.spec), dtype=torch.uint8, device=v.planes.device)
    check(lib().bfp_unpack_bfpraw(v.spec.c, v.planes.data_ptr(), count, out.data_ptr(), _stream()),
          "unpack_bfpraw")
    return out


def to_u64(encs: torch.Tensor, spec: format_spec) -> torch.Tensor:
    """Bit patterns of `unpack` as non-negative int64."""
    if spec.total_bits() >= 64:
        return encs.to(torch.int64)
    mask = (1 << spec.total_bits()) - 1
    return encs.to(torch.int64) & mask


def pack_f32(x: torch.Tensor, spec: format_spec) -> bfp_vector:
    """float32 -> encode_scalar((double)x) -> planes."""
    validate(spec)
    x = x.to(torch.float32).contiguous()
    out = empty(spec, x.numel(), x.device)
    check(lib().bfp_pack_f32(spec.c, x.data_ptr(), out.planes.data_ptr(), x.numel(), _stream()),
          "pack_f32")
    return out


def unpack_f32(v: bfp_vector, count: int | None = None) -> torch.Tensor:
    """planes -> (float)decode_scalar."""
    count = v.count if count is None else count
    if count > v.count:
        raise ValueError("unpack_f32: count exceeds vector width")
    out = torch.empty(count, dtype=torch.float32, device=v.planes.device)
    check(lib().bfp_unpack_f32(v.spec.c, v.planes.data_ptr(), out.data_ptr(), count, _stream()),
          "unpack_f32")
    return out


def pack_f64(x: torch.Tensor, spec: format_spec) -> bfp_vector:
    """binary64 -> encode_scalar (format.hpp:125-188, its own input type) -> planes."""
    validate(spec)
    x = x.to(torch.float64).contiguous()
    out = empty(spec, x.numel(), x.device)
    check(lib().bfp_pack_f64(spec.c, x.data_ptr(), out.planes.data_ptr(), x.numel(), _stream()),
          "pack_f64")
    return out


def unpack_f64(v: bfp_vector, count: int | None = None) -> torch.Tensor:
    """planes -> decode_scalar (format.hpp:101-123), exact binary64."""
    count = v.count if count is None else count
    if count > v.count:
        raise ValueError("unpack_f64: count exceeds vector width")
    out = torch.empty(count, dtype=torch.float64, device=v.planes.device)
    check(lib().bfp_unpack_f64(v.spec.c, v.planes.data_ptr(), out.data_ptr(), count, _stream()),
          "unpack_f64")
    return out


def _check_planes(v: bfp_vector, like: bfp_vector, what: str) -> None:
    """v must hold like.count elements of like.spec in contiguous int32 planes
    on like's device, large enough for every plane word a kernel touches: a
    short or foreign buffer is rejected before any launch writes past it."""
    require_same_shape(like.spec, v.spec)
    if v.count != like.count:
        raise ValueError(f"{what}: element count {v.count} != {like.count}")
    p = v.planes
    if p.dtype != torch.int32 or not p.is_contiguous() or not p.is_cuda:
        raise ValueError(f"{what}: planes must be a contiguous int32 CUDA tensor")
    if p.device != like.planes.device:
        raise ValueError(f"{what}: planes on {p.device}, operands on {like.planes.device}")
    if p.numel() * 4 < v.spec.plane_bytes(v.count):
        raise ValueError(f"{what}: {p.numel() * 4} plane bytes < {v.spec.plane_bytes(v.count)} needed")


def _binop(op: int, x: bfp_vector, y: bfp_vector, c: bfp_vector | None = None,
           out: bfp_vector | None = None, inputs_ready: bool = False,
           general_network: bool = False) -> bfp_vector:
    require_same_shape(x.spec, y.spec)
    if c is not None:
        require_same_shape(x.spec, c.spec)
    if x.count != y.count or (c is not None and c.count != x.count):
        raise ValueError("operands must have the same element count")
    _check_planes(x, x, "x")
    _check_planes(y, x, "y")
    if c is not None:
        _check_planes(c, x, "c")
    if out is not None:
        _check_planes(out, x, "out")
    z = out if out is not None else empty(x.spec, x.count, x.planes.device)
    check(lib().bfp_arith_ex(op, x.spec.c, x.planes.data_ptr(), y.planes.data_ptr(),
                             c.planes.data_ptr() if c is not None else None, z.planes.data_ptr(),
                             x.count, _stream(), (1 if inputs_ready else 0) | (2 if general_network else 0)),
          ("add", "sub", "mul", "div", "mul_add")[op])
    return z


def arith(op: int, x: bfp_vector, y: bfp_vector, c: bfp_vector | None = None,
          out: bfp_vector | None = None, inputs_ready: bool = False,
          general_network: bool = False) -> bfp_vector:
    """bfp_arith_ex: op 0 add, 1 sub, 2 mul, 3 div, 4 mul_add.  inputs_ready
    (BFP_INPUTS_READY) asserts that no work still running on the stream
    writes x / y / c, letting the kernel's first loads overlap the previous
    kernel's tail.  general_network (BFP_GENERAL_NETWORK) forces mul_add onto
    its general LOP3 cover (same results; include/bfpgpu.h)."""
    return _binop(op, x, y, c, out, inputs_ready, general_network)


def mul_add_fast_blocks(a: bfp_vector, b: bfp_vector, c: bfp_vector) -> int:
    """bfp_mul_add_fast_blocks: how many 1024-element blocks of bfp_mul_add(a, b, c)
    run the fast-domain cover; the rest run the general one."""
    require_same_shape(a.spec, b.spec)
    require_same_shape(a.spec, c.spec)
    if not (a.count == b.count == c.count):
        raise ValueError("operands must have the same element count")
    for v, name in ((a, "a"), (b, "b"), (c, "c")):
        _check_planes(v, a, name)
    n = torch.zeros(1, dtype=torch.int64, device=a.planes.device)
    check(lib().bfp_mul_add_fast_blocks(a.spec.c, a.planes.data_ptr(), b.planes.data_ptr(), c.planes.data_ptr(),
                                        a.count, n.data_ptr(), _stream()), "mul_add_fast_blocks")
    return int(n.item())


def bfp_add(x: bfp_vector, y: bfp_vector, out: bfp_vector | None = None) -> bfp_vector:
    """arith.hpp:235-320."""
    return _binop(OP_ADD, x, y, out=out)


def bfp_sub(x: bfp_vector, y: bfp_vector, out: bfp_vector | None = None) -> bfp_vector:
    """arith.hpp:322-328."""
    return _binop(OP_SUB, x, y, out=out)


def bfp_mul(x: bfp_vector, y: bfp_vector, out: bfp_vector | None = None) -> bfp_vector:
    """arith.hpp:330-373."""
    return _binop(OP_MUL, x, y, out=out)


def bfp_div(x: bfp_vector, y: bfp_vector, out: bfp_vector | None = None) -> bfp_vector:
    """arith.hpp:375-444."""
    return _binop(OP_DIV, x, y, out=out)


def bfp_mul_add(a: bfp_vector, b: bfp_vector, c: bfp_vector,
                out: bfp_vector | None = None) -> bfp_vector:
    """bfp_add(bfp_mul(a, b), c) -- two roundings, one kernel."""
    return _binop(OP_MUL_ADD, a, b, c, out=out)


def arith_f32(op: int, spec: format_spec, x: torch.Tensor, y: torch.Tensor,
              c: torch.Tensor | None = None) -> torch.Tensor:
    """Fused float32-in / float32-out op in `spec`:
    (float)decode(op(encode_scalar(x), encode_scalar(y)[, encode_scalar(c)]))
    in one kernel; bit-identical to unpack_f32(op(pack_f32(x), pack_f32(y)))."""
    validate(spec)
    x = x.to(torch.float32).contiguous()
    y = y.to(torch.float32).contiguous()
    if x.numel() != y.numel() or (c is not None and c.numel() != x.numel()):
        raise ValueError("operands must have the same element count")
    cc = c.to(torch.float32).contiguous() if c is not None else None
    z = torch.empty_like(x)
    check(lib().bfp_arith_f32(op, spec.c, x.data_ptr(), y.data_ptr(),
                              cc.data_ptr() if cc is not None else None, z.data_ptr(), x.numel(),
                              _stream()), "arith_f32")
    return z


def chain(program: str, *vs: bfp_vector, out: bfp_vector | None = None) -> bfp_vector:
    """Fused expression over bitslice vectors of one format (bfp_chain): postfix
    `program` over inputs 'a', 'b', ... (vs[0], vs[1], ...) and + - * /, e.g.
    chain("ab*cd*+", a, b, c, d) == bfp_add(bfp_mul(a, b), bfp_mul(c, d)) bit for
    bit, in one kernel with the intermediates in registers."""
    if not vs or len(vs) > 8:
        raise ValueError("between 1 and 8 input vectors")
    for v in vs[1:]:
        require_same_shape(vs[0].spec, v.spec)
        if v.count != vs[0].count:
            raise ValueError("operands must have the same element count")
    for k, v in enumerate(vs):
        _check_planes(v, vs[0], f"input {k}")
    if out is not None:
        _check_planes(out, vs[0], "out")
    z = out if out is not None else empty(vs[0].spec, vs[0].count, vs[0].planes.device)
    ptrs = (C.c_void_p * len(vs))(*[v.planes.data_ptr() for v in vs])
    check(lib().bfp_chain(vs[0].spec.c, program.encode(), len(vs), ptrs, z.planes.data_ptr(), vs[0].count,
                          _stream()), "chain")
    return z


def chain_f32(program: str, spec: format_spec, *xs: torch.Tensor) -> torch.Tensor:
    """bfp_chain_f32: the program over float32 tensors in `spec` (each input
    through encode_scalar, the result through decode_scalar), one kernel;
    == unpack_f32(chain(program, pack_f32(x0, spec), pack_f32(x1, spec), ...))."""
    validate(spec)
    if not xs or len(xs) > 8:
        raise ValueError("between 1 and 8 inputs")
    xs = tuple(x.to(torch.float32).contiguous() for x in xs)
    if any(x.numel() != xs[0].numel() for x in xs):
        raise ValueError("operands must have the same element count")
    z = torch.empty_like(xs[0])
    ptrs = (C.c_void_p * len(xs))(*[x.data_ptr() for x in xs])
    check(lib().bfp_chain_f32(spec.c, program.encode(), len(xs), ptrs, z.data_ptr(), xs[0].numel(), _stream()),
          "chain_f32")
    return z


# --------------------------------------------------------------------- host codec
def encode_scalar(x: float, f: format_spec) -> int:
    """format.hpp:125-188: correctly rounded binary64 -> format (host, scalar)."""
    bits = struct.unpack("<Q", struct.pack("<d", float(x)))[0]
    sign = bits >> 63
    e64 = (bits >> 52) & 0x7FF
    f64 = bits & ((1 << 52) - 1)
    if e64 == 0x7FF:
        return f.canonical_nan() if f64 else f.inf(sign)
    if e64 == 0 and f64 == 0:
        return f.make(sign, 0, 0)
    sig = ((1 << 52) | f64) if e64 else f64
    exp2 = (e64 - 1023 - 52) if e64 else (-1022 - 52)
    unb = exp2 + sig.bit_length() - 1
    s = f.sig_bits
    ulp_exp = max(unb, f.emin()) - s
    shift = ulp_exp - exp2
    guard = sticky = 0
    if shift <= 0:
        kept = sig << -shift
    else:
        kept = sig >> shift
        guard = (sig >> (shift - 1)) & 1
        sticky = int((sig & ((1 << (shift - 1)) - 1)) != 0)
    if f.rounding == rounding_mode.rn and guard and (sticky or (kept & 1)):
        kept += 1
    res_exp = ulp_exp + s
    if kept >= (2 << s):
        kept >>= 1
        res_exp += 1
    if kept == 0:
        return f.make(sign, 0, 0)
    if kept < (1 << s):
        return f.make(sign, 0, 0) if f.subnormals == subnormal_policy.ftz else f.make(sign, 0, kept)
    if res_exp > f.emax():
        return f.inf(sign) if f.rounding == rounding_mode.rn else f.max_finite(sign)
    return f.make(sign, res_exp + f.bias(), kept & f.frac_mask())


def decode_scalar(enc: int, f: format_spec) -> float:
    """format.hpp:101-123: exact value of an encoding (host, scalar)."""
    sign = (enc >> (f.exp_bits + f.sig_bits)) & 1
    be = (enc >> f.sig_bits) & f.exp_field_max()
    fr = enc & f.frac_mask()
    sg = -1.0 if sign else 1.0
    if be == f.exp_field_max():
        return math.nan if fr else sg * math.inf
    if be == 0:
        return sg * 0.0 if fr == 0 else sg * math.ldexp(float(fr), f.emin() - f.sig_bits)
    return sg * math.ldexp(float((1 << f.sig_bits) | fr), be - f.bias() - f.sig_bits)
