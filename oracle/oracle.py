"""oracle/oracle.py -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

ctypes views of
  * ``liboracle.so``   -- the plain-C restatement (oracle/bfp_oracle.c), and
  * ``_ref/libbfpref*.so`` -- the UNMODIFIED reference headers compiled in place
    (oracle/ref_capi.cpp + oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) import this module.  paper_1602_04716_b200/ never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_ORACLE = HERE / "liboracle.so"
REF_DIR = HERE / "_ref"

OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_MUL_ADD = 0, 1, 2, 3, 4
OPS = {"add": OP_ADD, "sub": OP_SUB, "mul": OP_MUL, "div": OP_DIV, "mul_add": OP_MUL_ADD}

_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_f32p = C.POINTER(C.c_float)
_u8p = C.POINTER(C.c_uint8)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def build(ref: bool = True) -> None:
    """Build liboracle.so (and oracle/_ref when /root/reference exists)."""
    target = "all" if ref else "oracle"
    subprocess.run(["make", "-s", "-C", str(HERE), target], check=True)


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        if not LIB_ORACLE.exists():
            build(ref=False)
        L = C.CDLL(str(LIB_ORACLE))
        L.orc_encode.restype = C.c_uint64
        L.orc_encode.argtypes = [C.c_double, C.c_uint, C.c_uint, C.c_int, C.c_int]
        L.orc_decode.restype = C.c_double
        L.orc_decode.argtypes = [C.c_uint64, C.c_uint, C.c_uint]
        L.orc_binop.restype = C.c_uint64
        L.orc_binop.argtypes = [C.c_int, C.c_uint, C.c_uint, C.c_int, C.c_int, C.c_uint64, C.c_uint64]
        L.orc_mul_add.restype = C.c_uint64
        L.orc_mul_add.argtypes = [C.c_uint, C.c_uint, C.c_int, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_pack_planes.restype = None
        L.orc_pack_planes.argtypes = [_u64p, C.c_size_t, _u32p, C.c_uint]
        L.orc_unpack_planes.restype = None
        L.orc_unpack_planes.argtypes = [_u32p, C.c_size_t, _u64p, C.c_uint]
        L.orc_binop_array.restype = None
        L.orc_binop_array.argtypes = [C.c_int, C.c_uint, C.c_uint, C.c_int, C.c_int,
                                      _u64p, _u64p, _u64p, _u64p, C.c_size_t]
        L.orc_encode_f32_array.restype = None
        L.orc_encode_f32_array.argtypes = [_f32p, C.c_size_t, _u64p, C.c_uint, C.c_uint, C.c_int, C.c_int]
        L.orc_decode_f32_array.restype = None
        L.orc_decode_f32_array.argtypes = [_u64p, C.c_size_t, _f32p, C.c_uint, C.c_uint]
        L.orc_encode_f64_array.restype = None
        L.orc_encode_f64_array.argtypes = [C.POINTER(C.c_double), C.c_size_t, _u64p, C.c_uint, C.c_uint,
                                           C.c_int, C.c_int]
        L.orc_decode_f64_array.restype = None
        L.orc_decode_f64_array.argtypes = [_u64p, C.c_size_t, C.POINTER(C.c_double), C.c_uint, C.c_uint]
        L.orc_verify.restype = C.c_uint64
        L.orc_verify.argtypes = [C.c_int, C.c_uint, C.c_uint, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                 C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int,
                                 _u64p, _u64p, _u64p]
        L.orc_verify_mul_add_pairs.restype = C.c_uint64
        L.orc_verify_mul_add_pairs.argtypes = [C.c_uint, C.c_uint, C.c_int, C.c_int, C.c_uint32, C.c_uint32,
                                               C.c_void_p, C.c_int, C.c_void_p, C.c_int, _u64p]
        L.orc_binop_exhaustive.restype = None
        L.orc_binop_exhaustive.argtypes = [C.c_int, C.c_uint, C.c_uint, C.c_int, C.c_int, _u64p]
        _orc = L
    return _orc


def _host_isa() -> set[str]:
    try:
        txt = Path("/proc/cpuinfo").read_text()
    except OSError:
        return set()
    import re
    return set(re.findall(r"\b(avx512[a-z0-9_]*|avx2|amx[a-z0-9_]*)\b", txt))


def ref_available() -> bool:
    return (REF_DIR / "libbfpref.so").exists()


def ref_lib_path() -> Path:
    """The native-tuned reference build when this host has its ISA, else x86-64-v3."""
    native = REF_DIR / "libbfpref_native.so"
    isa_file = REF_DIR / "native_isa.txt"
    if native.exists() and isa_file.exists():
        want = set(isa_file.read_text().split())
        if want <= _host_isa():
            return native
    return REF_DIR / "libbfpref.so"


def ref():
    global _ref
    if _ref is None:
        path = ref_lib_path()
        if not path.exists():
            raise FileNotFoundError(
                f"{path} missing: build it with `make -C oracle` where /root/reference exists")
        L = C.CDLL(str(path))
        L.ref_validate.restype = C.c_int
        L.ref_validate.argtypes = [C.c_uint, C.c_uint]
        L.ref_binop.restype = C.c_int
        L.ref_binop.argtypes = [C.c_int, C.c_uint, C.c_uint, C.c_int, C.c_int,
                                _u32p, _u32p, _u32p, _u32p, C.c_size_t, C.c_int, C.c_uint]
        L.ref_encode_f32.restype = C.c_int
        L.ref_encode_f32.argtypes = [_f32p, C.c_size_t, _u64p, C.c_uint, C.c_uint, C.c_int, C.c_int, C.c_int]
        L.ref_encode_f64.restype = C.c_uint64
        L.ref_encode_f64.argtypes = [C.c_double, C.c_uint, C.c_uint, C.c_int, C.c_int]
        L.ref_decode_f64.restype = C.c_double
        L.ref_decode_f64.argtypes = [C.c_uint64, C.c_uint, C.c_uint]
        L.ref_decode_f32.restype = C.c_int
        L.ref_decode_f32.argtypes = [_u64p, C.c_size_t, _f32p, C.c_uint, C.c_uint, C.c_int]
        for name in ("ref_pack_planes", "ref_pack_shipped"):
            fn = getattr(L, name)
            fn.restype = C.c_int
            fn.argtypes = [_u64p, C.c_size_t, _u32p, C.c_uint, C.c_uint]
        for name in ("ref_unpack_planes", "ref_unpack_shipped"):
            fn = getattr(L, name)
            fn.restype = C.c_int
            fn.argtypes = [_u32p, C.c_size_t, _u64p, C.c_uint, C.c_uint]
        L.ref_pack_f32_path.restype = C.c_int
        L.ref_pack_f32_path.argtypes = [_f32p, C.c_size_t, _u32p, C.c_uint, C.c_uint, C.c_int, C.c_int, C.c_int]
        L.ref_unpack_f32_path.restype = C.c_int
        L.ref_unpack_f32_path.argtypes = [_u32p, C.c_size_t, _f32p, C.c_uint, C.c_uint, C.c_int]
        L.ref_gate_count.restype = C.c_int
        L.ref_gate_count.argtypes = [C.c_int, C.c_uint, C.c_uint, C.c_int, C.c_int, _u64p]
        L.ref_bfpraw_stride.restype = C.c_size_t
        L.ref_bfpraw_stride.argtypes = [C.c_uint, C.c_uint]
        L.ref_to_bfpraw.restype = C.c_int
        L.ref_to_bfpraw.argtypes = [_u64p, C.c_size_t, _u8p, C.c_uint, C.c_uint]
        L.ref_from_bfpraw.restype = C.c_int
        L.ref_from_bfpraw.argtypes = [_u8p, C.c_size_t, _u64p, C.c_uint, C.c_uint]
        _ref = L
    return _ref


# ----------------------------------------------------------------------------
# numpy conveniences (encodings are np.uint64, planes are np.uint32)


def nblocks(n: int) -> int:
    return (n + 1023) // 1024


def pack_planes(enc: np.ndarray, nbits: int) -> np.ndarray:
    enc = np.ascontiguousarray(enc, dtype=np.uint64)
    out = np.zeros(nblocks(len(enc)) * nbits * 32, dtype=np.uint32)
    orc().orc_pack_planes(_p(enc, _u64p), len(enc), _p(out, _u32p), nbits)
    return out


def unpack_planes(planes: np.ndarray, n: int, nbits: int) -> np.ndarray:
    planes = np.ascontiguousarray(planes, dtype=np.uint32)
    out = np.zeros(n, dtype=np.uint64)
    orc().orc_unpack_planes(_p(planes, _u32p), n, _p(out, _u64p), nbits)
    return out


def binop(op: str, fmt, x: np.ndarray, y: np.ndarray, c: np.ndarray | None = None) -> np.ndarray:
    """Oracle (C restatement) z = op(x, y[, c]) over encodings."""
    e, s, rn, ftz = fmt
    x = np.ascontiguousarray(x, dtype=np.uint64)
    y = np.ascontiguousarray(y, dtype=np.uint64)
    cc = np.ascontiguousarray(c if c is not None else x, dtype=np.uint64)
    z = np.empty_like(x)
    orc().orc_binop_array(OPS[op], e, s, int(rn), int(ftz), _p(x, _u64p), _p(y, _u64p),
                          _p(cc, _u64p), _p(z, _u64p), len(x))
    return z


def encode_f32(fmt, xs: np.ndarray) -> np.ndarray:
    e, s, rn, ftz = fmt
    xs = np.ascontiguousarray(xs, dtype=np.float32)
    out = np.empty(len(xs), dtype=np.uint64)
    orc().orc_encode_f32_array(_p(xs, _f32p), len(xs), _p(out, _u64p), e, s, int(rn), int(ftz))
    return out


def decode_f32(fmt, enc: np.ndarray) -> np.ndarray:
    e, s = fmt[0], fmt[1]
    enc = np.ascontiguousarray(enc, dtype=np.uint64)
    out = np.empty(len(enc), dtype=np.float32)
    orc().orc_decode_f32_array(_p(enc, _u64p), len(enc), _p(out, _f32p), e, s)
    return out


def encode_f64(fmt, xs: np.ndarray) -> np.ndarray:
    e, s, rn, ftz = fmt
    xs = np.ascontiguousarray(xs, dtype=np.float64)
    out = np.empty(len(xs), dtype=np.uint64)
    orc().orc_encode_f64_array(xs.ctypes.data_as(C.POINTER(C.c_double)), len(xs), _p(out, _u64p),
                               e, s, int(rn), int(ftz))
    return out


def decode_f64(fmt, enc: np.ndarray) -> np.ndarray:
    enc = np.ascontiguousarray(enc, dtype=np.uint64)
    out = np.empty(len(enc), dtype=np.float64)
    orc().orc_decode_f64_array(_p(enc, _u64p), len(enc), out.ctypes.data_as(C.POINTER(C.c_double)),
                               fmt[0], fmt[1])
    return out


def ref_binop_planes(op: str, fmt, x: np.ndarray, y: np.ndarray, c: np.ndarray | None = None,
                     threads: int | None = None, lane_width: int = 1024) -> np.ndarray:
    """The reference templates themselves on plane images (lane<lane_width>)."""
    e, s, rn, ftz = fmt
    nb = 1 + e + s
    x = np.ascontiguousarray(x, dtype=np.uint32)
    y = np.ascontiguousarray(y, dtype=np.uint32)
    cc = np.ascontiguousarray(c if c is not None else x, dtype=np.uint32)
    z = np.zeros_like(x)
    blocks = len(x) // (nb * 32)
    rc = ref().ref_binop(OPS[op], e, s, int(rn), int(ftz), _p(x, _u32p), _p(y, _u32p),
                         _p(cc, _u32p), _p(z, _u32p), blocks, threads or os.cpu_count() or 1,
                         lane_width)
    if rc:
        raise ValueError(f"ref_binop rc={rc}")
    return z


def ref_binop_enc(op: str, fmt, x: np.ndarray, y: np.ndarray, c: np.ndarray | None = None,
                  threads: int | None = None) -> np.ndarray:
    nb = 1 + fmt[0] + fmt[1]
    px, py = pack_planes(x, nb), pack_planes(y, nb)
    pc = pack_planes(c, nb) if c is not None else None
    return unpack_planes(ref_binop_planes(op, fmt, px, py, pc, threads), len(x), nb)


def ref_encode_f32(fmt, xs: np.ndarray, threads: int = 1) -> np.ndarray:
    e, s, rn, ftz = fmt
    xs = np.ascontiguousarray(xs, dtype=np.float32)
    out = np.empty(len(xs), dtype=np.uint64)
    rc = ref().ref_encode_f32(_p(xs, _f32p), len(xs), _p(out, _u64p), e, s, int(rn), int(ftz), threads)
    if rc:
        raise ValueError(f"ref_encode_f32 rc={rc}")
    return out


def ref_decode_f32(fmt, enc: np.ndarray, threads: int = 1) -> np.ndarray:
    e, s = fmt[0], fmt[1]
    enc = np.ascontiguousarray(enc, dtype=np.uint64)
    out = np.empty(len(enc), dtype=np.float32)
    rc = ref().ref_decode_f32(_p(enc, _u64p), len(enc), _p(out, _f32p), e, s, threads)
    if rc:
        raise ValueError(f"ref_decode_f32 rc={rc}")
    return out


def ref_pack_planes(fmt, enc: np.ndarray, shipped: bool = False) -> np.ndarray:
    e, s = fmt[0], fmt[1]
    nb = 1 + e + s
    enc = np.ascontiguousarray(enc, dtype=np.uint64)
    out = np.zeros(nblocks(len(enc)) * nb * 32, dtype=np.uint32)
    fn = ref().ref_pack_shipped if shipped else ref().ref_pack_planes
    fn(_p(enc, _u64p), len(enc), _p(out, _u32p), e, s)
    return out


def ref_unpack_planes(fmt, planes: np.ndarray, n: int, shipped: bool = False) -> np.ndarray:
    e, s = fmt[0], fmt[1]
    planes = np.ascontiguousarray(planes, dtype=np.uint32)
    out = np.zeros(n, dtype=np.uint64)
    fn = ref().ref_unpack_shipped if shipped else ref().ref_unpack_planes
    fn(_p(planes, _u32p), n, _p(out, _u64p), e, s)
    return out


def ref_gate_count(op: str, fmt) -> dict:
    e, s, rn, ftz = fmt
    out = np.zeros(4, dtype=np.uint64)
    rc = ref().ref_gate_count(OPS[op], e, s, int(rn), int(ftz), _p(out, _u64p))
    if rc:
        raise ValueError(f"ref_gate_count rc={rc}")
    a, o, x, n = (int(v) for v in out)
    return {"and": a, "or": o, "xor": x, "not": n, "total": a + o + x + n}


VERIFY_OPS = dict(OPS, pack=5, unpack_f32=6)


def verify(op: str, fmt, a: np.ndarray, b: np.ndarray | None, c: np.ndarray | None, got: np.ndarray,
           n: int, threads: int | None = None) -> tuple[int, int, int, int]:
    """Full-size check on all host threads (orc_verify): the oracle's result of
    `op` on every element of (a, b, c) -- u32 encodings or float32 values
    through encode_scalar -- against the device output `got` (plane image, or
    float32 for op "unpack_f32").  Returns (mismatches, first index, got, want)."""
    e, s, rn, ftz = fmt
    kind = 1 if a.dtype == np.float32 else 0
    arrs = [np.ascontiguousarray(v, dtype=np.float32 if kind else np.uint32) if v is not None else None
            for v in (a, b, c)]
    got = np.ascontiguousarray(got)
    fi, fg, fw = C.c_uint64(), C.c_uint64(), C.c_uint64()
    bad = orc().orc_verify(VERIFY_OPS[op], e, s, int(rn), int(ftz), kind,
                           *[v.ctypes.data if v is not None else None for v in arrs],
                           got.ctypes.data, n, threads or os.cpu_count() or 1,
                           C.byref(fi), C.byref(fg), C.byref(fw))
    return int(bad), fi.value, fg.value, fw.value


def verify_mul_add_pairs(fmt, a0: int, na: int, cs: np.ndarray, got: list, threads: int | None = None):
    """All pairs (a0 <= a < a0 + na, every b) of a 16-bit format through
    z = add(mul(a, b), c_k) for each c_k in cs, against the device result planes
    got[k] (na * 65536 elements each).  Returns (mismatches, [index, k, got, want])."""
    e, s, rn, ftz = fmt
    assert 1 + e + s == 16
    tabs = np.stack([binop("add", fmt, np.arange(1 << 16, dtype=np.uint64),
                           np.full(1 << 16, int(c), dtype=np.uint64)) for c in cs]).astype(np.uint16)
    tabs = np.ascontiguousarray(tabs)
    gots = [np.ascontiguousarray(g, dtype=np.uint32) for g in got]
    ptrs = (C.c_void_p * len(gots))(*[g.ctypes.data for g in gots])
    info = np.zeros(4, dtype=np.uint64)
    bad = orc().orc_verify_mul_add_pairs(e, s, int(rn), int(ftz), a0, na, tabs.ctypes.data, len(cs), ptrs,
                                         threads or os.cpu_count() or 1, _p(info, _u64p))
    return int(bad), [int(v) for v in info]
