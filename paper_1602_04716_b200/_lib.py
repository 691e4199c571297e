"""ctypes binding of libbfpgpu.so (include/bfpgpu.h).

The library is built in-tree (``python -m paper_1602_04716_b200.build``).
There is no fallback: if the shared object is missing, importing the device
entry points raises, loudly.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# BFP_LIB: an alternative build of the same library (A/B measurements only)
LIB_PATH = Path(os.environ.get("BFP_LIB") or Path(__file__).resolve().parent / "libbfpgpu.so")

# bfp_status
BFP_OK, BFP_EFORMAT, BFP_EMISMATCH, BFP_ESIZE, BFP_EUNSUPPORTED, BFP_ECUDA, BFP_EARG = range(7)
BFP_INPUTS_READY = 1  # bfp_arith_ex flags (include/bfpgpu.h)
BFP_GENERAL_NETWORK = 2


class BfpFormat(C.Structure):
    _fields_ = [
        ("exp_bits", C.c_uint32),
        ("sig_bits", C.c_uint32),
        ("rounding", C.c_uint32),
        ("subnormals", C.c_uint32),
        ("name", C.c_char_p),
    ]


_F = C.POINTER(BfpFormat)
_u32p = C.c_void_p  # device or host pointers are passed as integers

# symbol -> (restype, argtypes); every function declared in include/bfpgpu.h
SIGNATURES = {
    "bfp_status_string": (C.c_char_p, [C.c_int]),
    "bfp_last_error": (C.c_char_p, []),
    "bfp_validate": (C.c_int, [_F]),
    "bfp_same_shape": (C.c_int, [_F, _F]),
    "bfp_is_supported": (C.c_int, [_F]),
    "bfp_is_compiled": (C.c_int, [_F]),
    "bfp_plane_bytes": (C.c_size_t, [_F, C.c_size_t]),
    "bfp_enc_bytes": (C.c_size_t, [_F]),
    "bfp_pack_enc": (C.c_int, [_F, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "bfp_unpack_enc": (C.c_int, [_F, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "bfp_pack_f32": (C.c_int, [_F, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "bfp_unpack_f32": (C.c_int, [_F, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "bfp_pack_f64": (C.c_int, [_F, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "bfp_unpack_f64": (C.c_int, [_F, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "bfp_bfpraw_stride": (C.c_size_t, [_F]),
    "bfp_pack_bfpraw": (C.c_int, [_F, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]),
    "bfp_unpack_bfpraw": (C.c_int, [_F, C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]),
    "bfp_add": (C.c_int, [_F, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "bfp_sub": (C.c_int, [_F, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "bfp_mul": (C.c_int, [_F, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "bfp_div": (C.c_int, [_F, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "bfp_mul_add": (C.c_int, [_F, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                              C.c_void_p]),
    "bfp_arith": (C.c_int, [C.c_int, _F, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                            C.c_size_t, C.c_void_p]),
    "bfp_arith_ex": (C.c_int, [C.c_int, _F, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t,
                               C.c_void_p, C.c_uint]),
    "bfp_arith_f32": (C.c_int, [C.c_int, _F, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_size_t, C.c_void_p]),
    "bfp_chain": (C.c_int, [_F, C.c_char_p, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "bfp_chain_f32": (C.c_int, [_F, C.c_char_p, C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "bfp_host_ctx_create": (C.c_void_p, [C.c_size_t]),
    "bfp_host_ctx_destroy": (None, [C.c_void_p]),
    "bfp_arith_host": (C.c_int, [C.c_void_p, C.c_int, _F, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_size_t]),
    "bfp_arith_host_batch": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int), _F, C.c_void_p,
                                       C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p), C.c_size_t]),
    "bfp_pack_f32_host": (C.c_int, [C.c_void_p, _F, C.c_void_p, C.c_void_p, C.c_size_t]),
    "bfp_unpack_f32_host": (C.c_int, [C.c_void_p, _F, C.c_void_p, C.c_void_p, C.c_size_t]),
    "bfp_host_alloc": (C.c_void_p, [C.c_size_t]),
    "bfp_host_free": (None, [C.c_void_p]),
    "bfp_kernel_attrs": (C.c_int, [_F, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.POINTER(C.c_int)]),
    "bfp_mul_add_fast_blocks": (C.c_int, [_F, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p,
                                          C.c_void_p]),
    "bfp_launch_count": (C.c_uint64, []),
    "bfp_probe_lop3": (C.c_int, [C.c_int, C.POINTER(C.c_float), C.POINTER(C.c_double)]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libbfpgpu.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing -- build it with `python -m paper_1602_04716_b200.build` "
                "(there is no CPU fallback for the bitslice kernels)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class BfpError(RuntimeError):
    def __init__(self, status: int, where: str):
        L = lib()
        msg = L.bfp_status_string(status).decode()
        detail = (L.bfp_last_error() or b"").decode()
        super().__init__(f"{where}: {msg} ({detail})")
        self.status = status


def check(status: int, where: str) -> None:
    if status != BFP_OK:
        if status in (BFP_EFORMAT, BFP_EMISMATCH, BFP_ESIZE, BFP_EARG):
            # the reference throws std::invalid_argument for these
            L = lib()
            raise ValueError(f"{where}: {L.bfp_status_string(status).decode()} "
                             f"({(L.bfp_last_error() or b'').decode()})")
        raise BfpError(status, where)
