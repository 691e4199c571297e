"""B200-native bitslice custom-precision floating point (arXiv 1602.04716 hot path).

The device work lives in libbfpgpu.so (C ABI: include/bfpgpu.h; CUDA sources
in csrc/).  This package is the host-side mirror of the reference operator
API (see bfp.py) plus the build script (build.py).
"""
from .bfp import (  # noqa: F401
    OP_ADD,
    OP_DIV,
    OP_MUL,
    OP_MUL_ADD,
    OP_SUB,
    arith,
    arith_f32,
    bfp_add,
    bfp_div,
    bfp_mul,
    bfp_mul_add,
    mul_add_fast_blocks,
    bfp_sub,
    bfp_vector,
    bfpraw_stride,
    chain,
    chain_f32,
    classify,
    scalar_custom,
    split,
    value_class,
    pack_bfpraw,
    unpack_bfpraw,
    decode_scalar,
    empty,
    encode_scalar,
    format_spec,
    make_spec,
    pack,
    pack_f32,
    pack_f64,
    require_same_shape,
    rounding_mode,
    subnormal_policy,
    to_u64,
    unpack,
    unpack_f32,
    unpack_f64,
    validate,
)
from ._lib import LIB_PATH, lib  # noqa: F401

# Formats with compiled networks (csrc/bfp_formats.h), each in RN/RZ x gradual/FTZ.
INSTANTIATED = [(3, 2), (4, 3), (5, 3), (5, 7), (5, 10), (6, 9), (8, 7), (8, 15), (8, 23)]
