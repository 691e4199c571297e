/* include/bfpgpu.h -- C ABI of the B200 bitslice custom-precision FP path.
 *
 * This is the drop-in boundary for the reference's public operator API
 * (reference: /root/reference/proj/include/bfp/, header-only C++20):
 *
 *   reference (C++ templates over lane<W>)              here (C ABI, device planes)
 *   -------------------------------------------------   -----------------------------
 *   format_spec / make_spec / validate                  bfp_format, bfp_validate
 *     format.hpp:23-73                                    (same ranges, same fields)
 *   detail::require_same_shape  arith.hpp:228-231       bfp_same_shape
 *   bfp_add   arith.hpp:235-320                         bfp_add
 *   bfp_sub   arith.hpp:322-328                         bfp_sub
 *   bfp_mul   arith.hpp:330-373                         bfp_mul
 *   bfp_div   arith.hpp:375-444                         bfp_div
 *   bfp_add(bfp_mul(a, b), c)  (two roundings)          bfp_mul_add (fused, one kernel)
 *   pack<L>(span<encoding>, spec)  pack.hpp:41-58       bfp_pack_enc   (documented layout,
 *   unpack<L>(v, count)            pack.hpp:60-76       bfp_unpack_enc  pack.hpp:13-15)
 *   encode_scalar + pack   format.hpp:125-188           bfp_pack_f32
 *   unpack + decode_scalar format.hpp:101-123           bfp_unpack_f32
 *   bfpraw_stride / to_bfpraw / from_bfpraw             bfp_bfpraw_stride, bfp_pack_bfpraw,
 *     pack.hpp:78-109                                     bfp_unpack_bfpraw
 *   encode_scalar(double) / decode_scalar -> double     bfp_pack_f64 / bfp_unpack_f64
 *   chains of bfp_add / sub / mul / div calls           bfp_chain (planes), bfp_chain_f32
 *                                                         (float32), one kernel per program
 *
 * Storage ("planes"): the memory image of an array of bitfield<lane<1024>>
 * (bitfield.hpp:10-28): element i, plane j (0 = fraction LSB, n-1 = sign) is
 * bit (i & 31) of uint32 word ((i >> 10) * n + j) * 32 + ((i >> 5) & 31),
 * n = 1 + exp_bits + sig_bits.  A vector of `count` elements occupies
 * bfp_plane_bytes(f, count) = ceil(count / 1024) * n * 128 bytes; elements
 * past `count` in the last block are zero (pack.hpp:50).
 *
 * Conventions: all pointers named d_* are device pointers owned by the
 * caller; calls are asynchronous on `stream` (a cudaStream_t, NULL = legacy
 * default stream) on the current device; no device memory is allocated by
 * the d_* entry points; errors are returned, never thrown.  Calls are
 * re-entrant.  The h_* entry points take host buffers (pinned for full
 * speed, see bfp_host_alloc) and run a chunked pipeline: inputs are copied
 * H2D in chunk order on one stream, kernels run on a second; outputs in
 * page-locked mapped memory (bfp_host_alloc) of calls up to 256 MiB are
 * written in place by the kernels over PCIe, others are staged in device
 * buffers and copied D2H in chunk order on a third stream.  The calls block
 * until the results are in host memory.
 */
#ifndef BFPGPU_H_
#define BFPGPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct bfp_format {
  uint32_t exp_bits;   /* format_spec::exp_bits, [2, 11]      (format.hpp:24,57-64) */
  uint32_t sig_bits;   /* stored fraction bits, [1, 52]       (format.hpp:25) */
  uint32_t rounding;   /* 0 = rz, 1 = rn (reference default)  (format.hpp:16,26) */
  uint32_t subnormals; /* 0 = gradual (default), 1 = ftz      (format.hpp:17,27) */
  const char* name;    /* format_spec::name; NULL == ""; compared by bfp_same_shape */
} bfp_format;

typedef enum bfp_status {
  BFP_OK = 0,
  BFP_EFORMAT = 1,      /* validate() rejects the format (format.hpp:57-64) */
  BFP_EMISMATCH = 2,    /* operands' formats differ (arith.hpp:228-231) */
  BFP_ESIZE = 3,        /* bad count / length (pack.hpp:43-44, 98-100) */
  BFP_EUNSUPPORTED = 4, /* legal format that has no compiled network */
  BFP_ECUDA = 5,        /* a CUDA call failed; see bfp_last_error() */
  BFP_EARG = 6          /* NULL pointer or bad argument */
} bfp_status;

/* ---- formats ----------------------------------------------------------- */
const char* bfp_status_string(bfp_status s);
const char* bfp_last_error(void); /* thread-local text of the last failure */
bfp_status bfp_validate(const bfp_format* f);
bfp_status bfp_same_shape(const bfp_format* a, const bfp_format* b);
/* 1 when the format can run: a compiled network (1/3/2, 1/4/3, 1/5/3, 1/5/7,
 * 1/5/10, 1/6/9, 1/8/7, 1/8/15, 1/8/23 x RN/RZ x gradual/FTZ) or, for every
 * other legal format, the NVRTC runtime backend (compiled on first use;
 * disable with BFP_JIT=0).  float32 conversions need e <= 8 and s <= 23
 * (BFP_EUNSUPPORTED otherwise); everything else covers n <= 64. */
int bfp_is_supported(const bfp_format* f);
int bfp_is_compiled(const bfp_format* f); /* 1 when an ahead-of-time network exists */
size_t bfp_plane_bytes(const bfp_format* f, size_t count);
size_t bfp_enc_bytes(const bfp_format* f); /* device encoding width: 1, 2, 4 or 8 */

/* ---- layout (device buffers) -------------------------------------------- */
/* d_enc holds `count` encodings of bfp_enc_bytes(f) bytes each,
 * little-endian, value = sign:exp:frac MSB..LSB (format.hpp:9-12). */
bfp_status bfp_pack_enc(const bfp_format* f, const void* d_enc, uint32_t* d_planes,
                        size_t count, void* stream);
bfp_status bfp_unpack_enc(const bfp_format* f, const uint32_t* d_planes, void* d_enc,
                          size_t count, void* stream);
/* float32 <-> format through encode_scalar((double)x) / (float)decode_scalar. */
bfp_status bfp_pack_f32(const bfp_format* f, const float* d_in, uint32_t* d_planes,
                        size_t count, void* stream);
bfp_status bfp_unpack_f32(const bfp_format* f, const uint32_t* d_planes, float* d_out,
                          size_t count, void* stream);

/* binary64 <-> format: encode_scalar(double) / decode_scalar -> double
 * (format.hpp:101-188) exactly -- the reference converter's own interface;
 * every legal format. */
bfp_status bfp_pack_f64(const bfp_format* f, const double* d_in, uint32_t* d_planes,
                        size_t count, void* stream);
bfp_status bfp_unpack_f64(const bfp_format* f, const uint32_t* d_planes, double* d_out,
                          size_t count, void* stream);
/* .bfpraw records (pack.hpp:78-109): count = nbytes / bfp_bfpraw_stride(f)
 * little-endian ceil(n/8)-byte encodings, back to back, no padding.
 * BFP_ESIZE when nbytes is not a multiple of the stride (pack.hpp:98-100). */
size_t bfp_bfpraw_stride(const bfp_format* f);
bfp_status bfp_pack_bfpraw(const bfp_format* f, const void* d_bytes, size_t nbytes,
                           uint32_t* d_planes, void* stream);
bfp_status bfp_unpack_bfpraw(const bfp_format* f, const uint32_t* d_planes, size_t count,
                             void* d_bytes, void* stream);

/* ---- arithmetic (device buffers, all operands in format f) --------------- */
bfp_status bfp_add(const bfp_format* f, const uint32_t* d_x, const uint32_t* d_y,
                   uint32_t* d_z, size_t count, void* stream);
bfp_status bfp_sub(const bfp_format* f, const uint32_t* d_x, const uint32_t* d_y,
                   uint32_t* d_z, size_t count, void* stream);
bfp_status bfp_mul(const bfp_format* f, const uint32_t* d_x, const uint32_t* d_y,
                   uint32_t* d_z, size_t count, void* stream);
bfp_status bfp_div(const bfp_format* f, const uint32_t* d_x, const uint32_t* d_y,
                   uint32_t* d_z, size_t count, void* stream);
/* z = round(round(a * b) + c): the reference chain bfp_add(bfp_mul(a, b), c). */
bfp_status bfp_mul_add(const bfp_format* f, const uint32_t* d_a, const uint32_t* d_b,
                       const uint32_t* d_c, uint32_t* d_z, size_t count, void* stream);
/* op: 0 add, 1 sub, 2 mul, 3 div, 4 mul_add (d_c only for 4). */
bfp_status bfp_arith(int op, const bfp_format* f, const uint32_t* d_x, const uint32_t* d_y,
                     const uint32_t* d_c, uint32_t* d_z, size_t count, void* stream);
/* bfp_arith with flags.  BFP_INPUTS_READY: the caller guarantees that no work
 * still running on `stream` writes d_x / d_y / d_c (they are resident, or
 * produced by work that has completed).  The kernel then issues its first
 * loads before waiting for the previous kernel on the stream (programmatic
 * dependent launch) and waits before its first store, so short kernels
 * overlap their load ramp with the predecessor's tail.  Results are
 * identical; only a violated guarantee (inputs written by the immediately
 * preceding kernel) could observe stale data. */
#define BFP_INPUTS_READY 1u
/* BFP_GENERAL_NETWORK: mul_add kernels carry two LOP3 covers -- the general
 * network and a smaller one valid when every element of a 1024-element block
 * lies in the "fast domain": a, b, c finite normals of moderate exponent whose
 * product can neither leave the normal range nor come near overflow, and a c
 * that is not tiny (exact bounds: csrc/bfp_circuits.cuh, mul_add_fast_domain;
 * for 1/6/9: 1 <= ea, eb < 48, 32 <= ea + eb <= 91, 16 <= ec < 48 on the
 * biased exponent fields).  Each warp tests its block and picks one cover;
 * zeros, subnormals, Inf and NaN take the general one.  Results are identical
 * either way.  This flag forces the general cover (tests, A/B measurement);
 * it is ignored by the other operations. */
#define BFP_GENERAL_NETWORK 2u
bfp_status bfp_arith_ex(int op, const bfp_format* f, const uint32_t* d_x, const uint32_t* d_y,
                        const uint32_t* d_c, uint32_t* d_z, size_t count, void* stream,
                        unsigned flags);

/* Fused float32-in / float32-out: z = (float)decode(op(encode(x), encode(y)
 * [, encode(c)])) in one kernel -- the same result as pack_f32 / op /
 * unpack_f32 without the bitslice intermediate in memory.  E <= 8, S <= 23. */
bfp_status bfp_arith_f32(int op, const bfp_format* f, const float* d_x, const float* d_y,
                         const float* d_c, float* d_z, size_t count, void* stream);

/* Fused expression: z = program(d_in[0], d_in[1], ...) over plane buffers
 * of one format, `count` elements each.  program is postfix over inputs
 * 'a', 'b', ... (d_in[0], d_in[1], ..., at most 8) and the ops + - * /, e.g.
 * "ab*c+" = (a*b)+c, "ab*cd*+" = a*b + c*d, "ab+c/" = (a+b)/c.  Every op
 * rounds to the format exactly as bfp_add / bfp_sub / bfp_mul / bfp_div do
 * (arith.hpp:235-444), so the result equals that sequence of calls; the
 * intermediates stay in registers (one kernel, HBM traffic = the inputs
 * once + the output).  Compiled for the format and program by NVRTC on first
 * use and cached (BFP_EUNSUPPORTED without NVRTC); programs that are one of
 * the ahead-of-time kernels -- "xy+", "xy-", "xy*", "xy/" and "xy*z+" (the
 * fused mul_add with its two covers) -- are sent to it.  Replaces chains of the
 * reference's bfp_* calls ("longer chains"). */
bfp_status bfp_chain(const bfp_format* f, const char* program, int n_inputs,
                     const uint32_t* const* d_in, uint32_t* d_z, size_t count, void* stream);
/* The same over float32 arrays: every input through encode_scalar, the
 * program in the format, the result through decode_scalar -- one kernel,
 * 4 B/elem per input + 4 B/elem out (E <= 8, S <= 23).  Equals
 * unpack_f32(bfp_chain(program, pack_f32(x0), pack_f32(x1), ...)). */
bfp_status bfp_chain_f32(const bfp_format* f, const char* program, int n_inputs,
                         const float* const* d_in, float* d_z, size_t count, void* stream);

/* ---- host-buffer entry points (pipelined H2D / kernel [/ D2H]) ---------- */
typedef struct bfp_host_ctx bfp_host_ctx;
bfp_host_ctx* bfp_host_ctx_create(size_t chunk_elems); /* 0 = default (2^22) */
void bfp_host_ctx_destroy(bfp_host_ctx* ctx);
/* h_x, h_y, h_c, h_z are plane images in host memory (bfp_plane_bytes each). */
bfp_status bfp_arith_host(bfp_host_ctx* ctx, int op, const bfp_format* f, const uint32_t* h_x,
                          const uint32_t* h_y, const uint32_t* h_c, uint32_t* h_z,
                          size_t count);
/* nops ops (0..4) over the same host operands; each input chunk crosses PCIe
 * once, result k goes to h_z[k]. */
bfp_status bfp_arith_host_batch(bfp_host_ctx* ctx, int nops, const int* ops, const bfp_format* f,
                                const uint32_t* h_x, const uint32_t* h_y, const uint32_t* h_c,
                                uint32_t* const* h_z, size_t count);
bfp_status bfp_pack_f32_host(bfp_host_ctx* ctx, const bfp_format* f, const float* h_in,
                             uint32_t* h_planes, size_t count);
bfp_status bfp_unpack_f32_host(bfp_host_ctx* ctx, const bfp_format* f,
                               const uint32_t* h_planes, float* h_out, size_t count);
void* bfp_host_alloc(size_t bytes); /* pinned host memory */
void bfp_host_free(void* p);

/* ---- introspection (for tests / bench) ----------------------------------- */
/* kernel: 0..4 = arith op, 10 pack_enc, 11 unpack_enc, 12 pack_f32, 13 unpack_f32,
 *         20 / 22 = fused float32 add / mul */
bfp_status bfp_kernel_attrs(const bfp_format* f, int kernel, int* regs_per_thread,
                            int* ctas_per_sm, int* threads_per_cta);
/* How many of the 1024-element blocks of bfp_mul_add(f, d_a, d_b, d_c, count)
 * run the fast-domain cover (BFP_GENERAL_NETWORK above): the kernel's own
 * predicate and warp vote, evaluated on the operands' exponent planes.
 * *d_blocks (device memory, 8 bytes) is zeroed and then written on `stream`.
 * Formats compiled at run time (NVRTC backend) return BFP_EUNSUPPORTED. */
bfp_status bfp_mul_add_fast_blocks(const bfp_format* f, const uint32_t* d_a, const uint32_t* d_b,
                                   const uint32_t* d_c, size_t count, unsigned long long* d_blocks,
                                   void* stream);
/* Number of kernel launches issued by this library in this process. */
uint64_t bfp_launch_count(void);
/* Measured LOP3 issue rate of this GPU (thread-ops/s): 8 independent chains
 * per thread on every SM; the logic leg of the roofline.  Synchronous. */
bfp_status bfp_probe_lop3(int iters, float* ms, double* lop3_per_s);

#ifdef __cplusplus
}
#endif
#endif /* BFPGPU_H_ */
