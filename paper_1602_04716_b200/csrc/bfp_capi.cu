// bfp_capi.cu -- the C ABI (include/bfpgpu.h): validation, dispatch to the
// compiled per-format networks, the host-buffer pipeline.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/bfpgpu.h"
#include "bfp_formats.h"
#include "bfp_kernels.cuh"

namespace bfpg {
#define DECLARE_IMPL(E_, S_) const Impl* impl_##E_##_##S_(int rn, int ftz);
BFP_FORMAT_LIST(DECLARE_IMPL)
#undef DECLARE_IMPL
const Impl* jit_impl(unsigned e, unsigned s, int rn, int ftz);  // bfp_jit.cu
bool jit_available();
cudaError_t chain_launch(unsigned e, unsigned s, int rn, int ftz, const char* prog, bool f32,
                         const void* const* in, int n_in, void* z, size_t count, cudaStream_t st);  // bfp_jit.cu
}  // namespace bfpg

using bfpg::Impl;

namespace bfpg {
int bulk_mode() {
  static const int m = [] {
    // Default off: under steady-state (graph-replayed) timing the plain loop
    // beat the bulk-copy ring on every network, logic-bound ones included
    // (its occupancy, limited by registers only, hides the LOP3 chains
    // better than the ring's smem-limited 12-16 warps/SM).
    const char* v = std::getenv("BFP_BULK");
    return v ? std::atoi(v) : 0;
  }();
  return m;
}
int grid_mult() {
  static const int m = [] {
    const char* v = std::getenv("BFP_GRID_MULT");
    const int k = v ? std::atoi(v) : 4;
    return k > 0 ? k : 1;
  }();
  return m;
}
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("BFP_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}
}  // namespace bfpg

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

bfp_status fail(bfp_status s, const char* what) {
  g_err = what;
  return s;
}

bfp_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return BFP_OK;
  if (e == cudaErrorNotSupported) return fail(BFP_EUNSUPPORTED, what);
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return BFP_ECUDA;
}

// validate(), format.hpp:57-64
bfp_status validate(const bfp_format* f) {
  if (!f) return fail(BFP_EARG, "null format");
  if (f->exp_bits < 2 || f->exp_bits > 11) return fail(BFP_EFORMAT, "exp_bits must be in [2, 11]");
  if (f->sig_bits < 1 || f->sig_bits > 52) return fail(BFP_EFORMAT, "sig_bits must be in [1, 52]");
  if (1 + f->exp_bits + f->sig_bits > 64)
    return fail(BFP_EFORMAT, "1 + exp_bits + sig_bits must not exceed 64");
  if (f->rounding > 1 || f->subnormals > 1) return fail(BFP_EFORMAT, "bad rounding / subnormal policy");
  return BFP_OK;
}

const Impl* lookup_compiled(const bfp_format* f) {
  const int rn = f->rounding == 1, ftz = f->subnormals == 1;
#define LOOKUP(E_, S_) \
  if (f->exp_bits == E_ && f->sig_bits == S_) return bfpg::impl_##E_##_##S_(rn, ftz);
  BFP_FORMAT_LIST(LOOKUP)
#undef LOOKUP
  return nullptr;
}

// Compiled network when the format is instantiated, else the NVRTC
// runtime-format backend (same templates, compiled on first use).
// BFP_FORCE_JIT=1 routes compiled formats through the runtime backend too
// (measurement / testing of the template path).
const Impl* lookup(const bfp_format* f) {
  static const bool force_jit = [] {
    const char* v = std::getenv("BFP_FORCE_JIT");
    return v && v[0] == '1';
  }();
  if (!force_jit)
    if (const Impl* c = lookup_compiled(f)) return c;
  return bfpg::jit_impl(f->exp_bits, f->sig_bits, f->rounding == 1, f->subnormals == 1);
}

bfp_status resolve(const bfp_format* f, const Impl** out) {
  const bfp_status s = validate(f);
  if (s != BFP_OK) return s;
  const Impl* impl = lookup(f);
  if (!impl) return fail(BFP_EUNSUPPORTED, "format has no compiled network and NVRTC is unavailable");
  *out = impl;
  return BFP_OK;
}

size_t nplanes(const bfp_format* f) { return 1 + f->exp_bits + f->sig_bits; }
size_t nblocks(size_t count) { return (count + 1023) / 1024; }

}  // namespace

extern "C" {

const char* bfp_status_string(bfp_status s) {
  switch (s) {
    case BFP_OK: return "ok";
    case BFP_EFORMAT: return "invalid format";
    case BFP_EMISMATCH: return "operands must share one format spec";
    case BFP_ESIZE: return "bad element count or length";
    case BFP_EUNSUPPORTED: return "format not instantiated";
    case BFP_ECUDA: return "CUDA error";
    case BFP_EARG: return "bad argument";
  }
  return "unknown";
}

const char* bfp_last_error(void) { return g_err.c_str(); }

bfp_status bfp_validate(const bfp_format* f) { return validate(f); }

// require_same_shape compares the whole format_spec including its name
// (format.hpp:54, arith.hpp:228-231).
bfp_status bfp_same_shape(const bfp_format* a, const bfp_format* b) {
  if (!a || !b) return fail(BFP_EARG, "null format");
  const char* na = a->name ? a->name : "";
  const char* nb = b->name ? b->name : "";
  if (a->exp_bits != b->exp_bits || a->sig_bits != b->sig_bits || a->rounding != b->rounding ||
      a->subnormals != b->subnormals || std::strcmp(na, nb) != 0)
    return fail(BFP_EMISMATCH, "operands must share one format spec");
  return BFP_OK;
}

int bfp_is_supported(const bfp_format* f) {
  return validate(f) == BFP_OK && (lookup_compiled(f) != nullptr || bfpg::jit_available());
}

int bfp_is_compiled(const bfp_format* f) {
  return validate(f) == BFP_OK && lookup_compiled(f) != nullptr;
}

size_t bfp_plane_bytes(const bfp_format* f, size_t count) {
  if (validate(f) != BFP_OK) return 0;
  return nblocks(count) * nplanes(f) * 128;
}

size_t bfp_enc_bytes(const bfp_format* f) {
  if (validate(f) != BFP_OK) return 0;
  const size_t n = nplanes(f);
  return n <= 8 ? 1 : (n <= 16 ? 2 : (n <= 32 ? 4 : 8));
}

bfp_status bfp_arith_ex(int op, const bfp_format* f, const uint32_t* d_x, const uint32_t* d_y,
                        const uint32_t* d_c, uint32_t* d_z, size_t count, void* stream, unsigned flags) {
  const Impl* impl = nullptr;
  const bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  if (op < 0 || op > 4) return fail(BFP_EARG, "bad op");
  if (flags & ~unsigned(BFP_INPUTS_READY | BFP_GENERAL_NETWORK)) return fail(BFP_EARG, "unknown flags");
  if (count == 0) return BFP_OK;
  if (!d_x || !d_y || !d_z || (op == 4 && !d_c)) return fail(BFP_EARG, "null operand");
  ++g_launches;
  return cuda_status(impl->arith(op, d_x, d_y, d_c, d_z, nblocks(count),
                                 static_cast<cudaStream_t>(stream), flags),
                     "arith launch");
}

bfp_status bfp_mul_add_fast_blocks(const bfp_format* f, const uint32_t* d_a, const uint32_t* d_b,
                                   const uint32_t* d_c, size_t count, unsigned long long* d_blocks,
                                   void* stream) {
  const Impl* impl = nullptr;
  const bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  if (!d_blocks || (count && (!d_a || !d_b || !d_c))) return fail(BFP_EARG, "null operand");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const cudaError_t e = cudaMemsetAsync(d_blocks, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return cuda_status(e, "fast_blocks memset");
  if (count == 0) return BFP_OK;
  const cudaError_t r = impl->fast_blocks(d_a, d_b, d_c, nblocks(count), d_blocks, st);
  if (r == cudaErrorNotSupported) return fail(BFP_EUNSUPPORTED, "no compiled network for this format");
  ++g_launches;
  return cuda_status(r, "fast_blocks launch");
}

bfp_status bfp_arith(int op, const bfp_format* f, const uint32_t* d_x, const uint32_t* d_y,
                     const uint32_t* d_c, uint32_t* d_z, size_t count, void* stream) {
  return bfp_arith_ex(op, f, d_x, d_y, d_c, d_z, count, stream, 0);
}

namespace {
bfp_status chain_common(const bfp_format* f, const char* program, int n_inputs, const void* const* d_in,
                        void* d_z, size_t count, void* stream, bool f32) {
  bfp_status s = validate(f);
  if (s != BFP_OK) return s;
  if (f32 && (f->exp_bits > 8 || f->sig_bits > 23))
    return fail(BFP_EUNSUPPORTED, "float32 codec needs exp_bits <= 8 and sig_bits <= 23");
  if (!program) return fail(BFP_EARG, "null program");
  if (n_inputs < 1 || n_inputs > 8) return fail(BFP_EARG, "n_inputs must be in [1, 8]");
  // canonical postfix: inputs 'a'.. (< n_inputs), ops + - * /, blanks ignored
  std::string prog;
  int depth = 0, ops = 0;
  bool used[8] = {};
  for (const char* c = program; *c; ++c) {
    const char ch = *c;
    if (ch == ' ' || ch == '\t') continue;
    if (ch >= 'a' && ch < 'a' + n_inputs) {
      used[ch - 'a'] = true;
      ++depth;
    } else if (ch == '+' || ch == '-' || ch == '*' || ch == '/') {
      if (depth < 2) return fail(BFP_EARG, "program: operator without two operands");
      --depth;
      ++ops;
    } else {
      return fail(BFP_EARG, "program: unexpected character (inputs a.. and + - * / only)");
    }
    prog += ch;
  }
  if (depth != 1) return fail(BFP_EARG, "program must leave exactly one value");
  if (ops > 64) return fail(BFP_EARG, "program: more than 64 operations");
  if (count == 0) return BFP_OK;
  if (!d_z || !d_in) return fail(BFP_EARG, "null operand");
  for (int i = 0; i < n_inputs; ++i)
    if (used[i] && !d_in[i]) return fail(BFP_EARG, "null operand");
  // Programs that ARE one of the ahead-of-time kernels go to it (no NVRTC; the
  // fused chain keeps its two covers): "xy<op>" and "xy*z+".
  if (!f32) {
    auto in = [&](char ch) { return static_cast<const uint32_t*>(d_in[ch - 'a']); };
    auto is_in = [](char ch) { return ch >= 'a' && ch <= 'h'; };
    if (prog.size() == 3 && is_in(prog[0]) && is_in(prog[1])) {
      const int op = prog[2] == '+' ? 0 : prog[2] == '-' ? 1 : prog[2] == '*' ? 2 : 3;
      return bfp_arith(op, f, in(prog[0]), in(prog[1]), nullptr, static_cast<uint32_t*>(d_z), count, stream);
    }
    if (prog.size() == 5 && is_in(prog[0]) && is_in(prog[1]) && prog[2] == '*' && is_in(prog[3]) && prog[4] == '+')
      return bfp_arith(4, f, in(prog[0]), in(prog[1]), in(prog[3]), static_cast<uint32_t*>(d_z), count, stream);
  }
  if (!bfpg::jit_available()) return fail(BFP_EUNSUPPORTED, "bfp_chain needs NVRTC");
  ++g_launches;
  return cuda_status(bfpg::chain_launch(f->exp_bits, f->sig_bits, f->rounding == 1, f->subnormals == 1,
                                        prog.c_str(), f32, d_in, n_inputs, d_z, count,
                                        static_cast<cudaStream_t>(stream)),
                     "chain launch");
}
}  // namespace

bfp_status bfp_chain(const bfp_format* f, const char* program, int n_inputs,
                     const uint32_t* const* d_in, uint32_t* d_z, size_t count, void* stream) {
  return chain_common(f, program, n_inputs, reinterpret_cast<const void* const*>(d_in), d_z, count, stream,
                      false);
}

bfp_status bfp_chain_f32(const bfp_format* f, const char* program, int n_inputs, const float* const* d_in,
                         float* d_z, size_t count, void* stream) {
  return chain_common(f, program, n_inputs, reinterpret_cast<const void* const*>(d_in), d_z, count, stream,
                      true);
}

bfp_status bfp_add(const bfp_format* f, const uint32_t* x, const uint32_t* y, uint32_t* z,
                   size_t count, void* stream) {
  return bfp_arith(0, f, x, y, nullptr, z, count, stream);
}
bfp_status bfp_sub(const bfp_format* f, const uint32_t* x, const uint32_t* y, uint32_t* z,
                   size_t count, void* stream) {
  return bfp_arith(1, f, x, y, nullptr, z, count, stream);
}
bfp_status bfp_mul(const bfp_format* f, const uint32_t* x, const uint32_t* y, uint32_t* z,
                   size_t count, void* stream) {
  return bfp_arith(2, f, x, y, nullptr, z, count, stream);
}
bfp_status bfp_div(const bfp_format* f, const uint32_t* x, const uint32_t* y, uint32_t* z,
                   size_t count, void* stream) {
  return bfp_arith(3, f, x, y, nullptr, z, count, stream);
}
bfp_status bfp_mul_add(const bfp_format* f, const uint32_t* a, const uint32_t* b,
                       const uint32_t* c, uint32_t* z, size_t count, void* stream) {
  return bfp_arith(4, f, a, b, c, z, count, stream);
}

bfp_status bfp_pack_enc(const bfp_format* f, const void* d_enc, uint32_t* d_planes,
                        size_t count, void* stream) {
  const Impl* impl = nullptr;
  const bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  if (count == 0) return BFP_OK;
  if (!d_enc || !d_planes) return fail(BFP_EARG, "null buffer");
  ++g_launches;
  return cuda_status(impl->pack_enc(d_enc, d_planes, count, static_cast<cudaStream_t>(stream)),
                     "pack_enc launch");
}

bfp_status bfp_unpack_enc(const bfp_format* f, const uint32_t* d_planes, void* d_enc,
                          size_t count, void* stream) {
  const Impl* impl = nullptr;
  const bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  if (count == 0) return BFP_OK;
  if (!d_enc || !d_planes) return fail(BFP_EARG, "null buffer");
  ++g_launches;
  return cuda_status(impl->unpack_enc(d_planes, d_enc, count, static_cast<cudaStream_t>(stream)),
                     "unpack_enc launch");
}

bfp_status bfp_pack_f32(const bfp_format* f, const float* d_in, uint32_t* d_planes,
                        size_t count, void* stream) {
  const Impl* impl = nullptr;
  const bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  if (count == 0) return BFP_OK;
  if (!d_in || !d_planes) return fail(BFP_EARG, "null buffer");
  ++g_launches;
  return cuda_status(impl->pack_f32(d_in, d_planes, count, static_cast<cudaStream_t>(stream)),
                     "pack_f32 launch");
}

bfp_status bfp_unpack_f32(const bfp_format* f, const uint32_t* d_planes, float* d_out,
                          size_t count, void* stream) {
  const Impl* impl = nullptr;
  const bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  if (count == 0) return BFP_OK;
  if (!d_out || !d_planes) return fail(BFP_EARG, "null buffer");
  ++g_launches;
  return cuda_status(impl->unpack_f32(d_planes, d_out, count, static_cast<cudaStream_t>(stream)),
                     "unpack_f32 launch");
}

bfp_status bfp_arith_f32(int op, const bfp_format* f, const float* d_x, const float* d_y,
                         const float* d_c, float* d_z, size_t count, void* stream) {
  const Impl* impl = nullptr;
  const bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  if (op < 0 || op > 4) return fail(BFP_EARG, "bad op");
  if (count == 0) return BFP_OK;
  if (!d_x || !d_y || !d_z || (op == 4 && !d_c)) return fail(BFP_EARG, "null operand");
  ++g_launches;
  return cuda_status(impl->arith_f32(op, d_x, d_y, d_c, d_z, count, static_cast<cudaStream_t>(stream)),
                     "arith_f32 launch");
}

// .bfpraw (pack.hpp:78-109): little-endian ceil(n/8)-byte records, no padding.
size_t bfp_bfpraw_stride(const bfp_format* f) {
  if (validate(f) != BFP_OK) return 0;
  return (nplanes(f) + 7) / 8;
}

bfp_status bfp_pack_bfpraw(const bfp_format* f, const void* d_bytes, size_t nbytes,
                           uint32_t* d_planes, void* stream) {
  const Impl* impl = nullptr;
  const bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  const size_t stride = bfp_bfpraw_stride(f);
  if (nbytes % stride != 0)
    return fail(BFP_ESIZE, "bfpraw: byte count not a multiple of the encoding stride");
  const size_t count = nbytes / stride;
  if (count == 0) return BFP_OK;
  if (!d_bytes || !d_planes) return fail(BFP_EARG, "null buffer");
  ++g_launches;
  return cuda_status(impl->pack_raw(d_bytes, d_planes, count, static_cast<cudaStream_t>(stream)),
                     "pack_bfpraw");
}

bfp_status bfp_unpack_bfpraw(const bfp_format* f, const uint32_t* d_planes, size_t count,
                             void* d_bytes, void* stream) {
  const Impl* impl = nullptr;
  const bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  if (count == 0) return BFP_OK;
  if (!d_bytes || !d_planes) return fail(BFP_EARG, "null buffer");
  ++g_launches;
  return cuda_status(impl->unpack_raw(d_planes, d_bytes, count, static_cast<cudaStream_t>(stream)),
                     "unpack_bfpraw");
}

bfp_status bfp_pack_f64(const bfp_format* f, const double* d_in, uint32_t* d_planes,
                        size_t count, void* stream) {
  const Impl* impl = nullptr;
  const bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  if (count == 0) return BFP_OK;
  if (!d_in || !d_planes) return fail(BFP_EARG, "null buffer");
  ++g_launches;
  return cuda_status(impl->pack_f64(d_in, d_planes, count, static_cast<cudaStream_t>(stream)),
                     "pack_f64 launch");
}

bfp_status bfp_unpack_f64(const bfp_format* f, const uint32_t* d_planes, double* d_out,
                          size_t count, void* stream) {
  const Impl* impl = nullptr;
  const bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  if (count == 0) return BFP_OK;
  if (!d_out || !d_planes) return fail(BFP_EARG, "null buffer");
  ++g_launches;
  return cuda_status(impl->unpack_f64(d_planes, d_out, count, static_cast<cudaStream_t>(stream)),
                     "unpack_f64 launch");
}

bfp_status bfp_kernel_attrs(const bfp_format* f, int kernel, int* regs, int* ctas_per_sm,
                            int* threads_per_cta) {
  const Impl* impl = nullptr;
  const bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  const void* k = impl->kernel(kernel);
  if (!k) return fail(BFP_EARG, "bad kernel id");
  cudaFuncAttributes a;
  cudaError_t e = cudaFuncGetAttributes(&a, k);
  if (e != cudaSuccess) return cuda_status(e, "cudaFuncGetAttributes");
  if (regs) *regs = a.numRegs;
  if (threads_per_cta) *threads_per_cta = bfpg::kThreads;
  if (ctas_per_sm) {
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, bfpg::kThreads, 0);
    if (e != cudaSuccess) return cuda_status(e, "occupancy");
    *ctas_per_sm = occ;
  }
  return BFP_OK;
}

uint64_t bfp_launch_count(void) { return g_launches.load(); }

// ------------------------------------------------------------ host pipeline
// Three streams in a fixed order: every H2D copy on s_in, every kernel on
// s_k, every D2H copy on s_out, with one event per stage and buffer slot.
// Copies of one direction therefore run strictly in chunk order (chunk 0's
// inputs arrive at the full link rate instead of sharing it with the chunks
// behind it), so the pipeline fills in one chunk time and drains in one.
struct bfp_host_ctx {
  static constexpr int kDepth = 4;   // buffer slots (chunks in flight)
  static constexpr int kMaxOut = 8;  // outputs per chunk (batched ops)
  size_t chunk_blocks = 0;
  size_t min_chunks = 8;  // a call splits into at least this many chunks
  size_t cap_bytes = 0;  // per buffer
  cudaStream_t s_in = nullptr, s_k = nullptr, s_out = nullptr;
  cudaEvent_t in_done[kDepth] = {}, k_done[kDepth] = {}, out_done[kDepth] = {};
  void* in[kDepth][3] = {};
  void* out[kDepth][kMaxOut] = {};
  int dev = 0;
  // lazily allocated output buffer j of slot i
  void* out_buf(int i, int j) {
    if (!out[i][j] && cudaMalloc(&out[i][j], cap_bytes) != cudaSuccess) out[i][j] = nullptr;
    return out[i][j];
  }
};

bfp_host_ctx* bfp_host_ctx_create(size_t chunk_elems) {
  if (!chunk_elems) chunk_elems = size_t(1) << 22;
  auto* c = new bfp_host_ctx;
  c->chunk_blocks = (chunk_elems + 1023) / 1024;
  if (const char* v = getenv("BFP_HOST_MIN_CHUNKS")) {  // tuning knob
    const long m = atol(v);
    if (m >= 1) c->min_chunks = size_t(m);
  }
  // 32 planes or float32 elements per chunk block; wider formats (up to 64
  // planes) run proportionally fewer blocks per chunk (chunk_for)
  c->cap_bytes = c->chunk_blocks * 1024 * 4;
  cudaGetDevice(&c->dev);
  for (cudaStream_t* st : {&c->s_in, &c->s_k, &c->s_out})
    if (cudaStreamCreateWithFlags(st, cudaStreamNonBlocking) != cudaSuccess) goto bad;
  for (int i = 0; i < bfp_host_ctx::kDepth; ++i) {
    for (cudaEvent_t* ev : {&c->in_done[i], &c->k_done[i], &c->out_done[i]})
      if (cudaEventCreateWithFlags(ev, cudaEventDisableTiming) != cudaSuccess) goto bad;
    for (int k = 0; k < 3; ++k)
      if (cudaMalloc(&c->in[i][k], c->cap_bytes) != cudaSuccess) goto bad;
    if (!c->out_buf(i, 0)) goto bad;
  }
  return c;
bad:
  g_err = "bfp_host_ctx_create: allocation failed";
  bfp_host_ctx_destroy(c);
  return nullptr;
}

void bfp_host_ctx_destroy(bfp_host_ctx* c) {
  if (!c) return;
  for (cudaStream_t st : {c->s_in, c->s_k, c->s_out})
    if (st) cudaStreamSynchronize(st);
  for (int i = 0; i < bfp_host_ctx::kDepth; ++i) {
    for (int k = 0; k < 3; ++k)
      if (c->in[i][k]) cudaFree(c->in[i][k]);
    for (int k = 0; k < bfp_host_ctx::kMaxOut; ++k)
      if (c->out[i][k]) cudaFree(c->out[i][k]);
    for (cudaEvent_t ev : {c->in_done[i], c->k_done[i], c->out_done[i]})
      if (ev) cudaEventDestroy(ev);
  }
  for (cudaStream_t st : {c->s_in, c->s_k, c->s_out})
    if (st) cudaStreamDestroy(st);
  delete c;
}

}  // extern "C"

namespace {

// Chunk size of one call: the context's chunk, but small enough that the call
// splits into >= min_chunks chunks (fill and drain cost one chunk each), and
// never below 512 blocks (2^19 elements) so per-copy overhead stays small.
// block_bytes = the widest per-block footprint of any staged buffer of the
// call (planes: n * 128 B, up to 8 KiB for 64-plane formats; float32: 4 KiB):
// a chunk never holds more than the slot buffers' cap_bytes.
size_t chunk_for(const bfp_host_ctx* c, size_t blocks, size_t block_bytes) {
  constexpr size_t kMinBlocks = 512;
  const size_t split = (blocks + c->min_chunks - 1) / c->min_chunks;
  size_t cb = split < kMinBlocks ? kMinBlocks : split;
  if (cb > c->chunk_blocks) cb = c->chunk_blocks;
  const size_t fit = c->cap_bytes / (block_bytes ? block_bytes : 1);
  if (cb > fit) cb = fit;
  return cb ? cb : 1;
}

struct Chunk {
  int slot;
  size_t b0, nb;  // first block, blocks
  size_t e0, ne;  // first element, elements
};

// Device-accessible alias of a host address when it lies in page-locked,
// mapped memory (bfp_host_alloc / cudaMallocHost / cudaHostRegister), else null.
void* mapped_alias(void* h) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();  // pageable memory on older runtimes reports an error
    return nullptr;
  }
  if (a.type != cudaMemoryTypeHost || !a.devicePointer || !a.hostPointer) return nullptr;
  return static_cast<char*>(a.devicePointer) + (static_cast<char*>(h) - static_cast<char*>(a.hostPointer));
}

// Generic pipeline over the chunks of `count` elements.
//   in_bytes(ch, a, &src, &bytes)  -> host source / size of input a
//   out_bytes(ch, q, &dst, &bytes) -> host destination / size of output q
//   body(ch, outs, st)             -> kernel launches on st, reading the slot's
//                                     input buffers, writing outs[q]
// Inputs are copied H2D in chunk order on s_in.  Outputs in page-locked
// mapped host memory of calls up to kDirectMaxBytes are written by the
// kernels in place (the stores cross PCIe as the kernel runs: no D2H copy
// stage); otherwise they land in the slot's device buffers and are copied
// D2H in chunk order on s_out.
template <typename In, typename Body, typename Out>
bfp_status host_pipeline(bfp_host_ctx* c, size_t count, size_t block_bytes, int n_in, int n_out,
                         In in_bytes, Body body, Out out_bytes) {
  if (!c) return fail(BFP_EARG, "null host context");
  if (count == 0) return BFP_OK;
  if (block_bytes > c->cap_bytes) return fail(BFP_ESIZE, "host ctx: chunk buffers smaller than one block");
  // In-place writes cross PCIe at ~52.6 GB/s against ~57 GB/s for a D2H copy
  // (B200 box, tools/pcie_probe.py) but drop the copy stage's per-chunk
  // event hops and its drain: they win on calls whose output is small next
  // to that fixed cost (2^24 fp8 add +10%, 2^26 mul+sub +2.5%) and lose on
  // large ones (2^28 float32 unpack -6%), hence the size cut-off.
  constexpr size_t kDirectMaxBytes = size_t(256) << 20;
  bool direct = true;
  {
    const Chunk ch0{0, 0, 1, 0, 1};
    const Chunk all{0, 0, nblocks(count), 0, count};
    size_t total = 0;
    for (int q = 0; q < n_out && direct; ++q) {
      void* dst;
      size_t bytes;
      out_bytes(ch0, q, &dst, &bytes);
      direct = mapped_alias(dst) != nullptr;
      out_bytes(all, q, &dst, &bytes);
      total += bytes;
    }
    direct = direct && total <= kDirectMaxBytes;
  }
  if (!direct)
    for (int q = 0; q < n_out; ++q)
      for (int i = 0; i < bfp_host_ctx::kDepth; ++i)
        if (!c->out_buf(i, q)) return fail(BFP_ECUDA, "host ctx: output buffer allocation failed");
  const size_t blocks = nblocks(count);
  const size_t cb = chunk_for(c, blocks, block_bytes);
  bool used[bfp_host_ctx::kDepth] = {};
  cudaError_t e = cudaSuccess;
  for (size_t b0 = 0, k = 0; b0 < blocks; b0 += cb, ++k) {
    Chunk ch;
    ch.slot = int(k % bfp_host_ctx::kDepth);
    ch.b0 = b0;
    ch.nb = (blocks - b0 < cb) ? blocks - b0 : cb;
    ch.e0 = b0 * 1024;
    ch.ne = (count - ch.e0 < ch.nb * 1024) ? count - ch.e0 : ch.nb * 1024;
    const int i = ch.slot;
    // inputs of slot i are free once its previous kernels are done
    if (used[i] && (e = cudaStreamWaitEvent(c->s_in, c->k_done[i], 0)) != cudaSuccess)
      return cuda_status(e, "wait");
    for (int a = 0; a < n_in; ++a) {
      const void* src;
      size_t bytes;
      in_bytes(ch, a, &src, &bytes);
      if ((e = cudaMemcpyAsync(c->in[i][a], src, bytes, cudaMemcpyHostToDevice, c->s_in)) !=
          cudaSuccess)
        return cuda_status(e, "H2D");
    }
    if ((e = cudaEventRecord(c->in_done[i], c->s_in)) != cudaSuccess) return cuda_status(e, "record");
    if ((e = cudaStreamWaitEvent(c->s_k, c->in_done[i], 0)) != cudaSuccess) return cuda_status(e, "wait");
    void* outs[bfp_host_ctx::kMaxOut];
    for (int q = 0; q < n_out; ++q) {
      if (direct) {
        void* dst;
        size_t bytes;
        out_bytes(ch, q, &dst, &bytes);
        outs[q] = mapped_alias(dst);
      } else {
        outs[q] = c->out[i][q];
      }
    }
    // outputs of slot i are free once its previous D2H copies are done
    if (!direct && used[i] && (e = cudaStreamWaitEvent(c->s_k, c->out_done[i], 0)) != cudaSuccess)
      return cuda_status(e, "wait");
    const bfp_status s = body(ch, outs, c->s_k);
    if (s != BFP_OK) return s;
    if ((e = cudaEventRecord(c->k_done[i], c->s_k)) != cudaSuccess) return cuda_status(e, "record");
    if (!direct) {
      if ((e = cudaStreamWaitEvent(c->s_out, c->k_done[i], 0)) != cudaSuccess)
        return cuda_status(e, "wait");
      for (int q = 0; q < n_out; ++q) {
        void* dst;
        size_t bytes;
        out_bytes(ch, q, &dst, &bytes);
        if ((e = cudaMemcpyAsync(dst, c->out[i][q], bytes, cudaMemcpyDeviceToHost, c->s_out)) !=
            cudaSuccess)
          return cuda_status(e, "D2H");
      }
      if ((e = cudaEventRecord(c->out_done[i], c->s_out)) != cudaSuccess)
        return cuda_status(e, "record");
    }
    used[i] = true;
  }
  for (cudaStream_t st : {c->s_in, c->s_k, c->s_out})
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_status(e, "sync");
  return BFP_OK;
}

}  // namespace

extern "C" {

bfp_status bfp_arith_host(bfp_host_ctx* c, int op, const bfp_format* f, const uint32_t* h_x,
                          const uint32_t* h_y, const uint32_t* h_c, uint32_t* h_z,
                          size_t count) {
  const int ops[1] = {op};
  uint32_t* outs[1] = {h_z};
  return bfp_arith_host_batch(c, 1, ops, f, h_x, h_y, h_c, outs, count);
}

// Several ops over the SAME host operands: each chunk's inputs cross PCIe
// once, every op runs on them, each op's result comes back (a caller doing
// z1 = x * y, z2 = x - y on host vectors).
bfp_status bfp_arith_host_batch(bfp_host_ctx* c, int nops, const int* ops, const bfp_format* f,
                                const uint32_t* h_x, const uint32_t* h_y, const uint32_t* h_c,
                                uint32_t* const* h_z, size_t count) {
  const Impl* impl = nullptr;
  bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  if (!c) return fail(BFP_EARG, "null host context");
  if (nops <= 0 || nops > bfp_host_ctx::kMaxOut || !ops || !h_z) return fail(BFP_EARG, "bad op list");
  bool need_c = false;
  for (int k = 0; k < nops; ++k) {
    if (ops[k] < 0 || ops[k] > 4) return fail(BFP_EARG, "bad op");
    if (!h_z[k]) return fail(BFP_EARG, "null output");
    need_c |= ops[k] == 4;
  }
  if (!h_x || !h_y || (need_c && !h_c)) return fail(BFP_EARG, "null operand");
  const size_t stride = nplanes(f) * 128;
  const void* ins[3] = {h_x, h_y, h_c};
  return host_pipeline(
      c, count, stride, need_c ? 3 : 2, nops,
      [&](const Chunk& ch, int a, const void** src, size_t* bytes) {
        *src = static_cast<const char*>(ins[a]) + ch.b0 * stride;
        *bytes = ch.nb * stride;
      },
      [&](const Chunk& ch, void* const* outs, cudaStream_t st) {
        const int i = ch.slot;
        for (int q = 0; q < nops; ++q) {
          ++g_launches;
          const bfp_status r = cuda_status(
              impl->arith(ops[q], static_cast<const uint32_t*>(c->in[i][0]),
                          static_cast<const uint32_t*>(c->in[i][1]),
                          static_cast<const uint32_t*>(c->in[i][2]),
                          static_cast<uint32_t*>(outs[q]), ch.nb, st),
              "arith launch");
          if (r != BFP_OK) return r;
        }
        return BFP_OK;
      },
      [&](const Chunk& ch, int q, void** dst, size_t* bytes) {
        *dst = reinterpret_cast<char*>(h_z[q]) + ch.b0 * stride;
        *bytes = ch.nb * stride;
      });
}

bfp_status bfp_pack_f32_host(bfp_host_ctx* c, const bfp_format* f, const float* h_in,
                             uint32_t* h_planes, size_t count) {
  const Impl* impl = nullptr;
  bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  if (!h_in || !h_planes) return fail(BFP_EARG, "null buffer");
  const size_t stride = nplanes(f) * 128;
  return host_pipeline(
      c, count, stride > 4096 ? stride : 4096, 1, 1,
      [&](const Chunk& ch, int, const void** src, size_t* bytes) {
        *src = h_in + ch.e0;
        *bytes = ch.ne * 4;
      },
      [&](const Chunk& ch, void* const* outs, cudaStream_t st) {
        ++g_launches;
        return cuda_status(impl->pack_f32(static_cast<const float*>(c->in[ch.slot][0]),
                                          static_cast<uint32_t*>(outs[0]), ch.ne, st),
                           "pack_f32 launch");
      },
      [&](const Chunk& ch, int, void** dst, size_t* bytes) {
        *dst = reinterpret_cast<char*>(h_planes) + ch.b0 * stride;
        *bytes = ch.nb * stride;
      });
}

bfp_status bfp_unpack_f32_host(bfp_host_ctx* c, const bfp_format* f, const uint32_t* h_planes,
                               float* h_out, size_t count) {
  const Impl* impl = nullptr;
  bfp_status s = resolve(f, &impl);
  if (s != BFP_OK) return s;
  if (!h_out || !h_planes) return fail(BFP_EARG, "null buffer");
  const size_t stride = nplanes(f) * 128;
  return host_pipeline(
      c, count, stride > 4096 ? stride : 4096, 1, 1,
      [&](const Chunk& ch, int, const void** src, size_t* bytes) {
        *src = reinterpret_cast<const char*>(h_planes) + ch.b0 * stride;
        *bytes = ch.nb * stride;
      },
      [&](const Chunk& ch, void* const* outs, cudaStream_t st) {
        ++g_launches;
        return cuda_status(impl->unpack_f32(static_cast<const uint32_t*>(c->in[ch.slot][0]),
                                            static_cast<float*>(outs[0]), ch.ne, st),
                           "unpack_f32 launch");
      },
      [&](const Chunk& ch, int, void** dst, size_t* bytes) {
        *dst = h_out + ch.e0;
        *bytes = ch.ne * 4;
      });
}

void* bfp_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaMallocHost(&p, bytes) != cudaSuccess) {
    g_err = "cudaMallocHost failed";
    return nullptr;
  }
  return p;
}

void bfp_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

}  // extern "C"
