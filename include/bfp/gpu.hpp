// include/bfp/gpu.hpp -- C++ drop-in for the reference's operator API, backed
// by the B200 kernels through the C ABI (include/bfpgpu.h, libbfpgpu.so).
//
// A reference user writes
//     #include <bfp/arith.hpp>                       // /root/reference/proj/include
//     auto spec = bfp::make_spec(4, 3);
//     bfp::bfp_vector<bfp::lane<1024>> x = bfp::pack<bfp::lane<1024>>(encs, spec);
//     auto z = bfp::bfp_add(x, y);
// and switches to
//     #include <bfp/gpu.hpp>                         // this repo's include/
//     auto spec = bfp::gpu::make_spec(4, 3);
//     bfp::gpu::bfp_vector x = bfp::gpu::pack(encs, spec);   // any length
//     auto z = bfp::gpu::bfp_add(x, y);
// Same names, argument meaning and error behaviour (std::invalid_argument for
// a bad format -- format.hpp:57-64 --, for operands whose specs differ, name
// included -- arith.hpp:228-231 --, and for unpack counts past the vector).
// The lane width template parameter disappears: a bfp_vector holds any number
// of elements in device-resident planes (the memory image of an array of
// bitfield<lane<1024>>, bitfield.hpp:10-28).  pack/unpack implement the
// DOCUMENTED layout (pack.hpp:13-15); the reference's shipped transpose64 is
// anti-diagonal and is not reproduced.
//
// Link: -L<repo>/paper_1602_04716_b200 -lbfpgpu -lcudart (or compile with nvcc).
#pragma once

#include <cuda_runtime_api.h>

#include <bit>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <initializer_list>
#include <limits>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../bfpgpu.h"

namespace bfp::gpu {

enum class rounding_mode { rz, rn };           // format.hpp:16
enum class subnormal_policy { gradual, ftz };  // format.hpp:17
enum class value_class { zero, subnormal, normal, infinity, nan };  // format.hpp:19
using encoding = std::uint64_t;                // format.hpp:21

struct format_spec {  // format.hpp:23-55
  unsigned exp_bits = 0;
  unsigned sig_bits = 0;
  rounding_mode rounding = rounding_mode::rn;
  subnormal_policy subnormals = subnormal_policy::gradual;
  std::string name;

  unsigned total_bits() const { return 1 + exp_bits + sig_bits; }
  int bias() const { return (1 << (exp_bits - 1)) - 1; }
  int emax() const { return bias(); }
  int emin() const { return 1 - bias(); }
  std::uint64_t exp_field_max() const { return (1ull << exp_bits) - 1; }
  encoding frac_mask() const { return (1ull << sig_bits) - 1; }
  encoding make(unsigned sign, std::uint64_t e, std::uint64_t f) const {
    return (encoding(sign & 1u) << (exp_bits + sig_bits)) | (e << sig_bits) | f;
  }
  encoding inf(unsigned sign) const { return make(sign, exp_field_max(), 0); }
  encoding max_finite(unsigned sign) const { return make(sign, exp_field_max() - 1, frac_mask()); }
  encoding canonical_nan() const { return make(0, exp_field_max(), 1ull << (sig_bits - 1)); }
  friend bool operator==(const format_spec&, const format_spec&) = default;

  bfp_format c() const {
    return bfp_format{exp_bits, sig_bits, rounding == rounding_mode::rn ? 1u : 0u,
                      subnormals == subnormal_policy::ftz ? 1u : 0u, name.c_str()};
  }
};

// Value-level view of one element (format.hpp:75-99): host helpers.
struct scalar_custom {
  unsigned sign = 0;
  std::uint64_t biased_exp = 0;
  std::uint64_t fraction = 0;
  value_class cls = value_class::zero;
};

inline scalar_custom split(encoding enc, const format_spec& f) {
  scalar_custom r;
  r.sign = static_cast<unsigned>((enc >> (f.exp_bits + f.sig_bits)) & 1u);
  r.biased_exp = (enc >> f.sig_bits) & f.exp_field_max();
  r.fraction = enc & f.frac_mask();
  const bool top = r.biased_exp == f.exp_field_max(), low = r.biased_exp == 0;
  r.cls = top ? (r.fraction ? value_class::nan : value_class::infinity)
              : low ? (r.fraction ? value_class::subnormal : value_class::zero) : value_class::normal;
  return r;
}

inline value_class classify(encoding enc, const format_spec& f) { return split(enc, f).cls; }

inline void validate(const format_spec& f) {  // format.hpp:57-64
  if (f.exp_bits < 2 || f.exp_bits > 11) throw std::invalid_argument("exp_bits must be in [2, 11]");
  if (f.sig_bits < 1 || f.sig_bits > 52) throw std::invalid_argument("sig_bits must be in [1, 52]");
  if (f.total_bits() > 64) throw std::invalid_argument("1 + exp_bits + sig_bits must not exceed 64");
}

inline format_spec make_spec(unsigned exp_bits, unsigned sig_bits,
                             rounding_mode r = rounding_mode::rn,
                             subnormal_policy sp = subnormal_policy::gradual,
                             std::string name = {}) {  // format.hpp:66-73
  format_spec f{exp_bits, sig_bits, r, sp, std::move(name)};
  validate(f);
  return f;
}

namespace detail {
inline void check(bfp_status s, const char* where) {
  if (s == BFP_OK) return;
  const std::string msg = std::string(where) + ": " + bfp_status_string(s) + " (" + bfp_last_error() + ")";
  if (s == BFP_EFORMAT || s == BFP_EMISMATCH || s == BFP_ESIZE || s == BFP_EARG)
    throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
inline void cuda(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(where) + ": " + cudaGetErrorString(e));
}
inline void require_same_shape(const format_spec& a, const format_spec& b) {  // arith.hpp:228-231
  if (!(a == b)) throw std::invalid_argument("operands must share one format spec");
}
}  // namespace detail

// Device-resident bitslice vector (pack.hpp:20-26 with the lane width
// replaced by an element count).  Move-only; owns its planes.
class bfp_vector {
 public:
  format_spec spec;

  bfp_vector() = default;
  // Zero planes like the reference's value-initialised lanes (pack.hpp:50).
  // The fill is ordered on `stream` -- the stream the producing kernel then
  // runs on -- so it can never land after that kernel's stores, whatever the
  // stream's flags (a legacy-stream cudaMemset does not order against a
  // cudaStreamNonBlocking stream).
  bfp_vector(format_spec s, std::size_t count, cudaStream_t stream = nullptr)
      : spec(std::move(s)), count_(count) {
    const bfp_format f = spec.c();
    bytes_ = bfp_plane_bytes(&f, count_);
    if (bytes_) detail::cuda(cudaMalloc(reinterpret_cast<void**>(&planes_), bytes_), "cudaMalloc planes");
    if (bytes_) detail::cuda(cudaMemsetAsync(planes_, 0, bytes_, stream), "cudaMemsetAsync planes");
  }
  bfp_vector(const bfp_vector&) = delete;
  bfp_vector& operator=(const bfp_vector&) = delete;
  bfp_vector(bfp_vector&& o) noexcept { swap(o); }
  bfp_vector& operator=(bfp_vector&& o) noexcept {
    swap(o);
    return *this;
  }
  ~bfp_vector() {
    if (planes_) cudaFree(planes_);
  }

  std::size_t size() const { return count_; }
  std::size_t plane_bytes() const { return bytes_; }
  std::uint32_t* planes() { return planes_; }
  const std::uint32_t* planes() const { return planes_; }

 private:
  void swap(bfp_vector& o) noexcept {
    std::swap(spec, o.spec);
    std::swap(planes_, o.planes_);
    std::swap(count_, o.count_);
    std::swap(bytes_, o.bytes_);
  }
  std::uint32_t* planes_ = nullptr;
  std::size_t count_ = 0;
  std::size_t bytes_ = 0;
};

// pack.hpp:41-58 (documented layout).  Host encodings -> device planes.
inline bfp_vector pack(std::span<const encoding> encs, const format_spec& spec,
                       cudaStream_t stream = nullptr) {
  validate(spec);
  const bfp_format f = spec.c();
  const std::size_t eb = bfp_enc_bytes(&f);
  bfp_vector v(spec, encs.size(), stream);
  if (encs.empty()) return v;
  std::vector<std::uint8_t> narrow(encs.size() * eb);
  for (std::size_t i = 0; i < encs.size(); ++i) std::memcpy(&narrow[i * eb], &encs[i], eb);
  void* d = nullptr;
  detail::cuda(cudaMalloc(&d, narrow.size()), "cudaMalloc enc");
  detail::cuda(cudaMemcpyAsync(d, narrow.data(), narrow.size(), cudaMemcpyHostToDevice, stream), "H2D");
  const bfp_status s = bfp_pack_enc(&f, d, v.planes(), encs.size(), stream);
  cudaStreamSynchronize(stream);
  cudaFree(d);
  detail::check(s, "pack");
  return v;
}

// pack.hpp:60-76 (documented layout).  Device planes -> host encodings.
inline std::vector<encoding> unpack(const bfp_vector& v, std::size_t count,
                                    cudaStream_t stream = nullptr) {
  if (count > v.size()) throw std::invalid_argument("unpack: count exceeds lane width");
  const bfp_format f = v.spec.c();
  const std::size_t eb = bfp_enc_bytes(&f);
  std::vector<encoding> out(count, 0);
  if (!count) return out;
  std::vector<std::uint8_t> narrow(count * eb);
  void* d = nullptr;
  detail::cuda(cudaMalloc(&d, narrow.size()), "cudaMalloc enc");
  const bfp_status s = bfp_unpack_enc(&f, v.planes(), d, count, stream);
  detail::cuda(cudaMemcpyAsync(narrow.data(), d, narrow.size(), cudaMemcpyDeviceToHost, stream), "D2H");
  cudaStreamSynchronize(stream);
  cudaFree(d);
  detail::check(s, "unpack");
  for (std::size_t i = 0; i < count; ++i) std::memcpy(&out[i], &narrow[i * eb], eb);
  return out;
}

// float32 -> encode_scalar -> planes, for data already on the device.
inline bfp_vector pack_f32(const float* d_in, std::size_t count, const format_spec& spec,
                           cudaStream_t stream = nullptr) {
  validate(spec);
  bfp_vector v(spec, count, stream);
  const bfp_format f = spec.c();
  detail::check(bfp_pack_f32(&f, d_in, v.planes(), count, stream), "pack_f32");
  return v;
}

inline void unpack_f32(const bfp_vector& v, float* d_out, cudaStream_t stream = nullptr) {
  const bfp_format f = v.spec.c();
  detail::check(bfp_unpack_f32(&f, v.planes(), d_out, v.size(), stream), "unpack_f32");
}

// binary64 -> encode_scalar -> planes (format.hpp:125-188), device input; any
// legal format.
inline bfp_vector pack_f64(const double* d_in, std::size_t count, const format_spec& spec,
                           cudaStream_t stream = nullptr) {
  validate(spec);
  bfp_vector v(spec, count, stream);
  const bfp_format f = spec.c();
  detail::check(bfp_pack_f64(&f, d_in, v.planes(), count, stream), "pack_f64");
  return v;
}

// planes -> decode_scalar (exact binary64) into device memory.
inline void unpack_f64(const bfp_vector& v, double* d_out, cudaStream_t stream = nullptr) {
  const bfp_format f = v.spec.c();
  detail::check(bfp_unpack_f64(&f, v.planes(), d_out, v.size(), stream), "unpack_f64");
}

// .bfpraw (pack.hpp:78-109): host codec, same as the reference's ...
inline std::size_t bfpraw_stride(const format_spec& spec) { return (spec.total_bits() + 7) / 8; }

inline std::vector<std::uint8_t> to_bfpraw(std::span<const encoding> encs, const format_spec& spec) {
  const std::size_t stride = bfpraw_stride(spec);
  std::vector<std::uint8_t> out;
  out.reserve(encs.size() * stride);
  for (const encoding e : encs)
    for (std::size_t b = 0; b < stride; ++b) out.push_back(static_cast<std::uint8_t>(e >> (8 * b)));
  return out;
}

inline std::vector<encoding> from_bfpraw(std::span<const std::uint8_t> bytes, const format_spec& spec) {
  const std::size_t stride = bfpraw_stride(spec);
  if (bytes.size() % stride != 0)
    throw std::invalid_argument("bfpraw: byte count not a multiple of the encoding stride");
  std::vector<encoding> out(bytes.size() / stride);
  for (std::size_t i = 0; i < out.size(); ++i) {
    encoding e = 0;
    for (std::size_t b = 0; b < stride; ++b) e |= static_cast<encoding>(bytes[i * stride + b]) << (8 * b);
    out[i] = e;
  }
  return out;
}

// ... and straight between .bfpraw bytes and device planes.
inline bfp_vector pack_bfpraw(std::span<const std::uint8_t> bytes, const format_spec& spec,
                              cudaStream_t stream = nullptr) {
  validate(spec);
  const std::size_t stride = bfpraw_stride(spec);
  if (bytes.size() % stride != 0)
    throw std::invalid_argument("bfpraw: byte count not a multiple of the encoding stride");
  bfp_vector v(spec, bytes.size() / stride, stream);
  if (bytes.empty()) return v;
  void* d = nullptr;
  detail::cuda(cudaMalloc(&d, bytes.size()), "cudaMalloc bfpraw");
  detail::cuda(cudaMemcpyAsync(d, bytes.data(), bytes.size(), cudaMemcpyHostToDevice, stream), "H2D");
  const bfp_format f = spec.c();
  const bfp_status s = bfp_pack_bfpraw(&f, d, bytes.size(), v.planes(), stream);
  cudaStreamSynchronize(stream);
  cudaFree(d);
  detail::check(s, "pack_bfpraw");
  return v;
}

inline std::vector<std::uint8_t> unpack_bfpraw(const bfp_vector& v, cudaStream_t stream = nullptr) {
  const std::size_t nb = v.size() * bfpraw_stride(v.spec);
  std::vector<std::uint8_t> out(nb);
  if (!nb) return out;
  void* d = nullptr;
  detail::cuda(cudaMalloc(&d, nb), "cudaMalloc bfpraw");
  const bfp_format f = v.spec.c();
  const bfp_status s = bfp_unpack_bfpraw(&f, v.planes(), v.size(), d, stream);
  detail::cuda(cudaMemcpyAsync(out.data(), d, nb, cudaMemcpyDeviceToHost, stream), "D2H");
  cudaStreamSynchronize(stream);
  cudaFree(d);
  detail::check(s, "unpack_bfpraw");
  return out;
}

namespace detail {
inline bfp_vector arith(int op, const bfp_vector& x, const bfp_vector& y, const bfp_vector* c,
                        cudaStream_t stream, const char* where) {
  require_same_shape(x.spec, y.spec);
  if (c) require_same_shape(x.spec, c->spec);
  if (x.size() != y.size() || (c && c->size() != x.size()))
    throw std::invalid_argument(std::string(where) + ": operand sizes differ");
  bfp_vector z(x.spec, x.size(), stream);
  const bfp_format f = x.spec.c();
  check(bfp_arith(op, &f, x.planes(), y.planes(), c ? c->planes() : nullptr, z.planes(), x.size(),
                  stream),
        where);
  return z;
}
}  // namespace detail

inline bfp_vector bfp_add(const bfp_vector& x, const bfp_vector& y, cudaStream_t st = nullptr) {
  return detail::arith(0, x, y, nullptr, st, "bfp_add");  // arith.hpp:235-320
}
inline bfp_vector bfp_sub(const bfp_vector& x, const bfp_vector& y, cudaStream_t st = nullptr) {
  return detail::arith(1, x, y, nullptr, st, "bfp_sub");  // arith.hpp:322-328
}
inline bfp_vector bfp_mul(const bfp_vector& x, const bfp_vector& y, cudaStream_t st = nullptr) {
  return detail::arith(2, x, y, nullptr, st, "bfp_mul");  // arith.hpp:330-373
}
inline bfp_vector bfp_div(const bfp_vector& x, const bfp_vector& y, cudaStream_t st = nullptr) {
  return detail::arith(3, x, y, nullptr, st, "bfp_div");  // arith.hpp:375-444
}
// bfp_add(bfp_mul(a, b), c) in one kernel (two roundings).
inline bfp_vector bfp_mul_add(const bfp_vector& a, const bfp_vector& b, const bfp_vector& c,
                              cudaStream_t st = nullptr) {
  return detail::arith(4, a, b, &c, st, "bfp_mul_add");
}
// Fused expression (bfp_chain): postfix program over inputs 'a', 'b', ...
// (ins[0], ins[1], ...) and + - * /; e.g. chain("ab*cd*+", {&a, &b, &c, &d})
// equals bfp_add(bfp_mul(a, b), bfp_mul(c, d)) bit for bit, in one kernel.
inline bfp_vector chain(const char* program, std::initializer_list<const bfp_vector*> ins,
                        cudaStream_t st = nullptr) {
  if (ins.size() == 0 || ins.size() > 8) throw std::invalid_argument("chain: 1..8 inputs");
  const bfp_vector& x = **ins.begin();
  std::vector<const std::uint32_t*> ptrs;
  for (const bfp_vector* v : ins) {
    detail::require_same_shape(x.spec, v->spec);
    if (v->size() != x.size()) throw std::invalid_argument("chain: operand sizes differ");
    ptrs.push_back(v->planes());
  }
  bfp_vector z(x.spec, x.size(), st);
  const bfp_format f = x.spec.c();
  detail::check(bfp_chain(&f, program, int(ptrs.size()), ptrs.data(), z.planes(), x.size(), st), "chain");
  return z;
}
// bfp_chain_f32: float32 device arrays in and out (count elements each).
inline void chain_f32(const char* program, const format_spec& spec, std::initializer_list<const float*> d_in,
                      float* d_out, std::size_t count, cudaStream_t st = nullptr) {
  validate(spec);
  const std::vector<const float*> ptrs(d_in);
  const bfp_format f = spec.c();
  detail::check(bfp_chain_f32(&f, program, int(ptrs.size()), ptrs.data(), d_out, count, st), "chain_f32");
}

// Host scalar codec (format.hpp:101-188).
inline double decode_scalar(encoding enc, const format_spec& f) {
  const unsigned sign = unsigned((enc >> (f.exp_bits + f.sig_bits)) & 1u);
  const std::uint64_t be = (enc >> f.sig_bits) & f.exp_field_max();
  const std::uint64_t fr = enc & f.frac_mask();
  const double sg = sign ? -1.0 : 1.0;
  if (be == f.exp_field_max()) return fr ? std::numeric_limits<double>::quiet_NaN()
                                         : sg * std::numeric_limits<double>::infinity();
  if (be == 0) return fr ? sg * std::ldexp(double(fr), f.emin() - int(f.sig_bits)) : sg * 0.0;
  return sg * std::ldexp(double((1ull << f.sig_bits) | fr), int(be) - f.bias() - int(f.sig_bits));
}

inline encoding encode_scalar(double x, const format_spec& f) {
  const std::uint64_t bits = std::bit_cast<std::uint64_t>(x);
  const unsigned sign = unsigned(bits >> 63);
  const std::uint64_t e64 = (bits >> 52) & 0x7ff, f64 = bits & ((1ull << 52) - 1);
  if (e64 == 0x7ff) return f64 ? f.canonical_nan() : f.inf(sign);
  if (e64 == 0 && f64 == 0) return f.make(sign, 0, 0);
  const std::uint64_t sig = e64 ? ((1ull << 52) | f64) : f64;
  const int exp2 = e64 ? int(e64) - 1075 : -1074;
  const int unb = exp2 + (63 - std::countl_zero(sig));
  const int s = int(f.sig_bits);
  const int ulp = (unb >= f.emin() ? unb : f.emin()) - s;
  const int shift = ulp - exp2;
  std::uint64_t kept;
  bool guard = false, sticky = false;
  if (shift <= 0) {
    kept = sig << -shift;
  } else if (shift > 64) {
    kept = 0;
    sticky = true;
  } else {
    kept = shift == 64 ? 0 : sig >> shift;
    guard = (sig >> (shift - 1)) & 1u;
    if (shift > 1) sticky = (sig & ((1ull << (shift - 1)) - 1)) != 0;
  }
  if (f.rounding == rounding_mode::rn && guard && (sticky || (kept & 1u))) ++kept;
  int res = ulp + s;
  if (kept >= (2ull << s)) {
    kept >>= 1;
    ++res;
  }
  if (kept == 0) return f.make(sign, 0, 0);
  if (kept < (1ull << s))
    return f.subnormals == subnormal_policy::ftz ? f.make(sign, 0, 0) : f.make(sign, 0, kept);
  if (res > f.emax()) return f.rounding == rounding_mode::rn ? f.inf(sign) : f.max_finite(sign);
  return f.make(sign, std::uint64_t(res + f.bias()), kept & f.frac_mask());
}

}  // namespace bfp::gpu
