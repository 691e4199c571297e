// integration/bfp/gpu_backend.hpp -- the B200 backend a maintainer would add
// to the REFERENCE tree, next to proj/include/bfp/arith.hpp.
//
// Reference code keeps its own types -- bfp_vector<lane<1024>> (pack.hpp:20-26)
// over bitfield<lane<1024>> (bitfield.hpp:16-28) -- and offloads the operator
// calls bfp_add / bfp_sub / bfp_mul / bfp_div (arith.hpp:235-444) and the chain
// bfp_add(bfp_mul(a, b), c) to libbfpgpu.so through the C ABI (bfpgpu.h).  The
// memory image of one bitfield<lane<1024>> IS one 1024-element block of device
// planes (lane j's 16 u64 granules = plane j's 32 u32 words), so the adapter
// is a copy: lane::u64_at / set_u64 (lane.hpp:97-110) on the host side.
//
// Two granularities: one vector per call (the reference's own call shape),
// and a batch of vectors per call (one H2D / kernel / D2H for all of them:
// the way to get throughput out of PCIe).  Errors keep the reference's
// behaviour: std::invalid_argument for mismatched specs (require_same_shape,
// arith.hpp:226-233) and bad formats; std::runtime_error for CUDA failures.
//
// Compiled against the unmodified reference headers (+ oracle/shim.hpp for the
// arith.hpp:162 defect) and checked byte for byte against the reference's own
// operators by tests/native/ref_backend_test.cpp (tests/test_ref_backend.py).
#pragma once
#include <bfp/arith.hpp>
#include <bfp/pack.hpp>
#include <bfpgpu.h>
#include <cuda_runtime_api.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace bfp {
namespace gpu_backend {

using L = lane<1024>;
using vec = bfp_vector<L>;

inline bfp_format to_c(const format_spec& f) {
  return {f.exp_bits, f.sig_bits, f.rounding == rounding_mode::rn ? 1u : 0u,
          f.subnormals == subnormal_policy::ftz ? 1u : 0u, f.name.c_str()};
}

namespace detail {
inline void cuda(cudaError_t e, const char* where) {
  if (e != cudaSuccess) throw std::runtime_error(std::string(where) + ": " + cudaGetErrorString(e));
}
inline void status(bfp_status s, const char* where) {
  if (s == BFP_OK) return;
  const std::string msg = std::string(where) + ": " + bfp_status_string(s) + " (" + bfp_last_error() + ")";
  if (s == BFP_EFORMAT || s == BFP_EMISMATCH || s == BFP_ESIZE || s == BFP_EARG) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
// block k of a host plane image <- / -> vector k's lanes
inline void put(const vec& v, std::uint64_t* blk, std::size_t nb) {
  if (v.field.size() != nb) throw std::invalid_argument("bitfield width does not match the format");
  for (std::size_t j = 0; j < nb; ++j)
    for (unsigned i = 0; i < L::u64_count; ++i) blk[j * L::u64_count + i] = v.field[j].u64_at(i);
}
inline void get(vec& v, const std::uint64_t* blk, std::size_t nb) {
  for (std::size_t j = 0; j < nb; ++j)
    for (unsigned i = 0; i < L::u64_count; ++i) v.field[j].set_u64(i, blk[j * L::u64_count + i]);
}
struct dev_buf {
  void* p = nullptr;
  explicit dev_buf(std::size_t bytes) { cuda(cudaMalloc(&p, bytes), "cudaMalloc"); }
  ~dev_buf() { cudaFree(p); }
  dev_buf(const dev_buf&) = delete;
  dev_buf& operator=(const dev_buf&) = delete;
};
}  // namespace detail

// ops[] of bfpgpu.h: 0 add, 1 sub, 2 mul, 3 div, 4 mul_add (z = x * y + c).
// xs[k], ys[k] (and cs[k]) are 1024-element vectors of one format spec.
inline std::vector<vec> arith_batch(int op, const std::vector<vec>& xs, const std::vector<vec>& ys,
                                    const std::vector<vec>* cs = nullptr) {
  if (xs.size() != ys.size() || (cs && cs->size() != xs.size()))
    throw std::invalid_argument("operand batches differ in length");
  if (op == 4 && !cs) throw std::invalid_argument("mul_add needs a third operand batch");
  std::vector<vec> out;
  if (xs.empty()) return out;
  const format_spec& spec = xs[0].spec;
  for (std::size_t k = 0; k < xs.size(); ++k) {
    ::bfp::detail::require_same_shape(spec, xs[k].spec);
    ::bfp::detail::require_same_shape(spec, ys[k].spec);
    if (cs) ::bfp::detail::require_same_shape(spec, (*cs)[k].spec);
  }
  const bfp_format f = to_c(spec);
  detail::status(bfp_validate(&f), "validate");
  const std::size_t nb = spec.total_bits(), per = nb * L::u64_count, blocks = xs.size();
  const std::size_t bytes = blocks * per * 8;
  const int nin = op == 4 ? 3 : 2;
  std::vector<std::uint64_t> h(nin * blocks * per), hz(blocks * per);
  for (std::size_t k = 0; k < blocks; ++k) {
    detail::put(xs[k], &h[k * per], nb);
    detail::put(ys[k], &h[(blocks + k) * per], nb);
    if (nin == 3) detail::put((*cs)[k], &h[(2 * blocks + k) * per], nb);
  }
  detail::dev_buf din(nin * bytes), dz(bytes);
  auto* d = static_cast<std::uint32_t*>(din.p);
  detail::cuda(cudaMemcpy(d, h.data(), nin * bytes, cudaMemcpyHostToDevice), "H2D");
  const std::size_t words = bytes / 4;
  detail::status(bfp_arith(op, &f, d, d + words, nin == 3 ? d + 2 * words : nullptr,
                           static_cast<std::uint32_t*>(dz.p), blocks * 1024, nullptr),
                 "bfp_arith");
  detail::cuda(cudaMemcpy(hz.data(), dz.p, bytes, cudaMemcpyDeviceToHost), "D2H");
  out.reserve(blocks);
  for (std::size_t k = 0; k < blocks; ++k) {
    vec z{spec, bitfield<L>(nb)};
    detail::get(z, &hz[k * per], nb);
    out.push_back(std::move(z));
  }
  return out;
}

inline vec binop(int op, const vec& x, const vec& y) {
  ::bfp::detail::require_same_shape(x.spec, y.spec);
  return std::move(arith_batch(op, {x}, {y})[0]);
}

}  // namespace gpu_backend

// The reference's operator names with a _gpu suffix (arith.hpp:235-444).
inline bfp_vector<lane<1024>> bfp_add_gpu(const bfp_vector<lane<1024>>& x, const bfp_vector<lane<1024>>& y) {
  return gpu_backend::binop(0, x, y);
}
inline bfp_vector<lane<1024>> bfp_sub_gpu(const bfp_vector<lane<1024>>& x, const bfp_vector<lane<1024>>& y) {
  return gpu_backend::binop(1, x, y);
}
inline bfp_vector<lane<1024>> bfp_mul_gpu(const bfp_vector<lane<1024>>& x, const bfp_vector<lane<1024>>& y) {
  return gpu_backend::binop(2, x, y);
}
inline bfp_vector<lane<1024>> bfp_div_gpu(const bfp_vector<lane<1024>>& x, const bfp_vector<lane<1024>>& y) {
  return gpu_backend::binop(3, x, y);
}
// bfp_add(bfp_mul(a, b), c): two roundings, one kernel
inline bfp_vector<lane<1024>> bfp_mul_add_gpu(const bfp_vector<lane<1024>>& a, const bfp_vector<lane<1024>>& b,
                                              const bfp_vector<lane<1024>>& c) {
  ::bfp::detail::require_same_shape(a.spec, b.spec);
  ::bfp::detail::require_same_shape(a.spec, c.spec);
  std::vector<bfp_vector<lane<1024>>> cs{c};
  return std::move(gpu_backend::arith_batch(4, {a}, {b}, &cs)[0]);
}

}  // namespace bfp
