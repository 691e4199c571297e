// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" harness around the UNMODIFIED reference headers, compiled
// in place from /root/reference/proj/include (recipe: oracle/Makefile, output
// oracle/_ref/libbfpref*.so, git-ignored).  It is the "reference" oracle:
// tests use it to pin the C restatement (oracle/bfp_oracle.c) and the GPU
// kernels, tests/golden/make_golden.py uses it to write fixtures, and
// bench.py --impl reference / cpu_baseline times it on the host cores.
// Nothing in paper_1602_04716_b200/ links or loads it.
//
// Memory image: an array of bitfield<lane<1024>> in the order
// [block][plane][16 x u64] is byte-identical to the device plane layout
// (element i, plane j -> u32 word ((i>>10)*n + j)*32 + ((i>>5)&31), bit i&31),
// SURVEY.md §8a row 3.  Operands are moved in and out of lanes with
// lane::set_u64 / u64_at (lane.hpp:96-113), which is pure data movement.
//
// The shipped pack/unpack (pack.hpp:41-76) are wrong (anti-diagonal
// transpose); parity uses field_from_elements / element_of
// (bitfield.hpp:33-52).  ref_pack_shipped/ref_unpack_shipped expose the
// shipped ones only so tests can record the defect and bench can time them.

#include <bfp/arith.hpp>
#include <bfp/bitfield.hpp>
#include <bfp/circuits.hpp>
#include <bfp/format.hpp>
#include <bfp/lane.hpp>
#include <bfp/pack.hpp>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <thread>
#include <vector>

using namespace bfp;

namespace {

enum { OP_ADD = 0, OP_SUB = 1, OP_MUL = 2, OP_DIV = 3, OP_MUL_ADD = 4 };

format_spec spec_of(unsigned e, unsigned s, int rn, int ftz) {
  return make_spec(e, s, rn ? rounding_mode::rn : rounding_mode::rz,
                   ftz ? subnormal_policy::ftz : subnormal_policy::gradual);
}

template <typename L>
L load_lane(const std::uint32_t* w) {
  L l = L::zeros();
  if constexpr (L::width >= 64) {
    for (unsigned i = 0; i < L::width / 64; ++i)
      l.set_u64(i, std::uint64_t(w[2 * i]) | (std::uint64_t(w[2 * i + 1]) << 32));
  } else {
    l.set_u64(0, w[0]);
  }
  return l;
}

template <typename L>
void store_lane(const L& l, std::uint32_t* w) {
  if constexpr (L::width >= 64) {
    for (unsigned i = 0; i < L::width / 64; ++i) {
      const std::uint64_t v = l.u64_at(i);
      w[2 * i] = std::uint32_t(v);
      w[2 * i + 1] = std::uint32_t(v >> 32);
    }
  } else {
    w[0] = std::uint32_t(l.u64_at(0));
  }
}

template <typename L>
bfp_vector<L> load_vec(const format_spec& spec, const std::uint32_t* planes,
                       std::size_t block, unsigned part) {
  const unsigned n = spec.total_bits();
  bfp_vector<L> v{spec, bitfield<L>(n)};
  constexpr unsigned wpl = (L::width >= 32) ? L::width / 32 : 1;  // u32 words per lane
  for (unsigned j = 0; j < n; ++j)
    v.field[j] = load_lane<L>(planes + (block * n + j) * 32 + part * wpl);
  return v;
}

template <typename L>
void store_vec(const bfp_vector<L>& v, std::uint32_t* planes, std::size_t block,
               unsigned part) {
  const unsigned n = v.spec.total_bits();
  constexpr unsigned wpl = (L::width >= 32) ? L::width / 32 : 1;
  for (unsigned j = 0; j < n; ++j)
    store_lane<L>(v.field[j], planes + (block * n + j) * 32 + part * wpl);
}

template <unsigned W>
void binop_range(int op, const format_spec& spec, const std::uint32_t* x,
                 const std::uint32_t* y, const std::uint32_t* c, std::uint32_t* z,
                 std::size_t b0, std::size_t b1) {
  using L = lane<W>;
  constexpr unsigned parts = 1024 / W;
  for (std::size_t b = b0; b < b1; ++b) {
    for (unsigned p = 0; p < parts; ++p) {
      const bfp_vector<L> vx = load_vec<L>(spec, x, b, p);
      const bfp_vector<L> vy = load_vec<L>(spec, y, b, p);
      bfp_vector<L> r;
      switch (op) {
        case OP_ADD: r = bfp_add(vx, vy); break;
        case OP_SUB: r = bfp_sub(vx, vy); break;
        case OP_MUL: r = bfp_mul(vx, vy); break;
        case OP_DIV: r = bfp_div(vx, vy); break;
        case OP_MUL_ADD: {
          const bfp_vector<L> vc = load_vec<L>(spec, c, b, p);
          r = bfp_add(bfp_mul(vx, vy), vc);
          break;
        }
        default: return;
      }
      store_vec<L>(r, z, b, p);
    }
  }
}

template <typename F>
void parallel_for(std::size_t n, int threads, F&& f) {
  if (threads <= 1 || n < 2) {
    f(std::size_t{0}, n);
    return;
  }
  const std::size_t t = std::min<std::size_t>(std::size_t(threads), n);
  std::vector<std::thread> pool;
  pool.reserve(t);
  for (std::size_t i = 0; i < t; ++i) {
    const std::size_t lo = n * i / t, hi = n * (i + 1) / t;
    pool.emplace_back([&f, lo, hi] { f(lo, hi); });
  }
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

// Returns 0 on success, 1 for a rejected format (validate(), format.hpp:57-64),
// 2 for an unsupported op or lane width.
int ref_validate(unsigned e, unsigned s) {
  try {
    (void)spec_of(e, s, 1, 0);
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// z = op(x, y[, c]) over nblocks 1024-element blocks of plane images, using
// bfp_add / bfp_sub / bfp_mul / bfp_div (arith.hpp:235-444) on lane<W>;
// op 4 is the chain bfp_add(bfp_mul(x, y), c).  W in {32,64,256,512,1024}.
int ref_binop(int op, unsigned e, unsigned s, int rn, int ftz,
              const std::uint32_t* x, const std::uint32_t* y,
              const std::uint32_t* c, std::uint32_t* z, std::size_t nblocks,
              int threads, unsigned lane_width) {
  format_spec spec;
  try {
    spec = spec_of(e, s, rn, ftz);
  } catch (const std::exception&) {
    return 1;
  }
  if (op < OP_ADD || op > OP_MUL_ADD) return 2;
  auto body = [&](std::size_t lo, std::size_t hi) {
    switch (lane_width) {
      case 32: binop_range<32>(op, spec, x, y, c, z, lo, hi); break;
      case 64: binop_range<64>(op, spec, x, y, c, z, lo, hi); break;
      case 256: binop_range<256>(op, spec, x, y, c, z, lo, hi); break;
      case 512: binop_range<512>(op, spec, x, y, c, z, lo, hi); break;
      default: binop_range<1024>(op, spec, x, y, c, z, lo, hi); break;
    }
  };
  if (lane_width != 32 && lane_width != 64 && lane_width != 256 &&
      lane_width != 512 && lane_width != 1024)
    return 2;
  parallel_for(nblocks, threads, body);
  return 0;
}

// encode_scalar((double)in[i]) -- format.hpp:125-188.
int ref_encode_f32(const float* in, std::size_t n, std::uint64_t* out,
                   unsigned e, unsigned s, int rn, int ftz, int threads) {
  format_spec spec;
  try {
    spec = spec_of(e, s, rn, ftz);
  } catch (const std::exception&) {
    return 1;
  }
  parallel_for(n, threads, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i)
      out[i] = encode_scalar(static_cast<double>(in[i]), spec);
  });
  return 0;
}

std::uint64_t ref_encode_f64(double x, unsigned e, unsigned s, int rn, int ftz) {
  return encode_scalar(x, spec_of(e, s, rn, ftz));
}

double ref_decode_f64(std::uint64_t enc, unsigned e, unsigned s) {
  return decode_scalar(enc, spec_of(e, s, 1, 0));
}

// (float)decode_scalar(enc[i]) -- format.hpp:101-123.
int ref_decode_f32(const std::uint64_t* enc, std::size_t n, float* out,
                   unsigned e, unsigned s, int threads) {
  format_spec spec;
  try {
    spec = spec_of(e, s, 1, 0);
  } catch (const std::exception&) {
    return 1;
  }
  parallel_for(n, threads, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t i = lo; i < hi; ++i)
      out[i] = static_cast<float>(decode_scalar(enc[i], spec));
  });
  return 0;
}

// Documented layout (pack.hpp:13-15) realised by field_from_elements
// (bitfield.hpp:33-43); the tail of the last block is zero (pack.hpp:50).
int ref_pack_planes(const std::uint64_t* enc, std::size_t n, std::uint32_t* planes,
                    unsigned e, unsigned s) {
  using L = lane<1024>;
  const unsigned nb = 1 + e + s;
  const std::size_t blocks = (n + 1023) / 1024;
  for (std::size_t b = 0; b < blocks; ++b) {
    const std::size_t cnt = std::min<std::size_t>(1024, n - b * 1024);
    const bitfield<L> f = field_from_elements<L>(
        nb, std::span<const std::uint64_t>(enc + b * 1024, cnt));
    for (unsigned j = 0; j < nb; ++j)
      store_lane<L>(f[j], planes + (b * nb + j) * 32);
  }
  return 0;
}

// element_of (bitfield.hpp:45-52).
int ref_unpack_planes(const std::uint32_t* planes, std::size_t n,
                      std::uint64_t* out, unsigned e, unsigned s) {
  using L = lane<1024>;
  const unsigned nb = 1 + e + s;
  const std::size_t blocks = (n + 1023) / 1024;
  for (std::size_t b = 0; b < blocks; ++b) {
    bitfield<L> f(nb);
    for (unsigned j = 0; j < nb; ++j)
      f[j] = load_lane<L>(planes + (b * nb + j) * 32);
    const std::size_t cnt = std::min<std::size_t>(1024, n - b * 1024);
    for (std::size_t k = 0; k < cnt; ++k)
      out[b * 1024 + k] = element_of<L>(f, static_cast<unsigned>(k));
  }
  return 0;
}

// The SHIPPED pack (pack.hpp:41-58), block by block -- defective (anti-
// diagonal transpose); exported to document Defect B and to time the
// reference's own float32 -> bitslice path (encode_scalar + pack).
int ref_pack_shipped(const std::uint64_t* enc, std::size_t n,
                     std::uint32_t* planes, unsigned e, unsigned s) {
  using L = lane<1024>;
  const format_spec spec = spec_of(e, s, 1, 0);
  const unsigned nb = spec.total_bits();
  const std::size_t blocks = (n + 1023) / 1024;
  for (std::size_t b = 0; b < blocks; ++b) {
    const std::size_t cnt = std::min<std::size_t>(1024, n - b * 1024);
    const bfp_vector<L> v =
        pack<L>(std::span<const encoding>(enc + b * 1024, cnt), spec);
    for (unsigned j = 0; j < nb; ++j)
      store_lane<L>(v.field[j], planes + (b * nb + j) * 32);
  }
  return 0;
}

int ref_unpack_shipped(const std::uint32_t* planes, std::size_t n,
                       std::uint64_t* out, unsigned e, unsigned s) {
  using L = lane<1024>;
  const format_spec spec = spec_of(e, s, 1, 0);
  const unsigned nb = spec.total_bits();
  const std::size_t blocks = (n + 1023) / 1024;
  for (std::size_t b = 0; b < blocks; ++b) {
    bfp_vector<L> v{spec, bitfield<L>(nb)};
    for (unsigned j = 0; j < nb; ++j)
      v.field[j] = load_lane<L>(planes + (b * nb + j) * 32);
    const std::size_t cnt = std::min<std::size_t>(1024, n - b * 1024);
    const std::vector<encoding> r = unpack<L>(v, cnt);
    std::memcpy(out + b * 1024, r.data(), cnt * sizeof(encoding));
  }
  return 0;
}

// The reference's CPU float32 -> bitslice path as a caller would write it:
// encode_scalar per element, then the shipped pack, threaded over blocks.
int ref_pack_f32_path(const float* in, std::size_t n, std::uint32_t* planes,
                      unsigned e, unsigned s, int rn, int ftz, int threads) {
  using L = lane<1024>;
  const format_spec spec = spec_of(e, s, rn, ftz);
  const unsigned nb = spec.total_bits();
  const std::size_t blocks = (n + 1023) / 1024;
  parallel_for(blocks, threads, [&](std::size_t lo, std::size_t hi) {
    std::vector<encoding> enc(1024);
    for (std::size_t b = lo; b < hi; ++b) {
      const std::size_t cnt = std::min<std::size_t>(1024, n - b * 1024);
      for (std::size_t k = 0; k < cnt; ++k)
        enc[k] = encode_scalar(static_cast<double>(in[b * 1024 + k]), spec);
      const bfp_vector<L> v =
          pack<L>(std::span<const encoding>(enc.data(), cnt), spec);
      for (unsigned j = 0; j < nb; ++j)
        store_lane<L>(v.field[j], planes + (b * nb + j) * 32);
    }
  });
  return 0;
}

// The reference's CPU bitslice -> float32 path: shipped unpack, then
// decode_scalar per element.
int ref_unpack_f32_path(const std::uint32_t* planes, std::size_t n, float* out,
                        unsigned e, unsigned s, int threads) {
  using L = lane<1024>;
  const format_spec spec = spec_of(e, s, 1, 0);
  const unsigned nb = spec.total_bits();
  const std::size_t blocks = (n + 1023) / 1024;
  parallel_for(blocks, threads, [&](std::size_t lo, std::size_t hi) {
    for (std::size_t b = lo; b < hi; ++b) {
      bfp_vector<L> v{spec, bitfield<L>(nb)};
      for (unsigned j = 0; j < nb; ++j)
        v.field[j] = load_lane<L>(planes + (b * nb + j) * 32);
      const std::size_t cnt = std::min<std::size_t>(1024, n - b * 1024);
      const std::vector<encoding> r = unpack<L>(v, cnt);
      for (std::size_t k = 0; k < cnt; ++k)
        out[b * 1024 + k] = static_cast<float>(decode_scalar(r[k], spec));
    }
  });
  return 0;
}

// Gate tally of one evaluation via counted_lane (lane.hpp:119-188); the
// circuits are data independent so zero operands suffice.
// counts = {and, or, xor, not}.
int ref_gate_count(int op, unsigned e, unsigned s, int rn, int ftz,
                   std::uint64_t* counts) {
  using L = counted_lane<32>;
  format_spec spec;
  try {
    spec = spec_of(e, s, rn, ftz);
  } catch (const std::exception&) {
    return 1;
  }
  const unsigned nb = spec.total_bits();
  const bfp_vector<L> x{spec, bitfield<L>(nb)}, y{spec, bitfield<L>(nb)};
  L::counter().reset();
  switch (op) {
    case OP_ADD: (void)bfp_add(x, y); break;
    case OP_SUB: (void)bfp_sub(x, y); break;
    case OP_MUL: (void)bfp_mul(x, y); break;
    case OP_DIV: (void)bfp_div(x, y); break;
    case OP_MUL_ADD: (void)bfp_add(bfp_mul(x, y), x); break;
    default: return 2;
  }
  const op_counter c = L::counter();
  counts[0] = c.and_count;
  counts[1] = c.or_count;
  counts[2] = c.xor_count;
  counts[3] = c.not_count;
  return 0;
}

// .bfpraw codec (pack.hpp:78-109).
std::size_t ref_bfpraw_stride(unsigned e, unsigned s) {
  return bfpraw_stride(spec_of(e, s, 1, 0));
}

int ref_to_bfpraw(const std::uint64_t* enc, std::size_t n, std::uint8_t* out,
                  unsigned e, unsigned s) {
  const std::vector<std::uint8_t> r =
      to_bfpraw(std::span<const encoding>(enc, n), spec_of(e, s, 1, 0));
  std::memcpy(out, r.data(), r.size());
  return 0;
}

int ref_from_bfpraw(const std::uint8_t* bytes, std::size_t nbytes,
                    std::uint64_t* out, unsigned e, unsigned s) {
  try {
    const std::vector<encoding> r = from_bfpraw(
        std::span<const std::uint8_t>(bytes, nbytes), spec_of(e, s, 1, 0));
    std::memcpy(out, r.data(), r.size() * sizeof(encoding));
  } catch (const std::exception&) {
    return 3;
  }
  return 0;
}

}  // extern "C"
