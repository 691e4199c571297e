// tests/native/cpp_api_test.cpp -- TEST ONLY: drives the C++ drop-in header
// (include/bfp/gpu.hpp) the way a reference user would, and checks results
// against the oracle's C restatement (oracle/liboracle.so).
#include <bfp/gpu.hpp>

#include <cstdio>
#include <random>
#include <stdexcept>
#include <vector>

extern "C" uint64_t orc_binop(int op, unsigned e, unsigned s, int rn, int ftz, uint64_t x, uint64_t y);
extern "C" uint64_t orc_encode(double x, unsigned e, unsigned s, int rn, int ftz);

int main() {
  namespace g = bfp::gpu;
  int fails = 0;
  {  // split / classify (format.hpp:83-99)
    const auto f = g::make_spec(5, 10);
    const g::encoding cases[] = {0x0000, 0x8001, 0x3c00, 0x7c00, 0xfe00, 0x03ff};
    const g::value_class want[] = {g::value_class::zero, g::value_class::subnormal, g::value_class::normal,
                                   g::value_class::infinity, g::value_class::nan, g::value_class::subnormal};
    for (int k = 0; k < 6; ++k)
      if (g::classify(cases[k], f) != want[k]) {
        std::printf("classify mismatch %d\n", k);
        ++fails;
      }
    const auto sc = g::split(0xbc01, f);
    if (sc.sign != 1 || sc.biased_exp != 15 || sc.fraction != 1) {
      std::printf("split mismatch\n");
      ++fails;
    }
  }
  std::mt19937_64 rng(42);
  for (auto [e, s] : {std::pair{4u, 3u}, std::pair{5u, 10u}, std::pair{8u, 15u}}) {
    for (int rn = 0; rn < 2; ++rn) {
      const auto spec = g::make_spec(e, s, rn ? g::rounding_mode::rn : g::rounding_mode::rz,
                                     g::subnormal_policy::gradual, "t");
      const std::size_t n = 3000;
      std::vector<g::encoding> xs(n), ys(n);
      for (auto& v : xs) v = rng() & ((1ull << spec.total_bits()) - 1);
      for (auto& v : ys) v = rng() & ((1ull << spec.total_bits()) - 1);
      const g::bfp_vector x = g::pack(xs, spec), y = g::pack(ys, spec);
      const g::bfp_vector zs[4] = {g::bfp_add(x, y), g::bfp_sub(x, y), g::bfp_mul(x, y), g::bfp_div(x, y)};
      for (int op = 0; op < 4; ++op) {
        const auto z = g::unpack(zs[op], n);
        for (std::size_t i = 0; i < n; ++i)
          if (z[i] != orc_binop(op, e, s, rn, 0, xs[i], ys[i])) {
            if (fails++ < 5) std::printf("mismatch 1/%u/%u op%d i=%zu\n", e, s, op, i);
          }
      }
      for (double v : {1.5, -3.25, 1e-6, 65504.0, 7e5})
        if (g::encode_scalar(v, spec) != orc_encode(v, e, s, rn, 0)) ++fails;
      // fused expression == the same ops one call at a time
      const auto ch = g::unpack(g::chain("ab*ab-/", {&x, &y}), n);
      const auto seq = g::unpack(g::bfp_div(g::bfp_mul(x, y), g::bfp_sub(x, y)), n);
      if (ch != seq) {
        std::printf("chain mismatch 1/%u/%u\n", e, s);
        ++fails;
      }
    }
  }
  // .bfpraw round trip through the device, a 51-bit format (runtime backend)
  {
    const auto spec = g::make_spec(10, 40);
    std::vector<g::encoding> xs(2000);
    for (auto& v : xs) v = rng() & ((1ull << spec.total_bits()) - 1);
    const auto raw = g::to_bfpraw(xs, spec);
    const g::bfp_vector v = g::pack_bfpraw(raw, spec);
    if (g::unpack_bfpraw(v) != raw) ++fails;
    if (g::unpack(v, xs.size()) != xs) ++fails;
    if (g::from_bfpraw(raw, spec) != xs) ++fails;
  }
  // error behaviour mirrors the reference: std::invalid_argument
  bool threw = false;
  try {
    (void)g::make_spec(1, 3);
  } catch (const std::invalid_argument&) { threw = true; }
  if (!threw) ++fails;
  threw = false;
  try {
    const auto a = g::pack(std::vector<g::encoding>{1, 2, 3}, g::make_spec(4, 3, g::rounding_mode::rn, g::subnormal_policy::gradual, "a"));
    const auto b = g::pack(std::vector<g::encoding>{1, 2, 3}, g::make_spec(4, 3, g::rounding_mode::rn, g::subnormal_policy::gradual, "b"));
    (void)g::bfp_add(a, b);
  } catch (const std::invalid_argument&) { threw = true; }
  if (!threw) ++fails;
  threw = false;
  try {
    const auto a = g::pack(std::vector<g::encoding>{1, 2, 3}, g::make_spec(4, 3));
    (void)g::unpack(a, 4);
  } catch (const std::invalid_argument&) { threw = true; }
  if (!threw) ++fails;
  std::printf("cpp_api_test: %s (%d failures)\n", fails ? "FAIL" : "ok", fails);
  return fails ? 1 : 0;
}
