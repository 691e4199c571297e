// oracle/shim.hpp -- TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// Force-included (g++ -include oracle/shim.hpp) when compiling the reference
// headers in place from /root/reference/proj/include.  The shipped arith.hpp
// declares `check_shapes(const bfp_vector_spec_pair_tag&) = delete;`
// (arith.hpp:162) with an undeclared type, so the header set does not compile
// as shipped ("Defect A").  A forward declaration of that tag
// in the same namespace is enough; nothing in the reference is modified.
#pragma once
namespace bfp {
namespace detail {
struct bfp_vector_spec_pair_tag;
}  // namespace detail
}  // namespace bfp
