// Instantiations of the fused kernel for the vector-k harmonic family
// a*cos(k1*x1+..+kd*xd) + b*sin(k1*x1+..+kd*xd), d = 1..8.
#include "kernels.cuh"

namespace mcb {
namespace detail {

template <int D>
static void put_vec(Table& t) {
  constexpr int F = MCB_FAMILY_HARMONIC_VEC;
  t.put<F, D, kFoldShift>();
  t.put<F, D, kFoldShift | kUnitDomain>();
  t.put<F, D, kSafe>();
  t.put_run<F, D, 0>();
  t.put_run<F, D, kSafe>();
}

void register_harmonic_vec(Table& t) {
#ifndef MCB_BENCH_ONLY
  put_vec<1>(t);
  put_vec<2>(t);
  put_vec<3>(t);
  put_vec<4>(t);
  put_vec<5>(t);
  put_vec<6>(t);
  put_vec<7>(t);
  put_vec<8>(t);
#endif
}

}  // namespace detail
}  // namespace mcb
