// Instantiations of the fused kernel for the harmonic family
// a*cos(k*(x1+..+xd)) + b*sin(k*(x1+..+xd)), d = 1..8.
#include "kernels.cuh"

namespace mcb {
namespace detail {

template <int D>
static void put_harmonic(Table& t) {
  constexpr int F = MCB_FAMILY_HARMONIC;
  t.put<F, D, kFoldShift>();
  t.put<F, D, kFoldShift | kUnitDomain>();
  t.put<F, D, kFoldShift | kUnitCoef>();
  t.put<F, D, kFoldShift | kUnitCoef | kUnitDomain>();
  t.put<F, D, kSafe>();
  t.put_run<F, D, 0>();
  t.put_run<F, D, kUnitCoef>();
  t.put_run<F, D, kSafe>();
}

void register_harmonic(Table& t) {
#ifdef MCB_BENCH_ONLY
  t.put<MCB_FAMILY_HARMONIC, 4, MCB_BENCH_ONLY>();
#else
  put_harmonic<1>(t);
  put_harmonic<2>(t);
  put_harmonic<3>(t);
  put_harmonic<4>(t);
  put_harmonic<5>(t);
  put_harmonic<6>(t);
  put_harmonic<7>(t);
  put_harmonic<8>(t);
#endif
}

}  // namespace detail
}  // namespace mcb
