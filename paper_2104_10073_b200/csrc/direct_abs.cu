// Instantiations of the fused kernel for a*|x1+x2| (d = 2..8) and
// a*|x1+x2-x3| (d = 3..8); draws of unused coordinates are skipped.
#include "kernels.cuh"

namespace mcb {
namespace detail {

template <int F, int D>
static void put_abs(Table& t) {
  t.put<F, D, 0>();
  t.put<F, D, kUnitDomain>();
  t.put<F, D, kSafe>();
  t.put_run<F, D, 0>();
  t.put_run<F, D, kSafe>();
}

void register_abs(Table& t) {
#ifndef MCB_BENCH_ONLY
  put_abs<MCB_FAMILY_ABS2, 2>(t);
  put_abs<MCB_FAMILY_ABS2, 3>(t);
  put_abs<MCB_FAMILY_ABS2, 4>(t);
  put_abs<MCB_FAMILY_ABS2, 5>(t);
  put_abs<MCB_FAMILY_ABS2, 6>(t);
  put_abs<MCB_FAMILY_ABS2, 7>(t);
  put_abs<MCB_FAMILY_ABS2, 8>(t);
  put_abs<MCB_FAMILY_ABS3, 3>(t);
  put_abs<MCB_FAMILY_ABS3, 4>(t);
  put_abs<MCB_FAMILY_ABS3, 5>(t);
  put_abs<MCB_FAMILY_ABS3, 6>(t);
  put_abs<MCB_FAMILY_ABS3, 7>(t);
  put_abs<MCB_FAMILY_ABS3, 8>(t);
#endif
}

}  // namespace detail
}  // namespace mcb
