// cell_est.hpp — compact per-cell result of a tree refinement round, written
// by k_combine in cell-list mode and read by the host driver (tree.cpp).
#pragma once

#include <cstdint>

namespace mcb {

// direct_mc estimate of one cell (reduce_chunks, ref src/estimator.cpp:55-73):
// value = V * mean, std_error = V * sqrt(m2/(n-1)/n) (+inf for one finite
// sample), n_nonfinite of the cell's spc samples; status MCB_TRIAL_OK or
// MCB_TRIAL_ALL_NONFINITE (no finite sample: a dead leaf).
struct CellEst {
  double value;
  double std_error;
  uint32_t n_nonfinite;
  uint32_t status;
};

}  // namespace mcb
