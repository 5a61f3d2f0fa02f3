// tree_device.cuh — device-resident tree refinement (tree_refine, ref
// src/estimator.cpp:212-318) for many trees at once.
//
// Leaves live in HBM for the whole run.  A round is four kernels and one
// small read-back: k_tree_select (a thread per tree: the reference's mean /
// sd of the leaf std_errors in leaf order, the threshold, the longest-edge
// splits with the budget check — writing the new cells' rectangles to a
// staging list), k_tree_layout (one CTA: tile ranges of the new cells in the
// launch groups, descriptor updates), the fused cell kernels + k_combine in
// cell-list mode (tree.hpp / mcb_device.cuh), and k_tree_scatter (estimates
// back into the leaves).  The host only reads the per-group tile counts to
// size the next launches.  k_tree_finish combines the leaves
// (combine_cells, src/estimator.cpp:145-159) per tree.
//
// Every floating-point step of the selection and split is the reference's,
// in its order, with explicitly rounded operations (the library is built
// with -fmad=false), so trees are identical to the host driver's (tree.cpp).
#pragma once

#include <cstdint>

#include "cell_est.hpp"
#include "mcb_device.cuh"

namespace mcb {
namespace tdev {

struct TreeConst {    // per tree, written once by the host
  uint64_t leaf_off;  // first leaf slot of this tree
  uint64_t rect_off;  // first double of its rectangle storage (leaf i: rect_off + 2*dim*i)
  uint64_t budget;    // total_budget (= n_samples)
  double sigma;       // sigma_multiplier
  uint32_t leaf_cap;  // leaf slots reserved
  uint32_t dim, spc, cpc;
  uint32_t max_depth;
  uint32_t warp_tiles;  // the tree's cell kernel is warp-per-tile: pad tile ranges to 8
  uint32_t group;       // launch group (trees are sorted by group)
  uint32_t reserved;
  uint64_t init_off;    // first double of its first-pass grid in the packed upload
};

struct TreeState {  // per tree, updated on the device
  uint64_t used, next_chunk, chunk0;
  uint32_t n_leaves, n_new, active, exhausted, fail, reserved;
};

struct Leaves {  // device arrays, indexed by leaf slot (leaf_off + i)
  double* rect;        // 2*dim doubles per leaf: {low[dim], high[dim]}
  double* se;          // std_error (the selection statistic)
  double* val;         // value
  uint32_t* nn;        // non-finite samples
  uint32_t* depth;
  uint32_t* dead;      // 1: the cell had no finite sample
  uint32_t* new_leaf;  // this round's new cells: the leaf each one estimates
  double* new_rect;    //   and its rectangle (same layout as rect)
  CellEst* est;        //   and its estimate
};

}  // namespace tdev

namespace detail {

cudaError_t launch_tree_init(const tdev::TreeConst* tc, const tdev::TreeState* ts, tdev::Leaves L,
                             const double* packed, uint32_t n_trees, cudaStream_t s);
cudaError_t launch_tree_select(const tdev::TreeConst* tc, tdev::TreeState* ts, tdev::Leaves L, uint32_t n_trees,
                               cudaStream_t s);
cudaError_t launch_tree_layout(const tdev::TreeConst* tc, const tdev::TreeState* ts, dev::FnDesc* fns,
                               tdev::Leaves L, uint32_t n_trees, uint64_t* group_tiles, uint32_t n_groups,
                               cudaStream_t s);
cudaError_t launch_tree_scatter(const tdev::TreeConst* tc, const tdev::TreeState* ts, tdev::Leaves L,
                                uint32_t n_trees, cudaStream_t s);
cudaError_t launch_tree_finish(const tdev::TreeConst* tc, const tdev::TreeState* ts, tdev::Leaves L,
                               uint32_t n_trees, mcb_trial_stats* out, cudaStream_t s);

}  // namespace detail
}  // namespace mcb
