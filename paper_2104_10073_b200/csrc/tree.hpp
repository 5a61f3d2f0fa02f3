// tree.hpp — host driver of the adaptive tree method,
// tree_refine of ref src/estimator.cpp:184-318 run for many (integrand,
// trial) trees at once.  The default path keeps the leaves on the device
// (tree_device.cuh); this host driver is the cross-check it is tested
// against (MCB_TREE_DEVICE=0) and shares its configuration rules.
//
// tree_refine is sequential per tree (each round's split choice depends on
// the previous round's cell estimates) but every cell estimate inside a round
// is independent, and so is every tree of a batch.  The driver therefore runs
// all trees in lock-step rounds: round 0 estimates every tree's initial grid,
// round r every cell split in round r; each round's cells of ALL trees go to
// the GPU as one launch set through `CellRunner`: per tree a cell-list
// descriptor + its cell rectangles, estimated by the fused kernels in
// cell-list mode and sharded over the devices (capi.cpp).  Selection, splitting and budget
// accounting repeat the reference's host arithmetic operation for operation.
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "cell_est.hpp"
#include "mcb/mcb.h"

namespace mcb::tree {

// One tree's new cells of a refinement round: cell c is a direct_mc unit of
// `fn` restricted to rects[c] with spc samples and key base
// {seed, fn->integrand_index, trial, chunk_base + c * chunk_count(spc)}
// (consecutive estimate_cell calls, ref src/estimator.cpp:238-253).
struct CellBatch {
  const mcb_integrand* fn;  // method TREE
  uint32_t trial;
  uint64_t chunk_base;
  uint32_t spc;
  uint32_t n_cells;
  const double* rects;      // n_cells x {low[dim], high[dim]}
  CellEst* est;             // n_cells per-cell estimates (status ALL_NONFINITE = no finite sample)
};

// Estimates every batch of a round.  Returns MCB_OK or an error status
// (message already recorded by the implementation).
using CellRunner = std::function<mcb_status(const std::vector<CellBatch>& batches)>;

struct TreeTask {
  const mcb_integrand* fn;   // method TREE; n_samples = total_budget
  uint32_t trial;
  uint64_t chunk_base;       // key_base.chunk_index
  mcb_trial_stats* out;      // the tree's McEstimate (status replaces exceptions)
  std::vector<mcb_leaf>* leaves = nullptr;  // optional leaves_out
};

// Resolved RefineConfig of a TREE descriptor.
struct Config {
  uint32_t init_cells_per_dim = 0;
  uint32_t samples_per_cell = 2048;
  uint32_t max_depth = 6;
  double sigma_multiplier = 1.0;
  uint64_t total_budget = 100000;
  uint64_t cell_cap = 1000000;
};
Config config_of(const mcb_integrand& f);

// Runs every task to completion.  Returns the first CellRunner error, else MCB_OK.
mcb_status run_trees(std::vector<TreeTask>& tasks, const CellRunner& run);

}  // namespace mcb::tree
