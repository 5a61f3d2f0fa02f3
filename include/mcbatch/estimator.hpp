// mcbatch/estimator.hpp — source-compatible face of the reference header
// include/mcbatch/estimator.hpp over libmcb.  The estimators take the
// reference's (CompiledProgram, params, rect, ..., StreamKey) arguments and
// run on the GPU (device 0): the same keys, chunking, ordered merge and
// McEstimate as the reference, per SURVEY.md §8(a).
//
// Not provided: ChunkAccum / accumulate_chunk / reduce_chunks (the per-chunk
// host Welford of the reference's task body, replaced by the fused kernels'
// on-chip reduction and k_combine).
#pragma once

#include <cstdint>
#include <functional>
#include <span>
#include <utility>
#include <vector>

#include "mcb/mcbatch.hpp"
#include "mcbatch/expr.hpp"
#include "mcbatch/sampling.hpp"

namespace mcbatch {

inline constexpr double kNonFiniteWarnFraction = mcb::kNonFiniteWarnFraction;

using mcb::AllSamplesNonFinite;
using mcb::CellBudgetExceeded;
using mcb::InsufficientTrials;
using mcb::McEstimate;
using mcb::RefineConfig;
using mcb::TrialSummary;

struct StratumNode {  // estimator.hpp:33-38
  HyperRect cell;
  McEstimate estimate;
  std::uint32_t depth = 0;
  std::vector<StratumNode> children;
};

using mcb::auto_cells_per_dim;
using mcb::cell_grid_size;
using mcb::chunk_count;
using mcb::combine_cells;
using mcb::grid_cell;
using mcb::repeated_trials;
using mcb::summarize_trials;

McEstimate direct_mc(const CompiledProgram& program, std::span<const double> params, const HyperRect& rect,
                     std::uint64_t n_samples, const StreamKey& key_base);

std::pair<McEstimate, std::vector<StratumNode>> stratified_mc(const CompiledProgram& program,
                                                              std::span<const double> params,
                                                              const HyperRect& rect, std::uint32_t cells_per_dim,
                                                              std::uint32_t samples_per_cell,
                                                              const StreamKey& key_base,
                                                              std::uint64_t cell_cap = 1000000);

McEstimate tree_refine(const CompiledProgram& program, std::span<const double> params, const HyperRect& rect,
                       const RefineConfig& config, const StreamKey& key_base,
                       std::vector<StratumNode>* leaves_out = nullptr);

}  // namespace mcbatch
