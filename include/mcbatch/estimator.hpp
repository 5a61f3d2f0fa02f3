// mcbatch/estimator.hpp — source-compatible face of the reference header
// include/mcbatch/estimator.hpp over libmcb.  The estimators take the
// reference's (CompiledProgram, params, rect, ..., StreamKey) arguments and
// run on the GPU (device 0): the same keys, chunking, ordered merge and
// McEstimate as the reference, per SURVEY.md §8(a).
//
// The per-chunk layer (ChunkAccum, accumulate_chunk, reduce_chunks) is here
// too: accumulate_chunk runs the chunk as one tile of the fused kernel on the
// GPU and returns its exact counts and (mean, m2) from the tile's shifted
// sums; ChunkAccum's add/merge and reduce_chunks are the reference's host
// recurrences on caller-held accumulators.
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

// estimator.hpp:59-68: one chunk's Welford accumulator.
struct ChunkAccum {
  std::uint64_t n = 0;
  std::uint64_t n_nonfinite = 0;
  double mean = 0.0;
  double m2 = 0.0;

  void add(double x);                    // non-finite x only counted (src/estimator.cpp:9-18)
  void merge(const ChunkAccum& other);   // Chan's pairwise update (src/estimator.cpp:20-34)
};

// estimator.hpp:70-74: the chunk `key` (count <= kChunkSize points of rect)
// evaluated and accumulated on the GPU.
ChunkAccum accumulate_chunk(const CompiledProgram& program, std::span<const double> params,
                            const HyperRect& rect, const StreamKey& key, std::size_t count);

// estimator.hpp:76-78: merge in the given (ascending chunk) order, then the
// McEstimate of src/estimator.cpp:55-73; AllSamplesNonFinite when nothing
// finite survived.
McEstimate reduce_chunks(double volume, std::span<const ChunkAccum> chunks);

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
