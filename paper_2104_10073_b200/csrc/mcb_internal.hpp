// mcb_internal.hpp — host-side declarations shared by the C-ABI layer and the
// CUDA translation unit.  Not part of the public interface.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "mcb/mcb.h"
#include "mcb_device.cuh"

namespace mcb {
namespace prog {
struct Program;
}
namespace detail {

#ifndef MCB_THREADS
#define MCB_THREADS 256
#endif
#ifndef MCB_MIN_BLOCKS
#define MCB_MIN_BLOCKS 2
#endif
#ifndef MCB_PIPELINE
#define MCB_PIPELINE 1
#endif
constexpr int kThreads = MCB_THREADS;  // CTA size of the fused kernel
constexpr int kProgThreads = 128;      // CTA size of the DSL-interpreter kernel

enum Variant : int {
  kUnitDomain = 1,  // low == 0, width == 1 on every axis
  kUnitCoef = 2,    // HARMONIC with a == b == 1 (Fig.1 source form)
  kSafe = 4,        // plain parameters, libdevice sincos, non-finite samples
                    // counted and skipped (used when the host cannot prove
                    // the FAST preconditions, see capi.cpp prepare())
  kFoldShift = 8,   // harmonic FAST, direct (not kStrat): the per-integrand
                    // shift c is folded into the CTA's table (A_m - c), so
                    // g = f - c costs no extra FP64 operation (mcb_device.cuh)
  kStrat = 16,      // STRATIFIED method: tiles are (trial, cell, chunk), the
                    // cell rectangle is derived on the device (grid_cell)
  kWarpTile = 32,   // with kStrat, small cells: one WARP per tile, so a CTA
                    // covers kTileAlign tiles of one (integrand, trial); each
                    // integrand's per-trial tile range is padded to a
                    // multiple of kTileAlign and its tile_base aligned
  kLaneCell = 64    // with kStrat (not kWarpTile), small cells of a large
                    // grid: one LANE per cell, a one-warp CTA covers
                    // kLaneAlign cells of one (integrand, trial); ranges
                    // padded / aligned to kLaneAlign (family kernels only)
};
constexpr int kNumVariants = 128;

// Tile alignment of kWarpTile integrands (= warps of the family kernel's CTA,
// a multiple of the interpreter's 4 warps) and the cell size up to which
// cell-structured integrands use it.
constexpr uint32_t kTileAlign = 8;
constexpr uint32_t kWarpTileMaxSpc = 8192;
// kLaneCell: cells per CTA (one warp) and the smallest grid that uses it.
constexpr uint32_t kLaneAlign = 32;
constexpr uint32_t kLaneCellMinCells = 256;

// DSL programs: a lane per cell on grids of at least this many cells
// (one CTA = kProgThreads cells, so ranges are padded to kProgThreads).
constexpr uint32_t kProgLaneMinCells = 1024;

// Tiles per CTA of a variant's kernel (family kernels / the DSL programs'
// interpreter and specialised kernels, kProgThreads per CTA).
constexpr uint32_t tiles_per_cta(int variant, bool program = false) {
  return program ? ((variant & kLaneCell) ? uint32_t(kProgThreads) : (variant & kWarpTile) ? uint32_t(kProgThreads / 32) : 1u)
                 : ((variant & kLaneCell) ? kLaneAlign : (variant & kWarpTile) ? kTileAlign : 1u);
}
// Alignment of a variant's tile ranges (per (integrand, trial) and per
// descriptor): the CTA's tiles, and kTileAlign for any warp-per-tile group.
constexpr uint32_t tile_align(int variant, bool program = false) {
  return (variant & kWarpTile) ? kTileAlign : tiles_per_cta(variant, program);
}
// Kernel mode of a DSL program group (jit_kernels.cuh, kernels_program.cu):
// 0 direct, 1 direct on [0,1]^d, 2 cells (CTA per tile), 3 small cells (warp
// per tile), 4 small cells of a large grid (lane per cell).
constexpr int program_kernel_mode(int variant) {
  return (variant & kLaneCell) ? 4 : (variant & kWarpTile) ? 3 : (variant & kStrat) ? 2 : (variant & kUnitDomain) ? 1 : 0;
}
static_assert(kThreads / 32 == int(kTileAlign), "family CTA = kTileAlign warps");
static_assert(kTileAlign % (kProgThreads / 32) == 0, "interpreter CTAs tile the aligned groups");

// One kernel launch = one (family, dim, variant) group of integrands whose
// tiles are contiguous in the plan's tile space.
struct GroupLaunch {
  int family, dim, variant;
  uint64_t tile0, n_tiles;
  uint32_t slots = 0;  // PROGRAM family: max stack depth of the group's programs
  const prog::Program* prog = nullptr;  // PROGRAM family: the group's one program (runtime-specialised)
  uint32_t tile_samples = MCB_CHUNK_SIZE;  // most samples one tile of the group draws (JIT policy)
};

bool variant_supported(int family, int dim, int variant);

cudaError_t launch_direct_group(const GroupLaunch& g, const dev::FnDesc* fns,
                                const uint32_t* tile_fn, dev::TilePartial* part,
                                cudaStream_t s);
cudaError_t launch_expand_tiles(const dev::FnDesc* fns, uint32_t n_fns, uint32_t trials,
                                uint32_t* tile_fn, cudaStream_t s);
cudaError_t launch_combine(const dev::FnDesc* fns, uint32_t n_fns, uint32_t trials,
                           const dev::TilePartial* part, mcb_trial_stats* out,
                           cudaStream_t s);
cudaError_t launch_debug_points(uint32_t key0, uint32_t key1, uint32_t trial, uint32_t chunk,
                                uint64_t first_point, uint64_t count, uint32_t dim,
                                const double* low, const double* width, double* out,
                                cudaStream_t s);
cudaError_t launch_debug_eval_impl(int family, int dim, int variant, const dev::FnDesc* fn,
                                   uint32_t trial, uint32_t chunk, uint32_t first_pair,
                                   uint32_t n_pairs, double* out, cudaStream_t s);
cudaError_t launch_program_group(const GroupLaunch& g, const dev::FnDesc* fns,
                                 const uint32_t* tile_fn, dev::TilePartial* part,
                                 const uint32_t* code, const double* consts, cudaStream_t s);
cudaError_t launch_program_eval(int dim, int variant, const dev::FnDesc* fn, const uint32_t* code,
                                const double* consts, uint32_t slots, uint32_t trial, uint32_t chunk,
                                uint32_t first_pair, uint32_t n_pairs, double* out, cudaStream_t s);
cudaError_t launch_program_points(int dim, const dev::FnDesc* fn, const uint32_t* code,
                                  const double* consts, uint32_t slots, const double* pts, uint64_t n,
                                  double* out, cudaStream_t s);
cudaError_t launch_philox_probe(const uint32_t* key, uint32_t* sink, int n_ctas, int iters,
                               cudaStream_t s);

}  // namespace detail
}  // namespace mcb
