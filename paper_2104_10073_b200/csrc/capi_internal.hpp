// capi_internal.hpp — shared internals of the C-ABI layer (not public):
// descriptor lowering and validation (capi_plan.cpp), device plans and the
// per-device contexts, the tree runners (capi_tree.cpp), the extern "C"
// entry points (capi.cpp).  Everything here has hidden visibility.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "cell_est.hpp"
#include "mcb/mcb.h"
#include "mcb_internal.hpp"
#include "program.hpp"
#include "tree.hpp"
#include "tree_device.cuh"

// Opaque compiled program of the C-ABI.
struct mcb_program {
  mcb::prog::Program p;
  std::vector<uint32_t> words;
};

namespace mcb {
namespace capi {

using mcb::detail::GroupLaunch;
using mcb::dev::FnDesc;
using mcb::dev::TilePartial;

extern thread_local std::string g_last_error;  // message of the last failing call on this thread
mcb_status fail(mcb_status st, const std::string& msg);
mcb_status cuda_fail(cudaError_t e, const char* what);
#define MCB_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
  } while (0)

template <class T>
T round_up(T v, T m) { return (v + m - 1) / m * m; }

struct StratPlan {
  uint32_t k = 1, spc = 2;
  uint64_t n_cells = 1;
  bool ok = false;
};
struct Prepared {
  FnDesc d;
  int variant;
};
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
// Host half of a plan: device descriptors grouped by (family, dim, variant)
// with tile bases assigned; no CUDA calls.
struct HostPlan {
  std::vector<FnDesc> descs;  // group order
  std::vector<GroupLaunch> groups;
  std::vector<uint32_t> code;  // PROGRAM family: all distinct programs' words
  std::vector<double> consts;  //   and constant pools
  std::vector<double> bounds;        // STRATIFIED: grid boundaries of every integrand
  std::vector<int64_t> bounds_off;   //   per descriptor: offset into `bounds` (-1: none)
  uint64_t n_tiles = 0, total_samples = 0, philox_blocks = 0;
};
// Growable device buffers of a plan.
struct DevBuf {
  FnDesc* fns = nullptr;
  uint32_t* tile_fn = nullptr;
  TilePartial* part = nullptr;
  mcb_trial_stats* out = nullptr;
  uint32_t* code = nullptr;
  double* consts = nullptr;
  double* bounds = nullptr;             // stratified grid boundaries
  size_t cap_bounds = 0;
  double* rects = nullptr;              // tree rounds: cell rectangles
  mcb::CellEst* cell_est = nullptr;     //   and per-cell estimates
  size_t cap_fns = 0, cap_tiles = 0, cap_part = 0, cap_out = 0, cap_code = 0, cap_consts = 0;
  size_t cap_rects = 0, cap_cell_est = 0;
  template <class T>
  static cudaError_t grow(T*& p, size_t& cap, size_t need) {
    if (need <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t n = std::max<size_t>(need, 1);
    cudaError_t e = cudaMalloc(&p, sizeof(T) * n);
    if (e == cudaSuccess) cap = n;
    return e;
  }
  cudaError_t reserve(size_t n_fns, size_t n_tiles, size_t n_out, size_t n_code = 0,
                      size_t n_consts = 0) {
    cudaError_t e;
    if ((e = grow(code, cap_code, n_code)) != cudaSuccess) return e;
    if ((e = grow(consts, cap_consts, n_consts)) != cudaSuccess) return e;
    if ((e = grow(fns, cap_fns, n_fns)) != cudaSuccess) return e;
    if ((e = grow(tile_fn, cap_tiles, n_tiles)) != cudaSuccess) return e;
    if ((e = grow(part, cap_part, n_tiles)) != cudaSuccess) return e;
    return grow(out, cap_out, n_out);
  }
  void release() {
    if (fns) cudaFree(fns);
    if (tile_fn) cudaFree(tile_fn);
    if (part) cudaFree(part);
    if (out) cudaFree(out);
    if (code) cudaFree(code);
    if (consts) cudaFree(consts);
    if (bounds) cudaFree(bounds);
    if (rects) cudaFree(rects);
    if (cell_est) cudaFree(cell_est);
    *this = DevBuf{};
  }
};
// Per-device context reused by mcb_run_direct: stream, device buffers and
// pinned staging, so a call costs H2D + kernels + D2H, not allocations.
struct DeviceCtx {
  std::mutex mu;
  bool ready = false;
  cudaStream_t stream = nullptr;
  DevBuf buf;
  FnDesc* h_descs = nullptr;
  size_t h_descs_cap = 0;
  mcb_trial_stats* h_out = nullptr;
  size_t h_out_cap = 0;
  double* h_rects = nullptr;
  size_t h_rects_cap = 0;
  mcb::CellEst* h_cell_est = nullptr;
  size_t h_cell_est_cap = 0;
  // device-resident tree runs
  mcb::tdev::TreeConst* t_const = nullptr;
  mcb::tdev::TreeState* t_state = nullptr;
  uint64_t* t_groups = nullptr;
  size_t cap_trees = 0, cap_tstate = 0, cap_tgroups = 0;
  double *l_rect = nullptr, *l_new_rect = nullptr, *l_se = nullptr, *l_val = nullptr;
  uint32_t *l_nn = nullptr, *l_depth = nullptr, *l_dead = nullptr, *l_new_leaf = nullptr;
  mcb::CellEst* l_est = nullptr;
  size_t cap_rect = 0, cap_new_rect = 0, cap_se = 0, cap_val = 0, cap_nn = 0, cap_depth = 0, cap_dead = 0,
         cap_new_leaf = 0, cap_est = 0;
};

template <class T>
cudaError_t grow_pinned(T*& p, size_t& cap, size_t need) {
  if (need <= cap && p) return cudaSuccess;
  if (p) cudaFreeHost(p);
  p = nullptr;
  cap = 0;
  const size_t n = need > 1 ? need : 1;
  cudaError_t e = cudaMallocHost(&p, sizeof(T) * n);
  if (e == cudaSuccess) cap = n;
  return e;
}

// ---- capi_plan.cpp: reference helpers, validation, descriptors, plans --------
uint64_t splitmix64(uint64_t z);
uint64_t chunk_count(uint64_t n);
bool cell_grid_size(uint32_t k, uint32_t d, uint64_t cap, uint64_t& cells);
uint32_t auto_cells_per_dim(uint32_t d, uint64_t limit);
uint32_t int_root_floor(uint64_t x, uint32_t d);
StratPlan stratified_plan(const mcb_integrand& f);
bool stratified(const mcb_integrand& f);
uint64_t trial_samples(const mcb_integrand& f);
double sample_cost(const mcb_integrand& f);
double host_eval(const mcb_integrand& f, const double* x);
std::string to_dsl(const mcb_integrand& f);
bool rect_valid(const mcb_integrand& f);
double volume(const mcb_integrand& f);
void violations_of(const mcb_integrand& f, uint32_t trials, std::vector<std::string>& out);
Prepared prepare(const mcb_integrand& f, uint64_t seed, uint32_t chunk_base, uint32_t trial_base,
                 bool tree_cells = false);
mcb_status check_device(int device);
mcb_status validate_for_run(const mcb_integrand* fns, size_t n_fns, uint32_t trials);
uint64_t blocks_per_pair(uint32_t family, uint32_t dim);
mcb_status build_host_plan(const mcb_integrand* fns, size_t n_fns, uint64_t seed, uint32_t trials,
                           uint32_t chunk_base, uint32_t trial_base, HostPlan& hp,
                           const uint32_t* chunk_bases = nullptr, const uint32_t* trial_bases = nullptr);
void prepare_programs(const HostPlan& hp, bool compile);
mcb_status enqueue_run(const HostPlan& hp, DevBuf& buf, uint32_t trials, const FnDesc* staged, bool upload,
                       cudaStream_t s);
DeviceCtx& device_ctx(int device);
mcb_status run_shard(const mcb_integrand* fns, size_t n_fns, uint64_t seed, uint32_t trials, int device,
                     mcb_trial_stats* out, const uint32_t* chunk_bases = nullptr,
                     const uint32_t* trial_bases = nullptr, TilePartial* tile_out = nullptr,
                     size_t tile_cap = 0);

// ---- capi_tree.cpp: tree rounds ----------------------------------------------
mcb_status run_cells(const std::vector<mcb::tree::CellBatch>& batches, uint64_t seed,
                     const std::vector<int>& devs);
mcb_status run_trees_on(std::vector<mcb::tree::TreeTask>& tasks, uint64_t seed, const std::vector<int>& devs);

}  // namespace capi
}  // namespace mcb
