// tree_kernels.cu — the device-resident tree rounds (see tree_device.cuh).
#include <cuda_runtime.h>

#include <cub/block/block_scan.cuh>

#include "mcb_internal.hpp"
#include "tree_device.cuh"

namespace mcb {
namespace detail {

using dev::FnDesc;
using tdev::Leaves;
using tdev::TreeConst;
using tdev::TreeState;

// First pass: each tree's grid (packed, n_leaves cells) into its leaf and
// round-0 cell storage; new cells = the leaves in order; depth 0.  A CTA per tree.
__global__ void k_tree_init(const TreeConst* __restrict__ tc, const TreeState* __restrict__ ts, Leaves L,
                            const double* __restrict__ packed, uint32_t n_trees) {
  const uint32_t t = blockIdx.x;
  if (t >= n_trees) return;
  const TreeConst c = tc[t];
  const uint32_t n = ts[t].n_leaves;
  const uint64_t nd = uint64_t(n) * 2 * c.dim;
  for (uint64_t i = threadIdx.x; i < nd; i += blockDim.x) {
    const double v = packed[c.init_off + i];
    L.rect[c.rect_off + i] = v;
    L.new_rect[c.rect_off + i] = v;
  }
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    L.new_leaf[c.leaf_off + i] = i;
    L.depth[c.leaf_off + i] = 0;
  }
}

// One refinement step per active tree (the `while (!exhausted)` body,
// src/estimator.cpp:265-297): selection over the current leaves, then the
// splits in leaf order while the budget allows; each split replaces leaf i
// by its lower half and appends the upper half, and both halves become this
// round's new cells (chunk keys next_chunk, next_chunk + cpc, ...).
__global__ void k_tree_select(const TreeConst* __restrict__ tc, TreeState* __restrict__ ts, Leaves L,
                              uint32_t n_trees) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_trees) return;
  TreeState st = ts[t];
  const TreeConst c = tc[t];
  st.n_new = 0;
  if (!st.active) {
    ts[t] = st;
    return;
  }
  const uint64_t off = c.leaf_off;
  const uint32_t n = st.n_leaves, D = c.dim;
  const double* se = L.se + off;
  double mean_err = 0.0;
  for (uint32_t i = 0; i < n; ++i) mean_err = __dadd_rn(mean_err, se[i]);
  mean_err = __ddiv_rn(mean_err, double(n));
  double ss = 0.0;
  for (uint32_t i = 0; i < n; ++i) {
    const double dlt = __dsub_rn(se[i], mean_err);
    ss = __dadd_rn(ss, __dmul_rn(dlt, dlt));
  }
  const double sd = n > 1 ? __dsqrt_rn(__ddiv_rn(ss, double(n - 1))) : 0.0;
  const double threshold = __dadd_rn(mean_err, __dmul_rn(c.sigma, sd));
  st.chunk0 = st.next_chunk;
  uint32_t n_new = 0;
  bool any = false;
  for (uint32_t i = 0; i < n; ++i) {
    const double e = se[i];
    if (!(L.depth[off + i] < c.max_depth && e > 0 && e > threshold)) continue;
    any = true;
    if (st.used + 2ull * c.spc > c.budget) {
      st.exhausted = 1;
      break;
    }
    if (st.next_chunk + 2ull * c.cpc - 1 > 0xFFFFFFFFull) {  // UniformStream throws (src/sampling.cpp:80-81)
      st.fail = MCB_TRIAL_CHUNK_RANGE;
      st.active = 0;
      st.n_new = 0;
      ts[t] = st;
      return;
    }
    // split_longest_edge (src/estimator.cpp:192-210)
    double* ri = L.rect + c.rect_off + uint64_t(2 * D) * i;
    const uint32_t h = st.n_leaves;
    double* rh = L.rect + c.rect_off + uint64_t(2 * D) * h;
    uint32_t axis = 0;
    double best = -1.0;
    for (uint32_t j = 0; j < D; ++j) {
      const double w = __dsub_rn(ri[D + j], ri[j]);
      if (w > best) {
        best = w;
        axis = j;
      }
    }
    const double mid = __dadd_rn(ri[axis], __dmul_rn(0.5, __dsub_rn(ri[D + axis], ri[axis])));
    for (uint32_t j = 0; j < 2 * D; ++j) rh[j] = ri[j];
    ri[D + axis] = mid;  // the lower half replaces leaf i
    rh[axis] = mid;      // the upper half is appended
    const uint32_t child = L.depth[off + i] + 1;
    L.depth[off + i] = child;
    L.depth[off + h] = child;
    double* s0 = L.new_rect + c.rect_off + uint64_t(2 * D) * n_new;
    for (uint32_t j = 0; j < 2 * D; ++j) s0[j] = ri[j];
    for (uint32_t j = 0; j < 2 * D; ++j) s0[2 * D + j] = rh[j];
    L.new_leaf[off + n_new] = i;
    L.new_leaf[off + n_new + 1] = h;
    n_new += 2;
    st.n_leaves = h + 1;
    st.next_chunk += 2ull * c.cpc;
    st.used += 2ull * c.spc;
  }
  if (!any || st.exhausted) st.active = 0;  // nothing selected, or the while condition
  st.n_new = n_new;
  ts[t] = st;
}

// Tile ranges of this round's cells: per launch group (trees are sorted by
// group), groups in order, warp-tile groups 8-aligned; every tree's
// descriptor gets its cells, tiles and chunk base.  One CTA.
constexpr int kLayoutThreads = 1024;
constexpr uint32_t kMaxGroups = 256;

__global__ void __launch_bounds__(kLayoutThreads)
    k_tree_layout(const TreeConst* __restrict__ tc, const TreeState* __restrict__ ts, FnDesc* __restrict__ fns,
                  Leaves L, uint32_t n_trees, uint64_t* __restrict__ group_tiles, uint32_t n_groups) {
  using Scan = cub::BlockScan<unsigned long long, kLayoutThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long total[kMaxGroups], start[kMaxGroups], before[kMaxGroups];
  __shared__ unsigned long long carry;
  auto tiles_of = [&](uint32_t t) -> unsigned long long {
    const TreeConst& c = tc[t];
    unsigned long long n = uint64_t(ts[t].n_new) * c.cpc;
    if (c.warp_tiles) n = (n + kTileAlign - 1) / kTileAlign * kTileAlign;
    return n;
  };
  for (uint32_t g = threadIdx.x; g < n_groups; g += kLayoutThreads) total[g] = 0;
  __syncthreads();
  for (uint32_t t = threadIdx.x; t < n_trees; t += kLayoutThreads) atomicAdd(&total[tc[t].group], tiles_of(t));
  __syncthreads();
  if (threadIdx.x == 0) {  // group starts: in order, warp-tile groups aligned
    unsigned long long pos = 0, unaligned = 0;
    for (uint32_t g = 0; g < n_groups; ++g) {
      pos = (pos + kTileAlign - 1) / kTileAlign * kTileAlign;
      start[g] = pos;
      before[g] = unaligned;
      pos += total[g];
      unaligned += total[g];
    }
    carry = 0;
  }
  __syncthreads();
  for (uint32_t base = 0; base < n_trees; base += kLayoutThreads) {
    const uint32_t t = base + threadIdx.x;
    const unsigned long long mine = t < n_trees ? tiles_of(t) : 0ull;
    unsigned long long prefix, sum;
    Scan(tmp).ExclusiveSum(mine, prefix, sum);
    prefix += carry;
    if (t < n_trees) {
      const TreeConst& c = tc[t];
      const TreeState& st = ts[t];
      FnDesc& f = fns[t];
      f.n_cells = st.n_new;
      f.n_chunks = uint32_t(mine);
      f.n_samples = uint64_t(st.n_new) * c.spc;
      f.tile_base = start[c.group] + (prefix - before[c.group]);
      f.chunk_base = uint32_t(st.chunk0);
      f.cell_rects = L.new_rect + c.rect_off;
      f.cell_est = L.est + c.leaf_off;
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += sum;
    __syncthreads();
  }
  for (uint32_t g = threadIdx.x; g < n_groups; g += kLayoutThreads) {
    group_tiles[2 * g] = start[g];
    group_tiles[2 * g + 1] = total[g];
  }
}

// The round's estimates into the leaves; a cell without a finite sample is
// a dead leaf (value 0, std_error 0, all spc samples non-finite).
__global__ void k_tree_scatter(const TreeConst* __restrict__ tc, const TreeState* __restrict__ ts, Leaves L,
                               uint32_t n_trees) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_trees) return;
  const TreeConst c = tc[t];
  const uint32_t n_new = ts[t].n_new;
  for (uint32_t k = 0; k < n_new; ++k) {
    const uint64_t leaf = c.leaf_off + L.new_leaf[c.leaf_off + k];
    const CellEst e = L.est[c.leaf_off + k];
    const bool ok = e.status == MCB_TRIAL_OK;
    L.se[leaf] = ok ? e.std_error : 0.0;
    L.val[leaf] = ok ? e.value : 0.0;
    L.nn[leaf] = ok ? e.n_nonfinite : c.spc;
    L.dead[leaf] = ok ? 0u : 1u;
  }
}

// combine_cells over the leaves in order (src/estimator.cpp:145-159, :299-306).
__global__ void k_tree_finish(const TreeConst* __restrict__ tc, const TreeState* __restrict__ ts, Leaves L,
                              uint32_t n_trees, mcb_trial_stats* __restrict__ out) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_trees) return;
  const TreeConst c = tc[t];
  const TreeState st = ts[t];
  mcb_trial_stats o;
  o.value = o.std_error = 0.0;
  o.n_samples = o.n_nonfinite = 0;
  o.status = MCB_TRIAL_OK;
  o.nonfinite_warning = 0;
  o.detail = 0;
  o.n_cells = 0;
  o.budget_exhausted = 0;
  o.max_depth = 0;
  if (st.fail) {
    o.status = st.fail;
    out[t] = o;
    return;
  }
  double value = 0.0, var = 0.0;
  uint64_t n_samples = 0, n_nonfinite = 0;
  uint32_t depth = 0;
  for (uint32_t i = 0; i < st.n_leaves; ++i) {
    const uint64_t l = c.leaf_off + i;
    value = __dadd_rn(value, L.val[l]);
    var = __dadd_rn(var, __dmul_rn(L.se[l], L.se[l]));
    n_samples += c.spc;
    n_nonfinite += L.nn[l];
    depth = max(depth, L.depth[l]);
  }
  o.n_samples = n_samples;
  o.n_nonfinite = n_nonfinite;
  o.n_cells = st.n_leaves;
  o.max_depth = depth;
  o.budget_exhausted = st.exhausted;
  if (n_samples == n_nonfinite) {
    o.status = MCB_TRIAL_ALL_NONFINITE;
  } else {
    o.value = value;
    o.std_error = __dsqrt_rn(var);
    o.nonfinite_warning = double(n_nonfinite) > MCB_NONFINITE_WARN_FRACTION * double(n_samples) ? 1u : 0u;
  }
  out[t] = o;
}

cudaError_t launch_tree_init(const TreeConst* tc, const TreeState* ts, Leaves L, const double* packed,
                             uint32_t n_trees, cudaStream_t s) {
  if (!n_trees) return cudaSuccess;
  k_tree_init<<<n_trees, 128, 0, s>>>(tc, ts, L, packed, n_trees);
  return cudaGetLastError();
}

cudaError_t launch_tree_select(const TreeConst* tc, TreeState* ts, Leaves L, uint32_t n_trees, cudaStream_t s) {
  if (!n_trees) return cudaSuccess;
  k_tree_select<<<(n_trees + 127) / 128, 128, 0, s>>>(tc, ts, L, n_trees);
  return cudaGetLastError();
}

cudaError_t launch_tree_layout(const TreeConst* tc, const TreeState* ts, FnDesc* fns, Leaves L, uint32_t n_trees,
                               uint64_t* group_tiles, uint32_t n_groups, cudaStream_t s) {
  if (n_groups > kMaxGroups) return cudaErrorInvalidValue;
  k_tree_layout<<<1, kLayoutThreads, 0, s>>>(tc, ts, fns, L, n_trees, group_tiles, n_groups);
  return cudaGetLastError();
}

cudaError_t launch_tree_scatter(const TreeConst* tc, const TreeState* ts, Leaves L, uint32_t n_trees,
                                cudaStream_t s) {
  if (!n_trees) return cudaSuccess;
  k_tree_scatter<<<(n_trees + 127) / 128, 128, 0, s>>>(tc, ts, L, n_trees);
  return cudaGetLastError();
}

cudaError_t launch_tree_finish(const TreeConst* tc, const TreeState* ts, Leaves L, uint32_t n_trees,
                               mcb_trial_stats* out, cudaStream_t s) {
  if (!n_trees) return cudaSuccess;
  k_tree_finish<<<(n_trees + 127) / 128, 128, 0, s>>>(tc, ts, L, n_trees, out);
  return cudaGetLastError();
}

}  // namespace detail
}  // namespace mcb
