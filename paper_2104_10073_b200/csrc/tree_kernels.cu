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

// Left-to-right double sum of g(0) + g(1) + ... + g(n-1) across a warp: the
// lanes load 32 terms at a time (coalesced) and every lane runs the same
// ordered chain over the shuffled terms — the reference's summation order,
// bit for bit, with the loads off the dependency chain.
template <class G>
__device__ __forceinline__ double warp_ordered_sum(uint32_t n, G g) {
  const uint32_t lane = threadIdx.x & 31;
  double acc = 0.0;
  double v = lane < n ? g(lane) : 0.0;
  for (uint32_t base = 0; base < n; base += 32) {
    const double next = base + 32 + lane < n ? g(base + 32 + lane) : 0.0;  // in flight during the chain
    const uint32_t m = min(32u, n - base);
#pragma unroll
    for (uint32_t j = 0; j < 32; ++j) {  // unrolled: the shuffles run ahead of the add chain
      const double x = __shfl_sync(0xffffffffu, v, j);
      if (j < m) acc = __dadd_rn(acc, x);
    }
    v = next;
  }
  return acc;
}

__device__ __forceinline__ uint32_t warp_of_tree() { return (blockIdx.x * blockDim.x + threadIdx.x) >> 5; }

// One refinement step per active tree (the `while (!exhausted)` body,
// src/estimator.cpp:265-297), a warp per tree: selection over the current
// leaves (mean and sd of the std_errors in leaf order), then the splits in
// leaf order while the budget allows; each split replaces leaf i by its lower
// half and appends the upper half, and both halves become this round's new
// cells (chunk keys next_chunk, next_chunk + cpc, ...).
//
// The sequential loop is restated lane-parallel: leaf i's selection test
// reads only leaf i (splits write leaf i and leaves >= n), so every leaf is
// tested at once; the k-th selected leaf (k = its rank in leaf order) passes
// the budget check iff used + 2*spc*(k+1) <= budget and the chunk-range check
// iff next_chunk + 2*cpc*(k+1) <= 2^32, so the first k that fails either
// check ends the round exactly where the sequential loop would (budget check
// first), and every lane whose rank is below it performs its own split into
// leaf n + k and new-cell slots 2k, 2k+1.
__global__ void k_tree_select(const TreeConst* __restrict__ tc, TreeState* __restrict__ ts, Leaves L,
                              uint32_t n_trees) {
  const uint32_t t = warp_of_tree(), lane = threadIdx.x & 31;
  if (t >= n_trees) return;
  TreeState st = ts[t];
  const TreeConst c = tc[t];
  st.n_new = 0;
  if (!st.active) {
    if (lane == 0) ts[t] = st;
    return;
  }
  const uint64_t off = c.leaf_off;
  const uint32_t n = st.n_leaves, D = c.dim;
  const double* se = L.se + off;
  double mean_err = warp_ordered_sum(n, [&](uint32_t i) { return se[i]; });
  mean_err = __ddiv_rn(mean_err, double(n));
  const double ss = warp_ordered_sum(n, [&](uint32_t i) {
    const double dlt = __dsub_rn(se[i], mean_err);
    return __dmul_rn(dlt, dlt);
  });
  const double sd = n > 1 ? __dsqrt_rn(__ddiv_rn(ss, double(n - 1))) : 0.0;
  const double threshold = __dadd_rn(mean_err, __dmul_rn(c.sigma, sd));
  // splits allowed by the budget (kb) and by the chunk range (kc)
  const uint64_t step_s = 2ull * c.spc, step_c = 2ull * c.cpc;
  const uint64_t kb = st.used <= c.budget ? (c.budget - st.used) / step_s : 0;
  const uint64_t kc = st.next_chunk <= (1ull << 32) ? ((1ull << 32) - st.next_chunk) / step_c : 0;
  const uint64_t lim = min(kb, kc);
  uint64_t rank = 0;  // selected leaves so far
  bool any = false;
  for (uint32_t base = 0; base < n; base += 32) {
    const uint32_t i = base + lane;
    const double e = i < n ? se[i] : 0.0;
    const bool sel = i < n && L.depth[off + i] < c.max_depth && e > 0 && e > threshold;
    const uint32_t mask = __ballot_sync(0xffffffffu, sel);
    if (!mask) continue;
    any = true;
    const uint64_t k = rank + __popc(mask & ((1u << lane) - 1u));
    if (sel && k < lim) {  // split_longest_edge (src/estimator.cpp:192-210)
      double* ri = L.rect + c.rect_off + uint64_t(2 * D) * i;
      const uint64_t h = uint64_t(n) + k;
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
      double* s0 = L.new_rect + c.rect_off + uint64_t(2 * D) * (2 * k);
      for (uint32_t j = 0; j < 2 * D; ++j) s0[j] = ri[j];
      for (uint32_t j = 0; j < 2 * D; ++j) s0[2 * D + j] = rh[j];
      L.new_leaf[off + 2 * k] = i;
      L.new_leaf[off + 2 * k + 1] = uint32_t(h);
    }
    rank += __popc(mask);
    if (rank > lim) break;
  }
  const uint64_t splits = min(rank, lim);
  st.chunk0 = st.next_chunk;
  st.n_leaves = n + uint32_t(splits);
  st.next_chunk += step_c * splits;
  st.used += step_s * splits;
  st.n_new = uint32_t(2 * splits);
  if (rank > lim) {
    if (kb <= kc) {
      st.exhausted = 1;
    } else {  // UniformStream throws (src/sampling.cpp:80-81)
      st.fail = MCB_TRIAL_CHUNK_RANGE;
      st.active = 0;
      st.n_new = 0;
    }
  }
  if (!any || st.exhausted) st.active = 0;  // nothing selected, or the while condition
  if (lane == 0) ts[t] = st;
}

// Tile ranges of this round's cells: per launch group (trees are sorted by
// group), groups in order, warp-tile groups 8-aligned; every tree's
// descriptor gets its cells, tiles and chunk base.  One CTA, two block scans
// over the trees: the first finds each group's unaligned tile offset (the
// prefix at its first tree) and so the group sizes and aligned starts, the
// second writes the descriptors.
constexpr int kLayoutThreads = 1024;
constexpr uint32_t kMaxGroups = 256;

__global__ void __launch_bounds__(kLayoutThreads)
    k_tree_layout(const TreeConst* __restrict__ tc, const TreeState* __restrict__ ts, FnDesc* __restrict__ fns,
                  Leaves L, uint32_t n_trees, uint64_t* __restrict__ group_tiles, uint32_t n_groups) {
  using Scan = cub::BlockScan<unsigned long long, kLayoutThreads>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long first[kMaxGroups + 1], start[kMaxGroups];
  __shared__ unsigned long long carry;
  constexpr unsigned long long kNone = ~0ull;
  auto tiles_of = [&](uint32_t t) -> unsigned long long {
    const TreeConst& c = tc[t];
    unsigned long long n = uint64_t(ts[t].n_new) * c.cpc;
    if (c.warp_tiles) n = (n + kTileAlign - 1) / kTileAlign * kTileAlign;
    return n;
  };
  for (uint32_t g = threadIdx.x; g <= n_groups; g += kLayoutThreads) first[g] = kNone;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < n_trees; base += kLayoutThreads) {
    const uint32_t t = base + threadIdx.x;
    const unsigned long long mine = t < n_trees ? tiles_of(t) : 0ull;
    unsigned long long prefix, sum;
    Scan(tmp).ExclusiveSum(mine, prefix, sum);
    if (t < n_trees && (t == 0 || tc[t].group != tc[t - 1].group)) first[tc[t].group] = carry + prefix;
    __syncthreads();
    if (threadIdx.x == 0) carry += sum;
    __syncthreads();
  }
  if (threadIdx.x == 0) {  // group starts: in order, warp-tile groups aligned
    first[n_groups] = carry;
    for (uint32_t g = n_groups; g-- > 0;)
      if (first[g] == kNone) first[g] = first[g + 1];  // a group without trees: empty
    unsigned long long pos = 0;
    for (uint32_t g = 0; g < n_groups; ++g) {
      pos = (pos + kTileAlign - 1) / kTileAlign * kTileAlign;
      start[g] = pos;
      pos += first[g + 1] - first[g];
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
      f.tile_base = start[c.group] + (prefix - first[c.group]);
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
    group_tiles[2 * g + 1] = first[g + 1] - first[g];
  }
}

// The round's estimates into the leaves; a cell without a finite sample is
// a dead leaf (value 0, std_error 0, all spc samples non-finite).  A warp
// per tree.
__global__ void k_tree_scatter(const TreeConst* __restrict__ tc, const TreeState* __restrict__ ts, Leaves L,
                               uint32_t n_trees) {
  const uint32_t t = warp_of_tree();
  if (t >= n_trees) return;
  const TreeConst c = tc[t];
  const uint32_t n_new = ts[t].n_new;
  for (uint32_t k = threadIdx.x & 31; k < n_new; k += 32) {
    const uint64_t leaf = c.leaf_off + L.new_leaf[c.leaf_off + k];
    const CellEst e = L.est[c.leaf_off + k];
    const bool ok = e.status == MCB_TRIAL_OK;
    L.se[leaf] = ok ? e.std_error : 0.0;
    L.val[leaf] = ok ? e.value : 0.0;
    L.nn[leaf] = ok ? e.n_nonfinite : c.spc;
    L.dead[leaf] = ok ? 0u : 1u;
  }
}

// combine_cells over the leaves in order (src/estimator.cpp:145-159, :299-306),
// a warp per tree.
__global__ void k_tree_finish(const TreeConst* __restrict__ tc, const TreeState* __restrict__ ts, Leaves L,
                              uint32_t n_trees, mcb_trial_stats* __restrict__ out) {
  const uint32_t t = warp_of_tree(), lane = threadIdx.x & 31;
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
    if (lane == 0) out[t] = o;
    return;
  }
  const uint32_t n = st.n_leaves;
  const double* val = L.val + c.leaf_off;
  const double* se = L.se + c.leaf_off;
  const double value = warp_ordered_sum(n, [&](uint32_t i) { return val[i]; });
  const double var = warp_ordered_sum(n, [&](uint32_t i) { return __dmul_rn(se[i], se[i]); });
  unsigned long long n_nonfinite = 0;
  uint32_t depth = 0;
  for (uint32_t i = lane; i < n; i += 32) {
    n_nonfinite += L.nn[c.leaf_off + i];
    depth = max(depth, L.depth[c.leaf_off + i]);
  }
  for (int s = 16; s > 0; s >>= 1) {
    n_nonfinite += __shfl_xor_sync(0xffffffffu, n_nonfinite, s);
    depth = max(depth, __shfl_xor_sync(0xffffffffu, depth, s));
  }
  const uint64_t n_samples = uint64_t(n) * c.spc;
  o.n_samples = n_samples;
  o.n_nonfinite = n_nonfinite;
  o.n_cells = n;
  o.max_depth = depth;
  o.budget_exhausted = st.exhausted;
  if (n_samples == n_nonfinite) {
    o.status = MCB_TRIAL_ALL_NONFINITE;
  } else {
    o.value = value;
    o.std_error = __dsqrt_rn(var);
    o.nonfinite_warning = double(n_nonfinite) > MCB_NONFINITE_WARN_FRACTION * double(n_samples) ? 1u : 0u;
  }
  if (lane == 0) out[t] = o;
}

constexpr uint32_t kTreeWarpThreads = 256;  // 8 trees per CTA

inline uint32_t tree_warp_blocks(uint32_t n_trees) {
  return (n_trees + kTreeWarpThreads / 32 - 1) / (kTreeWarpThreads / 32);
}

cudaError_t launch_tree_init(const TreeConst* tc, const TreeState* ts, Leaves L, const double* packed,
                             uint32_t n_trees, cudaStream_t s) {
  if (!n_trees) return cudaSuccess;
  k_tree_init<<<n_trees, 128, 0, s>>>(tc, ts, L, packed, n_trees);
  return cudaGetLastError();
}

cudaError_t launch_tree_select(const TreeConst* tc, TreeState* ts, Leaves L, uint32_t n_trees, cudaStream_t s) {
  if (!n_trees) return cudaSuccess;
  k_tree_select<<<tree_warp_blocks(n_trees), kTreeWarpThreads, 0, s>>>(tc, ts, L, n_trees);
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
  k_tree_scatter<<<tree_warp_blocks(n_trees), kTreeWarpThreads, 0, s>>>(tc, ts, L, n_trees);
  return cudaGetLastError();
}

cudaError_t launch_tree_finish(const TreeConst* tc, const TreeState* ts, Leaves L, uint32_t n_trees,
                               mcb_trial_stats* out, cudaStream_t s) {
  if (!n_trees) return cudaSuccess;
  k_tree_finish<<<tree_warp_blocks(n_trees), kTreeWarpThreads, 0, s>>>(tc, ts, L, n_trees, out);
  return cudaGetLastError();
}

}  // namespace detail
}  // namespace mcb
