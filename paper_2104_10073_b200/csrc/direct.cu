// direct.cu — launch side of the direct-MC kernels for sm_100a: dispatch
// table over the fused kernel instantiations (kernels.cuh, direct_*.cu), the
// tile-table expansion, the ordered combine and the test/measurement hooks.
//
// K4 k_combine: one warp per (integrand, trial) merges its chunk partials in
//    ascending chunk order (Chan, as ChunkAccum::merge, src/estimator.cpp:20-34,
//    55-73) and forms the McEstimate fields.  Deterministic: no float atomics anywhere, reduction
//    trees are fixed, so results do not depend on the GPU count or on the
//    order in which the hardware schedules CTAs.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "kernels.cuh"

namespace mcb {
namespace detail {

using dev::FnDesc;
using dev::PhiloxPrefix;
using dev::TilePartial;

// tile_fn[t] = integrand slot owning tile t (one warp per integrand).
__global__ void k_expand_tiles(const FnDesc* __restrict__ fns, uint32_t n_fns, uint32_t trials,
                               uint32_t* __restrict__ tile_fn) {
  const uint32_t fi = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  if (fi >= n_fns) return;
  const uint64_t base = fns[fi].tile_base;
  const uint64_t n = uint64_t(fns[fi].n_chunks) * trials;
  for (uint64_t t = threadIdx.x & 31; t < n; t += 32) tile_fn[base + t] = fi;
}

// Cell volume of stratified cell `cell` (runtime dim; same arithmetic as
// dev::grid_cell / the reference's grid_cell + HyperRect::volume).
// kmag (0: divide): ceil(2^32 / k), exact division of any rem < n_cells by k
// as (rem * kmag) >> 32 when n_cells * k < 2^32 (the rounding error of kmag is
// < k, so rem * error stays below 2^32); one multiply instead of a ~15-
// instruction integer division per axis.
__device__ __forceinline__ uint64_t cell_div_magic(const FnDesc& F) {
  const uint64_t k = F.strat_k;
  return k > 1 && uint64_t(F.n_cells) * k < (1ull << 32) ? ((1ull << 32) + k - 1) / k : 0;
}

__device__ double cell_volume(const FnDesc& F, uint32_t cell, uint64_t kmag = 0) {
  double w[MCB_MAX_DIM];
  uint32_t rem = cell;
  const uint32_t k = F.strat_k;
  for (int j = int(F.dim) - 1; j >= 0; --j) {
    const uint32_t q = kmag ? uint32_t((uint64_t(rem) * kmag) >> 32) : rem / k;
    const uint32_t digit = rem - q * k;
    rem = q;
    if (F.grid_bounds) {  // host-computed boundaries (same arithmetic)
      const double* b = F.grid_bounds + uint32_t(j) * (k + 1) + digit;
      w[j] = __dsub_rn(b[1], b[0]);
      continue;
    }
    const double lo = F.low[j], wd = F.width[j];
    const double cl = digit == 0 ? lo : __dadd_rn(lo, __dmul_rn(wd, __ddiv_rn(double(digit), double(k))));
    const double ch = digit + 1 == k ? F.high[j]
                                     : __dadd_rn(lo, __dmul_rn(wd, __ddiv_rn(double(digit + 1), double(k))));
    w[j] = __dsub_rn(ch, cl);
  }
  double v = 1.0;
  for (uint32_t j = 0; j < F.dim; ++j) v = __dmul_rn(v, w[j]);
  return v;
}

// HyperRect::volume of a listed cell (tree round), left to right from 1.0.
__device__ double rect_volume(const FnDesc& F, uint32_t cell) {
  const double* r = F.cell_rects + uint64_t(cell) * (2 * F.dim);
  double v = 1.0;
  for (uint32_t j = 0; j < F.dim; ++j) v = __dmul_rn(v, __dsub_rn(r[F.dim + j], r[j]));
  return v;
}

struct Accum {  // ChunkAccum (ref src/estimator.cpp:9-34): n, n_nonfinite, mean, m2
  uint64_t n = 0, nn = 0;
  double mean = 0.0, m2 = 0.0;
};

// ChunkAccum::merge (ref src/estimator.cpp:20-34) of one tile whose partial
// sums are taken about its own shift.
__device__ __forceinline__ void merge_tile(Accum& a, const TilePartial& p) {
  a.nn += p.n_nonfinite;
  if (p.n_finite == 0) return;
  const double n_b = double(p.n_finite);
  const double dev_b = __ddiv_rn(p.s1, n_b);
  const double mean_b = __dadd_rn(p.shift, dev_b);
  double m2_b = __dsub_rn(p.s2, __dmul_rn(p.s1, dev_b));
  // rounding can leave a tiny negative m2 (clamp to 0); inf - inf = NaN only
  // when the sum of squares overflowed, where Welford's m2 is +inf too
  m2_b = m2_b > 0.0 ? m2_b : (m2_b == m2_b ? 0.0 : __longlong_as_double(0x7FF0000000000000ll));
  if (a.n == 0) {
    a.n = p.n_finite;
    a.mean = mean_b;
    a.m2 = m2_b;
    return;
  }
  const double delta = __dsub_rn(mean_b, a.mean);
  const uint64_t total = a.n + p.n_finite;
  a.mean = __dadd_rn(a.mean, __dmul_rn(delta, __ddiv_rn(n_b, double(total))));
  a.m2 = __dadd_rn(a.m2, __dadd_rn(m2_b, __dmul_rn(__dmul_rn(delta, delta),
                                                    __ddiv_rn(__dmul_rn(double(a.n), n_b), double(total)))));
  a.n = total;
}

// K4: one WARP per (integrand, trial).
//  * direct: lane 0 merges the chunk partials (Chan) in ascending chunk
//    order and forms the McEstimate (reduce_chunks, src/estimator.cpp:55-73);
//  * cell-structured (stratified grid, tree round): lanes take cells
//    c = lane, lane + 32, ...; each cell's chunks merge (Chan) into the cell's
//    own direct_mc estimate.  Tree rounds store it per cell; stratified
//    cells are combined (combine_cells, src/estimator.cpp:145-159) with the
//    reference's sequential ascending-cell sums (32 cells per step, broadcast
//    lane by lane); the first dead cell (src/batch.cpp:176-180) is the
//    minimum over lanes.
__device__ __forceinline__ mcb_trial_stats cell_estimate(const FnDesc& F, const TilePartial* part, uint64_t base,
                                                         uint32_t c, Accum& a, uint64_t kmag) {
  for (uint32_t cc = 0; cc < F.cpc; ++cc) merge_tile(a, part[base + uint64_t(c) * F.cpc + cc]);
  mcb_trial_stats cs;
  const double vol = F.cell_rects ? rect_volume(F, c) : cell_volume(F, c, kmag);
  cs.value = a.n == 0 ? 0.0 : __dmul_rn(vol, a.mean);
  cs.std_error = a.n == 0 ? 0.0
                 : a.n >= 2 ? __dmul_rn(vol, __dsqrt_rn(__ddiv_rn(__ddiv_rn(a.m2, double(a.n - 1)), double(a.n))))
                            : __longlong_as_double(0x7FF0000000000000ll);
  return cs;
}

__global__ void k_combine(const FnDesc* __restrict__ fns, uint32_t n_fns, uint32_t trials,
                          const TilePartial* __restrict__ part, mcb_trial_stats* __restrict__ out) {
  const uint64_t idx = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;  // warp-uniform
  const uint32_t lane = threadIdx.x & 31;
  if (idx >= uint64_t(n_fns) * trials) return;
  const uint32_t fi = uint32_t(idx / trials), t = uint32_t(idx % trials);
  const FnDesc& F = fns[fi];
  const uint64_t base = F.tile_base + uint64_t(t) * F.n_chunks;
  mcb_trial_stats st;
  st.detail = 0;
  st.n_cells = 1;
  st.budget_exhausted = 0;
  st.max_depth = 0;
  if (F.strat_k > 0 || F.cell_rects) {
    double value = 0.0, var = 0.0;
    unsigned long long n_all = 0, nn_all = 0;
    uint32_t dead = 0xFFFFFFFFu;
    const uint64_t kmag = cell_div_magic(F);
    // a step's 32 cell estimates, read back in cell order by every lane
    // (shared-memory broadcast); a dead cell enters as (0, 0), which leaves
    // the sums unchanged — and its trial reports the dead cell, not the sums
    __shared__ double2 step[4][32];
    double2* my = step[(threadIdx.x >> 5) & 3];
    for (uint32_t c0 = 0; c0 < F.n_cells; c0 += 32) {
      const uint32_t c = c0 + lane;
      double cv = 0.0, cse2 = 0.0;
      bool live = false;
      if (c < F.n_cells) {
        Accum a;
        const mcb_trial_stats cs = cell_estimate(F, part, base, c, a, kmag);
        n_all += a.n + a.nn;
        nn_all += a.nn;
        if (F.cell_est) {  // tree round: the cell's own estimate
          CellEst ce;
          ce.value = cs.value;
          ce.std_error = cs.std_error;
          ce.n_nonfinite = uint32_t(a.nn);
          ce.status = a.n == 0 ? MCB_TRIAL_ALL_NONFINITE : MCB_TRIAL_OK;
          F.cell_est[c] = ce;
        } else if (a.n == 0) {
          dead = min(dead, c);
        } else {
          cv = cs.value;
          cse2 = __dmul_rn(cs.std_error, cs.std_error);
          live = true;
        }
      }
      if (F.cell_est) continue;
      // combine_cells order: the running sums take the cells one by one in
      // ascending order, exactly as the reference
      (void)live;
      my[lane] = make_double2(cv, cse2);
      __syncwarp();
      const uint32_t n = min(32u, F.n_cells - c0);
      for (uint32_t i = 0; i < n; ++i) {
        const double2 e = my[i];
        value = __dadd_rn(value, e.x);
        var = __dadd_rn(var, e.y);
      }
      __syncwarp();
    }
    if (F.cell_est) {
      if (lane == 0) {
        st.status = MCB_TRIAL_OK;
        st.value = st.std_error = 0.0;
        st.n_samples = st.n_nonfinite = 0;
        st.nonfinite_warning = 0;
        st.n_cells = F.n_cells;
        out[F.out_slot * trials + t] = st;
      }
      return;
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) {
      n_all += __shfl_xor_sync(0xFFFFFFFFu, n_all, m);
      nn_all += __shfl_xor_sync(0xFFFFFFFFu, nn_all, m);
    }
    dead = __reduce_min_sync(0xFFFFFFFFu, dead);
    if (lane != 0) return;
    st.n_cells = F.n_cells;
    st.n_samples = n_all;
    st.n_nonfinite = nn_all;
    st.nonfinite_warning = double(nn_all) > MCB_NONFINITE_WARN_FRACTION * double(n_all) ? 1u : 0u;
    if (dead != 0xFFFFFFFFu) {
      st.status = MCB_TRIAL_DEAD_CELL;
      st.detail = dead;
      st.value = 0.0;
      st.std_error = 0.0;
    } else {
      st.status = MCB_TRIAL_OK;
      st.value = value;
      st.std_error = __dsqrt_rn(var);
    }
    out[F.out_slot * trials + t] = st;
    return;
  }
  if (lane != 0) return;
  // reduce_chunks: ChunkAccum::merge of the chunk partials in ascending chunk
  // order (ref src/estimator.cpp:20-34,55-73); each tile's own (mean, m2)
  // about its shift, so no cancellation builds up across the chunks
  Accum a;
  for (uint32_t c = 0; c < F.n_chunks; ++c) merge_tile(a, part[base + c]);
  const uint64_t n = a.n, nb = a.nn;
  st.n_samples = n + nb;
  st.n_nonfinite = nb;
  st.nonfinite_warning = double(nb) > MCB_NONFINITE_WARN_FRACTION * double(n + nb) ? 1u : 0u;
  if (n == 0) {
    st.status = MCB_TRIAL_ALL_NONFINITE;
    st.value = 0.0;
    st.std_error = 0.0;
  } else {
    st.status = MCB_TRIAL_OK;
    st.value = __dmul_rn(F.volume, a.mean);
    if (n >= 2) {
      const double var = __ddiv_rn(a.m2, double(n - 1));
      st.std_error = __dmul_rn(F.volume, __dsqrt_rn(__ddiv_rn(var, double(n))));
    } else {
      st.std_error = __longlong_as_double(0x7FF0000000000000ll);  // +inf
    }
  }
  out[F.out_slot * trials + t] = st;
}

// ---- test hooks ----------------------------------------------------------

// sample_uniform (src/sampling.cpp:102-112): one thread per point.
__global__ void k_debug_points(uint32_t key0, uint32_t key1, uint32_t trial, uint32_t chunk,
                               uint64_t first_point, uint64_t count, uint32_t dim,
                               const double* __restrict__ low,
                               const double* __restrict__ width, double* __restrict__ out) {
  const uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= count) return;
  const PhiloxPrefix P = dev::make_prefix(key0, key1, chunk, trial);
  for (uint32_t j = 0; j < dim; ++j) {
    const uint64_t t = (first_point + p) * dim + j;
    uint32_t o[4];
    dev::philox_block(P, uint32_t(t >> 1), o);
    const double v = (t & 1) ? dev::u_scaled(o[2], o[3]) : dev::u_scaled(o[0], o[1]);
    const double u = __dmul_rn(v, dev::kTwoM64);
    out[p * dim + j] = __dadd_rn(low[j], __dmul_rn(width[j], u));
  }
}

// Philox-generation roofline probe: Philox4x32-10 blocks with nothing else
// (4 independent blocks per thread per iteration, the same philox_block_p and
// incremental round-1 products as the fused kernel, outputs XOR-folded so
// nothing is dead code).  On B200 the IMAD.WIDE multiplies of Philox run on
// the FP64 pipe, which also executes the integrand's FP64 work, so this is
// the ceiling for any sampler that must produce these exact streams.
__global__ void __launch_bounds__(256) k_philox_probe(const uint32_t* __restrict__ key,
                                                      uint32_t* sink, int iters) {
  const PhiloxPrefix P = dev::make_prefix(key[0], key[1], blockIdx.x & 15u, blockIdx.x >> 4);
  uint64_t pbase = uint64_t(dev::kM0) * uint64_t(threadIdx.x * 4u);
  constexpr uint64_t kStep = uint64_t(dev::kM0) * 1024u;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t o[4];
      dev::philox_block_p(P, pbase + uint64_t(i) * dev::kM0, o);
      acc ^= o[0] ^ o[1] ^ o[2] ^ o[3];
    }
    pbase += kStep;
  }
  if (acc == 0x12345678u) sink[blockIdx.x] = acc;
}

// ---- dispatch -------------------------------------------------------------

static const Table& table() {
  static const Table t = [] {
    Table x;
    register_harmonic(x);
    register_harmonic_vec(x);
    register_abs(x);
    return x;
  }();
  return t;
}

static const Entry* entry(int family, int dim, int variant) {
  if (family < 0 || family > 3 || dim < 1 || dim > int(MCB_MAX_DIM) || variant < 0 ||
      variant >= kNumVariants)
    return nullptr;
  const Entry* e = &table().e[family][dim][variant];
  return e->direct ? e : nullptr;
}

bool variant_supported(int family, int dim, int variant) {
  return entry(family, dim, variant) != nullptr;
}

cudaError_t launch_direct_group(const GroupLaunch& g, const FnDesc* fns, const uint32_t* tile_fn,
                                TilePartial* part, cudaStream_t s) {
  const Entry* e = entry(g.family, g.dim, g.variant);
  if (!e) return cudaErrorInvalidValue;
  const uint64_t per_cta = tiles_per_cta(g.variant);
  const uint32_t threads = (g.variant & kLaneCell) ? kLaneAlign : kThreads;
  const uint64_t n_ctas = g.n_tiles / per_cta;
  const uint64_t kMaxGrid = 0x7FFFFFF8ull;
  for (uint64_t off = 0; off < n_ctas; off += kMaxGrid) {
    const uint64_t n = n_ctas - off < kMaxGrid ? n_ctas - off : kMaxGrid;
    e->direct<<<dim3(uint32_t(n)), dim3(threads), 0, s>>>(fns, tile_fn, g.tile0 + off * per_cta, part);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
  }
  return cudaSuccess;
}

cudaError_t launch_expand_tiles(const FnDesc* fns, uint32_t n_fns, uint32_t trials,
                                uint32_t* tile_fn, cudaStream_t s) {
  if (n_fns == 0) return cudaSuccess;
  const uint32_t warps = 8;
  k_expand_tiles<<<(n_fns + warps - 1) / warps, warps * 32, 0, s>>>(fns, n_fns, trials, tile_fn);
  return cudaGetLastError();
}

cudaError_t launch_combine(const FnDesc* fns, uint32_t n_fns, uint32_t trials,
                           const TilePartial* part, mcb_trial_stats* out, cudaStream_t s) {
  const uint64_t n = uint64_t(n_fns) * trials;
  if (n == 0) return cudaSuccess;
  k_combine<<<uint32_t((n + 3) / 4), 128, 0, s>>>(fns, n_fns, trials, part, out);  // a warp per (fn, trial)
  return cudaGetLastError();
}

cudaError_t launch_debug_points(uint32_t key0, uint32_t key1, uint32_t trial, uint32_t chunk,
                                uint64_t first_point, uint64_t count, uint32_t dim,
                                const double* low, const double* width, double* out,
                                cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  k_debug_points<<<uint32_t((count + 127) / 128), 128, 0, s>>>(key0, key1, trial, chunk,
                                                               first_point, count, dim, low,
                                                               width, out);
  return cudaGetLastError();
}

cudaError_t launch_debug_eval_impl(int family, int dim, int variant, const FnDesc* fn,
                                   uint32_t trial, uint32_t chunk, uint32_t first_pair,
                                   uint32_t n_pairs, double* out, cudaStream_t s) {
  const Entry* e = entry(family, dim, variant);
  if (!e) return cudaErrorInvalidValue;
  if (n_pairs == 0) return cudaSuccess;
  e->eval<<<(n_pairs + 127) / 128, 128, 0, s>>>(fn, trial, chunk, first_pair, n_pairs, out);
  return cudaGetLastError();
}

cudaError_t launch_philox_probe(const uint32_t* key, uint32_t* sink, int n_ctas, int iters,
                               cudaStream_t s) {
  k_philox_probe<<<n_ctas, 256, 0, s>>>(key, sink, iters);
  return cudaGetLastError();
}

}  // namespace detail
}  // namespace mcb
