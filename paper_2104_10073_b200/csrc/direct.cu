// direct.cu — launch side of the direct-MC kernels for sm_100a: dispatch
// table over the fused kernel instantiations (kernels.cuh, direct_*.cu), the
// tile-table expansion, the ordered combine and the test/measurement hooks.
//
// K4 k_combine: one thread per (integrand, trial) sums its chunk partials in
//    ascending chunk order (src/estimator.cpp:55-73 ordering) and forms the
//    McEstimate fields.  Deterministic: no float atomics anywhere, reduction
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

// K4: ascending-chunk combine per (integrand, trial) and McEstimate fields
// (reduce_chunks, src/estimator.cpp:55-73).
__global__ void k_combine(const FnDesc* __restrict__ fns, uint32_t n_fns, uint32_t trials,
                          const TilePartial* __restrict__ part, mcb_trial_stats* __restrict__ out) {
  const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= uint64_t(n_fns) * trials) return;
  const uint32_t fi = uint32_t(idx / trials), t = uint32_t(idx % trials);
  const FnDesc& F = fns[fi];
  const uint64_t base = F.tile_base + uint64_t(t) * F.n_chunks;
  double s1 = 0.0, s2 = 0.0;
  uint64_t n = 0, nb = 0;
  for (uint32_t c = 0; c < F.n_chunks; ++c) {
    const TilePartial p = part[base + c];
    s1 = __dadd_rn(s1, p.s1);
    s2 = __dadd_rn(s2, p.s2);
    n += p.n_finite;
    nb += p.n_nonfinite;
  }
  mcb_trial_stats st;
  st.n_samples = n + nb;
  st.n_nonfinite = nb;
  st.nonfinite_warning = double(nb) > MCB_NONFINITE_WARN_FRACTION * double(n + nb) ? 1u : 0u;
  if (n == 0) {
    st.status = MCB_TRIAL_ALL_NONFINITE;
    st.value = 0.0;
    st.std_error = 0.0;
  } else {
    st.status = MCB_TRIAL_OK;
    const double dn = double(n);
    const double dev_mean = __ddiv_rn(s1, dn);
    const double mean = __dadd_rn(F.shift, dev_mean);
    st.value = __dmul_rn(F.volume, mean);
    if (n >= 2) {
      double m2 = __dsub_rn(s2, __dmul_rn(s1, dev_mean));
      m2 = m2 > 0.0 ? m2 : 0.0;
      const double var = __ddiv_rn(m2, double(n - 1));
      st.std_error = __dmul_rn(F.volume, __dsqrt_rn(__ddiv_rn(var, dn)));
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
      variant > 15)
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
  const uint64_t kMaxGrid = 0x7FFFFFFFull;
  for (uint64_t off = 0; off < g.n_tiles; off += kMaxGrid) {
    const uint64_t n = g.n_tiles - off < kMaxGrid ? g.n_tiles - off : kMaxGrid;
    e->direct<<<dim3(uint32_t(n)), dim3(kThreads), 0, s>>>(fns, tile_fn, g.tile0 + off, part);
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
  k_combine<<<uint32_t((n + 127) / 128), 128, 0, s>>>(fns, n_fns, trials, part, out);
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
