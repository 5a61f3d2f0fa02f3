// direct.cu — the fused direct-MC kernels for sm_100a.
//
// K3 k_direct<FAM,D,V>: one CTA per tile = (integrand, trial, chunk) unit of
//    <= 65536 samples (reference task, src/batch.cpp:235-253).  Each thread
//    walks sample pairs: Philox in registers (K1) -> FP64 family value (K2)
//    -> running sums of g = f - shift and g^2 -> warp butterfly -> fixed
//    CTA tree -> one TilePartial.  Replaces accumulate_chunk
//    (src/estimator.cpp:36-49) + ChunkAccum::add (:9-18).  No global memory
//    traffic besides the descriptor read and a 24-byte partial per tile.
// K4 k_combine: one thread per (integrand, trial) sums its chunk partials in
//    ascending chunk order (src/estimator.cpp:55-73 ordering) and forms the
//    McEstimate fields.  Deterministic: no float atomics anywhere, reduction
//    trees are fixed, so results do not depend on the GPU count or on the
//    order in which the hardware schedules CTAs.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "mcb_internal.hpp"

namespace mcb {
namespace detail {

using dev::FnDesc;
using dev::PhiloxPrefix;
using dev::TilePartial;

__constant__ dev::SinCosConsts c_sincos = MCB_SINCOS_CONSTS;

__device__ __forceinline__ bool finite64(double x) {
  // exponent != 0x7FF
  return (uint32_t(__double2hiint(x)) & 0x7FF00000u) != 0x7FF00000u;
}

__device__ __forceinline__ double shfl_xor_d(double v, int m) {
  return __shfl_xor_sync(0xFFFFFFFFu, v, m);
}

template <int FAM, int D, int V>
__global__ void __launch_bounds__(kThreads) k_direct(const FnDesc* __restrict__ fns,
                                                     const uint32_t* __restrict__ tile_fn,
                                                     uint64_t tile0,
                                                     TilePartial* __restrict__ part) {
  constexpr bool UNIT_DOM = (V & kUnitDomain) != 0;
  constexpr bool UNIT_COEF = (V & kUnitCoef) != 0;
  constexpr bool CHECK = (V & kSafe) != 0;

  const uint64_t tile = tile0 + blockIdx.x;
  const uint32_t fi = __ldg(tile_fn + tile);
  const FnDesc& F = fns[fi];
  const FnDesc f = F;  // uniform; ptxas keeps only the fields this variant reads

  const uint32_t rem = uint32_t(tile - f.tile_base);
  const uint32_t trial = rem / f.n_chunks;
  const uint32_t chunk = rem - trial * f.n_chunks;
  const uint32_t count =
      (chunk + 1 == f.n_chunks) ? uint32_t(f.n_samples - uint64_t(chunk) * MCB_CHUNK_SIZE)
                                : MCB_CHUNK_SIZE;
  const uint32_t pairs = (count + 1) >> 1;
  const PhiloxPrefix P = dev::make_prefix(f.key0, f.key1, f.chunk_base + chunk, f.trial_base + trial);
  __shared__ dev::QuadCoef tab[4];
  if (threadIdx.x < 4) tab[threadIdx.x] = dev::quad_coef(f.a, f.b, int(threadIdx.x));
  __syncthreads();

  double s1 = 0.0, s2 = 0.0;
  uint32_t nbad = 0;
  // Software pipeline: iteration i folds pair q_i's transcendental part
  // (FP64-heavy) while generating pair q_{i+1} (integer-heavy), so the two
  // independent streams interleave in one instruction window.  The last
  // iteration generates one pair past the chunk; it is discarded.
  const uint32_t iters = threadIdx.x < pairs ? (pairs - threadIdx.x + kThreads - 1) / kThreads : 0u;
  double a0, a1;
  dev::gen_pair<FAM, D, UNIT_DOM, CHECK>(f, P, threadIdx.x, a0, a1);
  for (uint32_t it = 0; it < iters; ++it) {
    const uint32_t q = threadIdx.x + it * kThreads;
    double b0, b1;
    dev::gen_pair<FAM, D, UNIT_DOM, CHECK>(f, P, q + kThreads, b0, b1);
    const double f0 = dev::finish<FAM, UNIT_COEF, CHECK>(f, c_sincos, tab, a0);
    const double f1 = dev::finish<FAM, UNIT_COEF, CHECK>(f, c_sincos, tab, a1);
    a0 = b0;
    a1 = b1;
    const bool has1 = 2 * q + 1 < count;
    double g0 = __dsub_rn(f0, f.shift);
    double g1 = __dsub_rn(f1, f.shift);
    if (CHECK) {
      const bool ok0 = finite64(f0), ok1 = finite64(f1) && has1;
      nbad += (ok0 ? 0u : 1u) + ((has1 && !ok1) ? 1u : 0u);
      g0 = ok0 ? g0 : 0.0;
      g1 = ok1 ? g1 : 0.0;
    } else {
      g1 = has1 ? g1 : 0.0;
    }
    s1 = __dadd_rn(s1, g0);
    s2 = fma(g0, g0, s2);
    s1 = __dadd_rn(s1, g1);
    s2 = fma(g1, g1, s2);
  }

  // fixed-shape reduction: warp butterfly, then warps 0..7 in order
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    s1 = __dadd_rn(s1, shfl_xor_d(s1, m));
    s2 = __dadd_rn(s2, shfl_xor_d(s2, m));
    if (CHECK) nbad += __shfl_xor_sync(0xFFFFFFFFu, nbad, m);
  }
  __shared__ double sh1[kThreads / 32], sh2[kThreads / 32];
  __shared__ uint32_t shb[kThreads / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sh1[warp] = s1;
    sh2[warp] = s2;
    shb[warp] = nbad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t1 = sh1[0], t2 = sh2[0];
    uint32_t tb = shb[0];
#pragma unroll
    for (int w = 1; w < kThreads / 32; ++w) {
      t1 = __dadd_rn(t1, sh1[w]);
      t2 = __dadd_rn(t2, sh2[w]);
      tb += shb[w];
    }
    TilePartial p;
    p.s1 = t1;
    p.s2 = t2;
    p.n_nonfinite = CHECK ? tb : 0u;
    p.n_finite = count - p.n_nonfinite;
    part[tile] = p;
  }
}

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

// Family values of the pairs [first_pair, first_pair + n_pairs) of one chunk,
// through exactly the eval_pair instantiation the fused kernel uses.
template <int FAM, int D, int V>
__global__ void k_debug_eval(const FnDesc* __restrict__ fn, uint32_t trial, uint32_t chunk,
                             uint32_t first_pair, uint32_t n_pairs, double* __restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const FnDesc f = *fn;
  const PhiloxPrefix P = dev::make_prefix(f.key0, f.key1, chunk, trial);
  __shared__ dev::QuadCoef tab[4];
  if (threadIdx.x < 4) tab[threadIdx.x] = dev::quad_coef(f.a, f.b, int(threadIdx.x));
  __syncthreads();
  if (i >= n_pairs) return;
  double f0, f1;
  dev::eval_pair<FAM, D, (V & kUnitDomain) != 0, (V & kUnitCoef) != 0, (V & kSafe) != 0>(
      f, c_sincos, tab, P, first_pair + i, f0, f1);
  out[2 * uint64_t(i)] = f0;
  out[2 * uint64_t(i) + 1] = f1;
}

// Integer-multiply pipe probe: 16 independent 32x32->64 multiply chains per
// thread (the same mulhilo as Philox, i.e. IMAD.WIDE.U32 by a constant),
// folded with one LOP3 each like a Philox round.  The result feeds `sink`
// so nothing is dead code.
__global__ void __launch_bounds__(256) k_mul_probe(uint32_t* sink, int iters) {
  uint32_t x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 2654435761u + i * 40503u + blockIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      uint32_t hi, lo;
      dev::mulhilo(i & 1 ? dev::kM1 : dev::kM0, x[i], hi, lo);
      x[i] = hi ^ lo;
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc ^= x[i];
  if (acc == 0x12345678u) sink[blockIdx.x] = acc;
}

// ---- dispatch -------------------------------------------------------------

using DirectFn = void (*)(const FnDesc*, const uint32_t*, uint64_t, TilePartial*);
using EvalFn = void (*)(const FnDesc*, uint32_t, uint32_t, uint32_t, uint32_t, double*);

struct Entry {
  DirectFn direct = nullptr;
  EvalFn eval = nullptr;
};

struct Table {
  Entry e[4][MCB_MAX_DIM + 1][8];
  template <int FAM, int D, int V>
  void put() {
    e[FAM][D][V].direct = k_direct<FAM, D, V>;
    e[FAM][D][V].eval = k_debug_eval<FAM, D, V>;
  }
  template <int FAM, int D>
  void put_common() {
    put<FAM, D, 0>();
    put<FAM, D, kUnitDomain>();
    put<FAM, D, kSafe>();
  }
  template <int D>
  void put_dim() {
    put_common<MCB_FAMILY_HARMONIC, D>();
    put<MCB_FAMILY_HARMONIC, D, kUnitCoef>();
    put<MCB_FAMILY_HARMONIC, D, kUnitCoef | kUnitDomain>();
    put_common<MCB_FAMILY_HARMONIC_VEC, D>();
    if constexpr (D >= 2) put_common<MCB_FAMILY_ABS2, D>();
    if constexpr (D >= 3) put_common<MCB_FAMILY_ABS3, D>();
  }
  Table() {
    put_dim<1>();
    put_dim<2>();
    put_dim<3>();
    put_dim<4>();
    put_dim<5>();
    put_dim<6>();
    put_dim<7>();
    put_dim<8>();
  }
};

static const Table& table() {
  static const Table t;
  return t;
}

static const Entry* entry(int family, int dim, int variant) {
  if (family < 0 || family > 3 || dim < 1 || dim > int(MCB_MAX_DIM) || variant < 0 ||
      variant > 7)
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

cudaError_t launch_mul_probe(uint32_t* sink, int n_ctas, int iters, cudaStream_t s) {
  k_mul_probe<<<n_ctas, 256, 0, s>>>(sink, iters);
  return cudaGetLastError();
}

}  // namespace detail
}  // namespace mcb
