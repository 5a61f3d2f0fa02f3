// jit_kernels.cuh — kernel templates for runtime-specialised DSL programs.
//
// Compiled at run time by NVRTC (csrc/jit.cpp) together with one generated
// struct per program:
//     struct P { static __device__ double eval(const double* x, const double* p); };
// whose body is the program's scheduled instruction list as straight-line
// register code — the same operations, in the same order, as the GPU
// interpreter executes (kernels_program.cu: __dadd_rn/__dsub_rn/__dmul_rn/
// __ddiv_rn, libdevice sin/cos/sincos/tan/asin/acos/atan/log/pow, dev::mcb_exp, exact
// sqrt/fabs/floor/fmin/fmax).  Sample generation, the per-thread pair loop,
// the non-finite handling and the warp/CTA reduction shapes are exactly
// those of k_program / k_program_warp with the same CTA size, so every
// TilePartial is bit-identical to the interpreter's; only the dispatch and
// the shared-memory evaluation stack are gone.
//
// Modes (the interpreter's variants): 0 direct, 1 direct on [0,1]^d,
// 2 cell-structured (stratified / tree round, CTA per tile), 3 small cells
// (warp per tile, kTileAlign-aligned tile groups), 4 small cells of a large
// grid (thread per cell, kProgThreads-aligned).
#pragma once

#include "mcb_device.cuh"

#ifndef MCB_JIT_THREADS
#define MCB_JIT_THREADS 128  // = kProgThreads
#endif
#ifndef MCB_JIT_WARP_MIN_BLOCKS
#define MCB_JIT_WARP_MIN_BLOCKS 8  // small-cell kernels are latency-bound: occupancy pays
#endif

namespace mcb {
namespace jit {

using dev::FnDesc;
using dev::PhiloxPrefix;
using dev::TilePartial;

constexpr int T = MCB_JIT_THREADS;

__device__ __forceinline__ bool finite64(double x) {
  return (uint32_t(__double2hiint(x)) & 0x7FF00000u) != 0x7FF00000u;
}

// Coordinates of the two samples of pair q (gen_points of the interpreter,
// into registers).
template <int D, bool UNIT_DOM>
__device__ __forceinline__ void gen_points(const FnDesc& f, const PhiloxPrefix& P, uint32_t q, double* x0,
                                           double* x1) {
  const uint64_t pbase = uint64_t(dev::kM0) * uint64_t(q * uint32_t(D));
#pragma unroll
  for (int i = 0; i < D; ++i) {
    uint32_t o[4];
    dev::philox_block_p(P, pbase + uint64_t(i) * dev::kM0, o);
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int t = 2 * i + hh, h = t / D, j = t % D;
      const double u = __dmul_rn(hh ? dev::u_scaled(o[2], o[3]) : dev::u_scaled(o[0], o[1]), dev::kTwoM64);
      const double x = UNIT_DOM ? u : __dadd_rn(f.low[j], __dmul_rn(f.width[j], u));
      if (h == 0) x0[j] = x;
      else x1[j] = x;
    }
  }
}

__device__ __forceinline__ void add_pair(const FnDesc& f, uint32_t q, uint32_t count, double f0, double f1,
                                         double& s1, double& s2, uint32_t& nbad) {
  const bool has1 = 2 * q + 1 < count;
  const bool ok0 = finite64(f0), ok1 = has1 && finite64(f1);
  nbad += (ok0 ? 0u : 1u) + ((has1 && !ok1) ? 1u : 0u);
  const double g0 = ok0 ? __dsub_rn(f0, f.shift) : 0.0;
  const double g1 = ok1 ? __dsub_rn(f1, f.shift) : 0.0;
  s1 = __dadd_rn(s1, g0);
  s2 = fma(g0, g0, s2);
  s1 = __dadd_rn(s1, g1);
  s2 = fma(g1, g1, s2);
}

// Shared pair loop + accumulation: sums of g = f - shift over the finite
// samples of pairs q = first, first + stride, ... (< pairs).
template <class P, int D, bool UNIT_DOM>
__device__ __forceinline__ void accumulate(const FnDesc& f, const PhiloxPrefix& Ph, const double* params,
                                           uint32_t first, uint32_t stride, uint32_t pairs, uint32_t count,
                                           double& s1, double& s2, uint32_t& nbad) {
  // two pairs per iteration: independent Philox / evaluation chains interleave
  // (the sums still take the pairs in ascending order, as the interpreter)
  uint32_t q = first;
  for (; q + stride < pairs; q += 2 * stride) {
    double x0[D], x1[D], y0[D], y1[D];
    gen_points<D, UNIT_DOM>(f, Ph, q, x0, x1);
    gen_points<D, UNIT_DOM>(f, Ph, q + stride, y0, y1);
    const double a0 = P::eval(x0, params), a1 = P::eval(x1, params);
    const double b0 = P::eval(y0, params), b1 = P::eval(y1, params);
    add_pair(f, q, count, a0, a1, s1, s2, nbad);
    add_pair(f, q + stride, count, b0, b1, s1, s2, nbad);
  }
  if (q < pairs) {
    double x0[D], x1[D];
    gen_points<D, UNIT_DOM>(f, Ph, q, x0, x1);
    add_pair(f, q, count, P::eval(x0, params), P::eval(x1, params), s1, s2, nbad);
  }
}

__device__ __forceinline__ void warp_sum(double& s1, double& s2, uint32_t& nbad) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    s1 = __dadd_rn(s1, __shfl_xor_sync(0xFFFFFFFFu, s1, o));
    s2 = __dadd_rn(s2, __shfl_xor_sync(0xFFFFFFFFu, s2, o));
    nbad += __shfl_xor_sync(0xFFFFFFFFu, nbad, o);
  }
}

// Modes 0-2: one CTA per tile (k_program).
template <class P, int D, int MODE>
__device__ __forceinline__ void tile_cta(const FnDesc* __restrict__ fns, const uint32_t* __restrict__ tile_fn,
                                         uint64_t tile0, TilePartial* __restrict__ part) {
  constexpr bool UNIT_DOM = MODE == 1;
  constexpr bool STRAT = MODE == 2;
  const uint64_t tile = tile0 + blockIdx.x;
  const uint32_t fi = __ldg(tile_fn + tile);
  FnDesc f = fns[fi];
  const uint32_t rem = uint32_t(tile - f.tile_base);
  const uint32_t trial = rem / f.n_chunks;
  const uint32_t chunk = rem - trial * f.n_chunks;
  uint32_t count;
  if (STRAT) {
    const uint32_t cell = chunk / f.cpc, cc = chunk - cell * f.cpc;
    count = (cc + 1 == f.cpc) ? f.spc - cc * MCB_CHUNK_SIZE : MCB_CHUNK_SIZE;
    dev::cell_rect<D>(f, cell, 1.0);
  } else {
    count = (chunk + 1 == f.n_chunks) ? uint32_t(f.n_samples - uint64_t(chunk) * MCB_CHUNK_SIZE)
                                      : MCB_CHUNK_SIZE;
  }
  const uint32_t pairs = (count + 1) >> 1;
  const PhiloxPrefix Ph = dev::make_prefix(f.key0, f.key1, f.chunk_base + chunk, f.trial_base + trial);
  double params[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) params[i] = f.k[i];
  if (STRAT) {  // per-tile shift = f(first sample of the tile)
    __shared__ double s_shift;
    if (threadIdx.x == 0) {
      double x0[D], x1[D];
      gen_points<D, false>(f, Ph, 0, x0, x1);
      const double f0 = P::eval(x0, params);
      s_shift = finite64(f0) ? f0 : 0.0;
    }
    __syncthreads();
    f.shift = s_shift;
  }
  double s1 = 0.0, s2 = 0.0;
  uint32_t nbad = 0;
  accumulate<P, D, UNIT_DOM>(f, Ph, params, threadIdx.x, T, pairs, count, s1, s2, nbad);
  warp_sum(s1, s2, nbad);
  __shared__ double sh1[T / 32], sh2[T / 32];
  __shared__ uint32_t shb[T / 32];
  if ((threadIdx.x & 31) == 0) {
    sh1[threadIdx.x >> 5] = s1;
    sh2[threadIdx.x >> 5] = s2;
    shb[threadIdx.x >> 5] = nbad;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t1 = sh1[0], t2 = sh2[0];
    uint32_t tb = shb[0];
#pragma unroll
    for (int w = 1; w < T / 32; ++w) {
      t1 = __dadd_rn(t1, sh1[w]);
      t2 = __dadd_rn(t2, sh2[w]);
      tb += shb[w];
    }
    TilePartial p;
    p.s1 = t1;
    p.s2 = t2;
    p.shift = f.shift;
    p.n_nonfinite = tb;
    p.n_finite = count - tb;
    part[tile] = p;
  }
}

// Mode 3: small cells, one warp per tile (k_program_warp).
template <class P, int D>
__device__ __forceinline__ void tile_warp(const FnDesc* __restrict__ fns, const uint32_t* __restrict__ tile_fn,
                                          uint64_t tile0, TilePartial* __restrict__ part) {
  constexpr uint32_t kTilesPerCta = T / 32;
  const uint64_t group = tile0 + uint64_t(blockIdx.x) * kTilesPerCta;
  const uint32_t fi = __ldg(tile_fn + group);
  FnDesc f = fns[fi];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t tile = group + warp;
  const uint32_t rem = uint32_t(tile - f.tile_base);
  const uint32_t trial = rem / f.n_chunks;
  const uint32_t chunk = rem - trial * f.n_chunks;
  const uint32_t cell = chunk / f.cpc, cc = chunk - cell * f.cpc;
  if (cell >= f.n_cells) return;  // padding tile of the aligned range
  const uint32_t count = (cc + 1 == f.cpc) ? f.spc - cc * MCB_CHUNK_SIZE : MCB_CHUNK_SIZE;
  dev::cell_rect<D>(f, cell, 1.0);
  const uint32_t pairs = (count + 1) >> 1;
  const PhiloxPrefix Ph = dev::make_prefix(f.key0, f.key1, f.chunk_base + chunk, f.trial_base + trial);
  double params[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) params[i] = f.k[i];
  double s1 = 0.0, s2 = 0.0;
  uint32_t nbad = 0;
  {  // first pair of every lane; lane 0's sample 0 is the per-tile shift
    double f0 = 0.0, f1 = 0.0;
    if (lane < pairs) {
      double x0[D], x1[D];
      gen_points<D, false>(f, Ph, lane, x0, x1);
      f0 = P::eval(x0, params);
      f1 = P::eval(x1, params);
    }
    const double c = __shfl_sync(0xFFFFFFFFu, f0, 0);
    f.shift = finite64(c) ? c : 0.0;
    if (lane < pairs) add_pair(f, lane, count, f0, f1, s1, s2, nbad);
  }
  accumulate<P, D, false>(f, Ph, params, lane + 32, 32, pairs, count, s1, s2, nbad);
  warp_sum(s1, s2, nbad);
  if (lane == 0) {
    TilePartial p;
    p.s1 = s1;
    p.s2 = s2;
    p.shift = f.shift;
    p.n_nonfinite = nbad;
    p.n_finite = count - nbad;
    part[tile] = p;
  }
}

// Mode 4: small cells of a large grid, one thread per cell (k_program_lane).
template <class P, int D>
__device__ __forceinline__ void tile_lane(const FnDesc* __restrict__ fns, const uint32_t* __restrict__ tile_fn,
                                          uint64_t tile0, TilePartial* __restrict__ part) {
  const uint64_t group = tile0 + uint64_t(blockIdx.x) * T;
  const uint32_t fi = __ldg(tile_fn + group);
  FnDesc f = fns[fi];
  const uint64_t tile = group + threadIdx.x;
  const uint32_t rem = uint32_t(tile - f.tile_base);
  const uint32_t trial = rem / f.n_chunks;
  const uint32_t cell = rem - trial * f.n_chunks;
  if (cell >= f.n_cells) return;  // padding thread of the aligned range
  const uint32_t count = f.spc;
  dev::cell_rect<D>(f, cell, 1.0);
  const uint32_t pairs = (count + 1) >> 1;
  const PhiloxPrefix Ph = dev::make_prefix(f.key0, f.key1, f.chunk_base + cell, f.trial_base + trial);
  double params[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) params[i] = f.k[i];
  double s1 = 0.0, s2 = 0.0;
  uint32_t nbad = 0;
  {  // pair 0: its first sample is the cell's shift
    double x0[D], x1[D];
    gen_points<D, false>(f, Ph, 0, x0, x1);
    const double f0 = P::eval(x0, params), f1 = P::eval(x1, params);
    f.shift = finite64(f0) ? f0 : 0.0;
    add_pair(f, 0, count, f0, f1, s1, s2, nbad);
  }
  accumulate<P, D, false>(f, Ph, params, 1, 1, pairs, count, s1, s2, nbad);
  TilePartial p;
  p.s1 = s1;
  p.s2 = s2;
  p.shift = f.shift;
  p.n_nonfinite = nbad;
  p.n_finite = count - nbad;
  part[tile] = p;
}

}  // namespace jit
}  // namespace mcb

// One entry point `NAME` for kernel mode MODE (0 direct, 1 unit cube,
// 2 cells CTA-per-tile, 3 small cells warp-per-tile): only the mode a
// launch needs is compiled.
template <int MODE>
struct JitBounds {
  static constexpr int min_blocks = MODE >= 3 ? MCB_JIT_WARP_MIN_BLOCKS : 1;
};
#define MCB_JIT_KERNEL(NAME, PROG, D, MODE)                                                         \
  extern "C" __global__ void __launch_bounds__(MCB_JIT_THREADS, JitBounds<MODE>::min_blocks)        \
      NAME(const mcb::dev::FnDesc* f, const uint32_t* t, uint64_t t0, mcb::dev::TilePartial* p) {   \
    if constexpr (MODE == 4)                                                                        \
      mcb::jit::tile_lane<PROG, D>(f, t, t0, p);                                                    \
    else if constexpr (MODE == 3)                                                                   \
      mcb::jit::tile_warp<PROG, D>(f, t, t0, p);                                                    \
    else                                                                                            \
      mcb::jit::tile_cta<PROG, D, MODE>(f, t, t0, p);                                               \
  }
