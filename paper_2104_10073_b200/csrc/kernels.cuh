// kernels.cuh — the fused direct-MC kernel template (K3) and its test twin.
//
// K3 k_direct<FAM,D,V>: one CTA per tile = (integrand, trial, chunk) unit of
//    <= 65536 samples (the reference task, src/batch.cpp:235-253).  Each
//    thread walks sample pairs: Philox in registers (K1) -> FP64 family value
//    (K2) -> running sums of g = f - shift and g^2 -> warp butterfly -> fixed
//    CTA tree -> one TilePartial.  Replaces accumulate_chunk
//    (src/estimator.cpp:36-49) + ChunkAccum::add (:9-18).  Global memory
//    traffic is the descriptor, the 8 KB trig table (L2-resident) and a
//    24-byte partial per tile.  No float atomics: the reduction shape is
//    fixed, so results do not depend on scheduling or the GPU count.
//
// Included by the per-family translation units (direct_*.cu), which
// instantiate the (family, dim, variant) combinations and register them in
// the dispatch table (direct.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "mcb_internal.hpp"

namespace mcb {
namespace detail {

using dev::FnDesc;
using dev::PhiloxPrefix;
using dev::TilePartial;
using dev::TrigAB;

// Reduction / trig constants (constant bank: DFMA takes them as operands).
static __constant__ dev::TrigConsts c_trig = MCB_TRIG_CONSTS;

__device__ __forceinline__ bool finite64(double x) {
  return (uint32_t(__double2hiint(x)) & 0x7FF00000u) != 0x7FF00000u;  // exponent != 0x7FF
}

// Per-CTA A_m/B_m table of the FAST harmonic form (see mcb_device.cuh).
template <bool UNIT_COEF>
__device__ __forceinline__ void build_trig_table(TrigAB* ab, double a, double b) {
  for (int m = threadIdx.x; m < 512; m += blockDim.x)
    ab[m] = dev::trig_ab<UNIT_COEF>(dev::g_trig_dev[m], a, b);
}

// kFoldShift table: {A_m - c, B_m, A_m} per entry (mcb_device.cuh).
template <bool UNIT_COEF>
__device__ __forceinline__ void build_trig_table_shifted(dev::TrigABS* tab, double a, double b,
                                                         double c) {
  for (int m = threadIdx.x; m < 512; m += blockDim.x)
    tab[m] = dev::trig_abs_entry(dev::g_trig_dev[m], a, b, c, UNIT_COEF);
}

template <int FAM, int D, int V>
__global__ void __launch_bounds__(kThreads, MCB_MIN_BLOCKS)
    k_direct(const FnDesc* __restrict__ fns, const uint32_t* __restrict__ tile_fn, uint64_t tile0,
             TilePartial* __restrict__ part) {
  constexpr bool UNIT_DOM = (V & kUnitDomain) != 0;
  constexpr bool UNIT_COEF = (V & kUnitCoef) != 0;
  constexpr bool SAFE = (V & kSafe) != 0;
  constexpr bool FOLD = (V & kFoldShift) != 0;
  constexpr bool STRAT = (V & kStrat) != 0;
  constexpr bool HARM = FAM == MCB_FAMILY_HARMONIC || FAM == MCB_FAMILY_HARMONIC_VEC;
  constexpr bool TABLE = HARM && !SAFE;
  static_assert(!FOLD || (TABLE && !STRAT), "folded shift: FAST harmonic, direct method");

  const uint64_t tile = tile0 + blockIdx.x;
  const uint32_t fi = __ldg(tile_fn + tile);
  FnDesc f = fns[fi];  // uniform; ptxas keeps only the fields this variant reads

  const uint32_t rem = uint32_t(tile - f.tile_base);
  const uint32_t trial = rem / f.n_chunks;
  const uint32_t chunk = rem - trial * f.n_chunks;  // STRAT: cell * cpc + chunk in cell
  uint32_t count;
  if (STRAT) {
    // stratified_mc cell `cell`: direct_mc over grid_cell(domain, k, cell) with
    // spc samples and chunk keys cell * cpc + c (ref src/batch.cpp:255-275);
    // a tree round's listed cell likewise (ref src/estimator.cpp:238-253)
    const uint32_t cell = chunk / f.cpc, cc = chunk - cell * f.cpc;
    count = (cc + 1 == f.cpc) ? f.spc - cc * MCB_CHUNK_SIZE : MCB_CHUNK_SIZE;
    dev::cell_rect<D>(f, cell, SAFE ? 1.0 : dev::kTwoM64);
  } else {
    count = (chunk + 1 == f.n_chunks) ? uint32_t(f.n_samples - uint64_t(chunk) * MCB_CHUNK_SIZE)
                                      : MCB_CHUNK_SIZE;
  }
  const PhiloxPrefix P =
      dev::make_prefix(f.key0, f.key1, f.chunk_base + chunk, f.trial_base + trial);
  __shared__ TrigAB ab[TABLE && !FOLD ? 512 : 1];
  __shared__ dev::TrigABS abs_tab[FOLD ? 512 : 1];
  if (TABLE) {
    if (FOLD)
      build_trig_table_shifted<UNIT_COEF>(abs_tab, f.a, f.b, f.shift);
    else
      build_trig_table<UNIT_COEF>(ab, f.a, f.b);
    __syncthreads();
  }
  // STRAT: per-tile shift = f(first sample of the tile); tiles merge by
  // Chan's formula in k_combine, so cells (often near-constant) keep an
  // exactly zero variance when f is constant on them.
  if (STRAT) {
    __shared__ double s_shift;
    if (threadIdx.x == 0) {
      double st0, st1;
      dev::gen_pair<FAM, D, false, SAFE>(f, P, 0ull, st0, st1);
      const double f0 = dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, st0);
      s_shift = finite64(f0) ? f0 : 0.0;
    }
    __syncthreads();
    f.shift = s_shift;
  }

  double s1 = 0.0, s2 = 0.0;
  uint32_t nbad = 0;
  // g of one sample (f - shift; non-finite samples counted and dropped in SAFE)
  auto take = [&](double st) {
    double g;
    bool ok = true;
    if constexpr (FOLD) {  // g = f - shift straight from the folded table
      g = dev::finish_shifted<FAM>(f, c_trig, abs_tab, st);
    } else {
      const double fv = dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, st);
      ok = !SAFE || finite64(fv);
      g = __dsub_rn(fv, f.shift);
    }
    nbad += ok ? 0u : 1u;
    return ok ? g : 0.0;
  };
  // Software pipeline over the tile's FULL pairs: iteration i finishes pair
  // q_i (FP64-heavy) while generating pair q_{i+1} (integer-heavy); the last
  // iteration generates one pair past its range, which is discarded.  An odd
  // count's last sample (first half of pair `full`) is taken after the loop
  // by the thread whose pair sequence it ends, so every thread's sums keep
  // the sample order.  Round-1 Philox products advance by 64-bit adds:
  // M0 * (q + T) * D = M0 * q * D + M0 * T * D.
  const uint32_t full = count >> 1;
  const uint32_t iters = threadIdx.x < full ? (full - threadIdx.x + kThreads - 1) / kThreads : 0u;
  uint64_t pbase = uint64_t(dev::kM0) * uint64_t(threadIdx.x * uint32_t(D));
  constexpr uint64_t kStep = uint64_t(dev::kM0) * uint64_t(kThreads * D);
  double a0, a1;
  dev::gen_pair<FAM, D, UNIT_DOM, SAFE>(f, P, pbase, a0, a1);
  for (uint32_t it = iters; it != 0; --it) {
    pbase = dev::add64(pbase, kStep);
    double b0, b1;
    dev::gen_pair<FAM, D, UNIT_DOM, SAFE>(f, P, pbase, b0, b1);
    const double g0 = take(a0), g1 = take(a1);
    a0 = b0;
    a1 = b1;
    s1 = __dadd_rn(s1, g0);
    s2 = fma(g0, g0, s2);
    s1 = __dadd_rn(s1, g1);
    s2 = fma(g1, g1, s2);
  }
  if ((count & 1u) && threadIdx.x == full % kThreads) {
    // pbase now addresses pair `full` (iters steps past this thread's first
    // pair), already generated into a0, a1; only its first sample exists
    const double g0 = take(a0);
    s1 = __dadd_rn(s1, g0);
    s2 = fma(g0, g0, s2);
  }

  // fixed-shape reduction: warp butterfly, then warps 0..W-1 in order
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    s1 = __dadd_rn(s1, __shfl_xor_sync(0xFFFFFFFFu, s1, m));
    s2 = __dadd_rn(s2, __shfl_xor_sync(0xFFFFFFFFu, s2, m));
    if (SAFE) nbad += __shfl_xor_sync(0xFFFFFFFFu, nbad, m);
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
    p.shift = f.shift;
    p.n_nonfinite = SAFE ? tb : 0u;
    p.n_finite = count - p.n_nonfinite;
    part[tile] = p;
  }
}

// K3w k_direct_warp<FAM,D,V> (V has kStrat | kWarpTile): small cells.  The
// CTA covers kTileAlign consecutive tiles of ONE (integrand, trial) (the host
// pads each integrand's per-trial tile range to a multiple of kTileAlign), so
// the descriptor and the trig table stay CTA-uniform while each warp runs one
// tile start to finish: per-warp shift (lane 0, broadcast), lane-strided
// pairs, warp butterfly, one TilePartial per tile — no CTA barrier after the
// table.  Same sums per tile as K3 up to the (fixed) reduction shape.
// Resident CTAs per SM of k_direct_warp: the warp-per-tile loop is latency-
// bound, so occupancy pays as long as nothing spills (ptxas -v: 64 registers
// suffice up to 4-D, 80 up to 6-D; SAFE calls libdevice sincos).
constexpr int warp_tile_min_blocks(int D, int V) {
  return (V & kSafe) ? 2 : (D <= 4 ? 4 : (D <= 6 ? 3 : 2));
}

template <int FAM, int D, int V>
__global__ void __launch_bounds__(kThreads, warp_tile_min_blocks(D, V))
    k_direct_warp(const FnDesc* __restrict__ fns, const uint32_t* __restrict__ tile_fn, uint64_t tile0,
                  TilePartial* __restrict__ part) {
  constexpr bool UNIT_COEF = (V & kUnitCoef) != 0;
  constexpr bool SAFE = (V & kSafe) != 0;
  constexpr bool HARM = FAM == MCB_FAMILY_HARMONIC || FAM == MCB_FAMILY_HARMONIC_VEC;
  constexpr bool TABLE = HARM && !SAFE;
  static_assert((V & kStrat) && (V & kWarpTile), "cell-structured warp-tile variant");

  const uint64_t group = tile0 + uint64_t(blockIdx.x) * kTileAlign;
  const uint32_t fi = __ldg(tile_fn + group);
  FnDesc f = fns[fi];
  // Unit coefficients: A_m, B_m do not depend on the integrand, read through
  // L1 from global memory — no per-CTA table, no barrier.  Otherwise the
  // CTA's (a, b) table is staged in shared memory as in K3.
  constexpr bool STAGE = TABLE && !UNIT_COEF;
  __shared__ TrigAB ab_smem[STAGE ? 512 : 1];
  const TrigAB* ab = ab_smem;
  if (TABLE && UNIT_COEF) ab = dev::g_trig_unit_ab;
  if (STAGE) {
    build_trig_table<UNIT_COEF>(ab_smem, f.a, f.b);
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t tile = group + warp;
  const uint32_t rem = uint32_t(tile - f.tile_base);
  const uint32_t trial = rem / f.n_chunks;
  const uint32_t chunk = rem - trial * f.n_chunks;
  const uint32_t cell = chunk / f.cpc, cc = chunk - cell * f.cpc;
  if (cell >= f.n_cells) return;  // padding tile of the aligned range
  const uint32_t count = (cc + 1 == f.cpc) ? f.spc - cc * MCB_CHUNK_SIZE : MCB_CHUNK_SIZE;
  dev::cell_rect<D>(f, cell, SAFE ? 1.0 : dev::kTwoM64);
  const uint32_t pairs = (count + 1) >> 1;
  const PhiloxPrefix P = dev::make_prefix(f.key0, f.key1, f.chunk_base + chunk, f.trial_base + trial);
  double s1 = 0.0, s2 = 0.0;
  uint32_t nbad = 0;
  auto add = [&](uint32_t q, double f0, double f1) {
    const bool has1 = 2 * q + 1 < count;
    double g0 = __dsub_rn(f0, f.shift);
    double g1 = __dsub_rn(f1, f.shift);
    if (SAFE) {
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
  };
  // First pair of every lane; lane 0's first sample is sample 0 of the tile,
  // whose value is the per-tile shift (as K3) — broadcast, not re-evaluated.
  {
    double f0 = 0.0, f1 = 0.0;
    if (lane < pairs) {
      double x0, x1;
      dev::gen_pair<FAM, D, false, SAFE>(f, P, uint64_t(dev::kM0) * uint64_t(lane * uint32_t(D)), x0, x1);
      f0 = dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, x0);
      f1 = dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, x1);
    }
    {
      const double c = __shfl_sync(0xFFFFFFFFu, f0, 0);
      f.shift = finite64(c) ? c : 0.0;
    }
    if (lane < pairs) add(lane, f0, f1);
  }
  // two pairs per iteration (q, q + 32): independent Philox / trig chains
  // interleave, as K3's software pipeline does; sums keep ascending q order
  // round-1 products advance by 64-bit adds (as K3): M0*(q+32)D = M0*qD + M0*32D
  constexpr uint64_t kStep32 = uint64_t(dev::kM0) * uint64_t(32 * D);
  uint32_t q = lane + 32;
  uint64_t pq = uint64_t(dev::kM0) * uint64_t(q * uint32_t(D));
  for (; q + 32 < pairs; q += 64, pq += 2 * kStep32) {
    double x0, x1, y0, y1;
    dev::gen_pair<FAM, D, false, SAFE>(f, P, pq, x0, x1);
    dev::gen_pair<FAM, D, false, SAFE>(f, P, pq + kStep32, y0, y1);
    const double a0 = dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, x0);
    const double a1 = dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, x1);
    const double b0 = dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, y0);
    const double b1 = dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, y1);
    add(q, a0, a1);
    add(q + 32, b0, b1);
  }
  if (q < pairs) {
    double x0, x1;
    dev::gen_pair<FAM, D, false, SAFE>(f, P, pq, x0, x1);
    add(q, dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, x0), dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, x1));
  }
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) {
    s1 = __dadd_rn(s1, __shfl_xor_sync(0xFFFFFFFFu, s1, m));
    s2 = __dadd_rn(s2, __shfl_xor_sync(0xFFFFFFFFu, s2, m));
    if (SAFE) nbad += __shfl_xor_sync(0xFFFFFFFFu, nbad, m);
  }
  if (lane == 0) {
    TilePartial p;
    p.s1 = s1;
    p.s2 = s2;
    p.shift = f.shift;
    p.n_nonfinite = SAFE ? nbad : 0u;
    p.n_finite = count - p.n_nonfinite;
    part[tile] = p;
  }
}

// K3l k_direct_lane<FAM,D,V> (V has kStrat | kLaneCell): the small cells of a
// large stratified grid (one chunk per cell), one LANE per cell.  A one-warp
// CTA covers kLaneAlign consecutive cells of one (integrand, trial) (ranges
// padded / aligned by the host), so the descriptor is CTA-uniform; each lane
// runs its cell start to finish like a K3 thread runs its pairs — sample 0 is
// the cell's shift, the pairs in ascending order, two per iteration — and
// writes the cell's TilePartial: no shuffles, no reduction, no idle lanes on
// a partial last round of pairs.  Tables: unit coefficients (read through
// L1) or none (SAFE / abs); the host keeps general-coefficient harmonic
// grids on K3w.
template <int FAM, int D, int V>
__global__ void __launch_bounds__(kLaneAlign, 8 * warp_tile_min_blocks(D, V))
    k_direct_lane(const FnDesc* __restrict__ fns, const uint32_t* __restrict__ tile_fn, uint64_t tile0,
                  TilePartial* __restrict__ part) {
  constexpr bool UNIT_COEF = (V & kUnitCoef) != 0;
  constexpr bool SAFE = (V & kSafe) != 0;
  constexpr bool HARM = FAM == MCB_FAMILY_HARMONIC || FAM == MCB_FAMILY_HARMONIC_VEC;
  constexpr bool TABLE = HARM && !SAFE;
  static_assert((V & kStrat) && (V & kLaneCell) && !(V & kWarpTile), "cell-per-lane variant");
  static_assert(!TABLE || UNIT_COEF, "general-coefficient tables stay on K3w");

  const uint64_t group = tile0 + uint64_t(blockIdx.x) * kLaneAlign;
  const uint32_t fi = __ldg(tile_fn + group);
  FnDesc f = fns[fi];
  const TrigAB* ab = TABLE ? dev::g_trig_unit_ab : nullptr;
  const uint64_t tile = group + threadIdx.x;
  const uint32_t rem = uint32_t(tile - f.tile_base);
  const uint32_t trial = rem / f.n_chunks;
  const uint32_t cell = rem - trial * f.n_chunks;  // one chunk per cell
  if (cell >= f.n_cells) return;                   // padding lane of the aligned range
  const uint32_t count = f.spc;
  dev::cell_rect<D>(f, cell, SAFE ? 1.0 : dev::kTwoM64);
  const uint32_t pairs = (count + 1) >> 1;
  const PhiloxPrefix P = dev::make_prefix(f.key0, f.key1, f.chunk_base + cell, f.trial_base + trial);
  double s1 = 0.0, s2 = 0.0;
  uint32_t nbad = 0;
  auto add = [&](uint32_t q, double f0, double f1) {
    const bool has1 = 2 * q + 1 < count;
    double g0 = __dsub_rn(f0, f.shift);
    double g1 = __dsub_rn(f1, f.shift);
    if (SAFE) {
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
  };
  constexpr uint64_t kStep = uint64_t(dev::kM0) * uint64_t(D);  // round-1 product step per pair
  {  // pair 0: its first sample is the cell's shift
    double x0, x1;
    dev::gen_pair<FAM, D, false, SAFE>(f, P, 0, x0, x1);
    const double f0 = dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, x0);
    const double f1 = dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, x1);
    f.shift = finite64(f0) ? f0 : 0.0;
    add(0, f0, f1);
  }
  uint32_t q = 1;
  uint64_t pq = kStep;
  for (; q + 1 < pairs; q += 2, pq += 2 * kStep) {  // two independent chains per iteration
    double x0, x1, y0, y1;
    dev::gen_pair<FAM, D, false, SAFE>(f, P, pq, x0, x1);
    dev::gen_pair<FAM, D, false, SAFE>(f, P, pq + kStep, y0, y1);
    const double a0 = dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, x0);
    const double a1 = dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, x1);
    const double b0 = dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, y0);
    const double b1 = dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, y1);
    add(q, a0, a1);
    add(q + 1, b0, b1);
  }
  if (q < pairs) {
    double x0, x1;
    dev::gen_pair<FAM, D, false, SAFE>(f, P, pq, x0, x1);
    add(q, dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, x0), dev::finish<FAM, UNIT_COEF, SAFE>(f, c_trig, ab, x1));
  }
  TilePartial p;
  p.s1 = s1;
  p.s2 = s2;
  p.shift = f.shift;
  p.n_nonfinite = SAFE ? nbad : 0u;
  p.n_finite = count - p.n_nonfinite;
  part[tile] = p;
}

// Family values of the pairs [first_pair, first_pair + n_pairs) of one chunk,
// through exactly the gen_pair/finish instantiation the fused kernel uses.
template <int FAM, int D, int V>
__global__ void k_debug_eval(const FnDesc* __restrict__ fn, uint32_t trial, uint32_t chunk,
                             uint32_t first_pair, uint32_t n_pairs, double* __restrict__ out) {
  constexpr bool UNIT_COEF = (V & kUnitCoef) != 0;
  constexpr bool SAFE = (V & kSafe) != 0;
  constexpr bool TABLE =
      (FAM == MCB_FAMILY_HARMONIC || FAM == MCB_FAMILY_HARMONIC_VEC) && !SAFE;
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const FnDesc f = *fn;
  const PhiloxPrefix P = dev::make_prefix(f.key0, f.key1, chunk, trial);
  constexpr bool FOLD = (V & kFoldShift) != 0;
  __shared__ TrigAB ab[TABLE && !FOLD ? 512 : 1];
  __shared__ dev::TrigABS abs_tab[FOLD ? 512 : 1];
  if (TABLE) {
    if (FOLD)
      build_trig_table_shifted<UNIT_COEF>(abs_tab, f.a, f.b, f.shift);
    else
      build_trig_table<UNIT_COEF>(ab, f.a, f.b);
    __syncthreads();
  }
  if (i >= n_pairs) return;
  double f0, f1;
  if constexpr (FOLD) {  // the fused kernel's g, reported as g + shift
    double st0, st1;
    dev::gen_pair<FAM, D, (V & kUnitDomain) != 0, SAFE>(
        f, P, uint64_t(dev::kM0) * uint64_t((first_pair + i) * uint32_t(D)), st0, st1);
    f0 = __dadd_rn(dev::finish_shifted<FAM>(f, c_trig, abs_tab, st0), f.shift);
    f1 = __dadd_rn(dev::finish_shifted<FAM>(f, c_trig, abs_tab, st1), f.shift);
  } else {
    dev::eval_pair<FAM, D, (V & kUnitDomain) != 0, UNIT_COEF, SAFE>(f, c_trig, ab, P, first_pair + i,
                                                                     f0, f1);
  }
  out[2 * uint64_t(i)] = f0;
  out[2 * uint64_t(i) + 1] = f1;
}

// ---- dispatch table ----------------------------------------------------------

using DirectFn = void (*)(const FnDesc*, const uint32_t*, uint64_t, TilePartial*);
using EvalFn = void (*)(const FnDesc*, uint32_t, uint32_t, uint32_t, uint32_t, double*);

struct Entry {
  DirectFn direct = nullptr;
  EvalFn eval = nullptr;
};

struct Table {
  Entry e[4][MCB_MAX_DIM + 1][kNumVariants];
  template <int FAM, int D, int V>
  void put() {
    e[FAM][D][V].direct = k_direct<FAM, D, V>;
    e[FAM][D][V].eval = k_debug_eval<FAM, D, V>;
  }
  // stratified variants: the fused kernel only (cell values are tested
  // through the direct variants on the cell rectangle)
  template <int FAM, int D, int V>
  void put_run() {
    e[FAM][D][V | kStrat].direct = k_direct<FAM, D, V | kStrat>;
    e[FAM][D][V | kStrat | kWarpTile].direct = k_direct_warp<FAM, D, V | kStrat | kWarpTile>;
    constexpr bool TABLE = (FAM == MCB_FAMILY_HARMONIC || FAM == MCB_FAMILY_HARMONIC_VEC) && !(V & kSafe);
    if constexpr (!TABLE || (V & kUnitCoef))
      e[FAM][D][V | kStrat | kLaneCell].direct = k_direct_lane<FAM, D, V | kStrat | kLaneCell>;
  }
};

void register_harmonic(Table& t);
void register_harmonic_vec(Table& t);
void register_abs(Table& t);

}  // namespace detail
}  // namespace mcb
