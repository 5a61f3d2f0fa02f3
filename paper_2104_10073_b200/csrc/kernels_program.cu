// kernels_program.cu — the direct-MC kernel for arbitrary DSL integrands
// (MCB_FAMILY_PROGRAM): same sampler, tiles, reduction and combine as the
// family kernels, with the integrand evaluated by a GPU interpreter of the
// compiled postfix program (reference CompiledProgram::evaluate,
// ref/src/expr.cpp:520-553).
//
// Interpreter layout (one CTA = one tile = one integrand, so the program is
// uniform across the CTA and every switch is warp-uniform):
//   * code words and constants staged in shared memory;
//   * the evaluation stack as shared memory slots S[slot][h][tid] (h = the
//     two samples of a pair, so every instruction is dispatched once for two
//     samples), conflict-free because consecutive threads hit consecutive
//     words;
//   * the sample coordinates likewise, X[j][h][tid].
// Every operation is the reference's: IEEE +,-,*,/ (correctly rounded, as
// on the host), libdevice sin/cos/tan/asin/acos/atan/log/pow and dev::mcb_exp (<= 2 ulp of
// glibc), exact sqrt/fabs/floor/fmin/fmax, and the fused cos + sin of one
// argument in the Fig. 1 table form (dev::cos_plus_sin).  Points are the same bit-exact
// Philox stream; non-finite values are counted and skipped.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <set>

#include "jit.hpp"
#include "kernels.cuh"
#include "program.hpp"

namespace mcb {
namespace detail {

constexpr int T = kProgThreads;

// Operand fetch for the NH samples of one dispatch (h = 0..NH-1): slots and
// variables live in shared memory [index][h][tid]; constants and parameters
// are uniform.
template <int NH>
__device__ __forceinline__ void fetch(uint32_t kind, uint32_t idx, const double* S, const double* X,
                                      const double* consts, const double* params, double (&v)[NH]) {
  if (kind <= prog::kVar) {
    const double* p = (kind == prog::kSlot ? S : X) + idx * NH * T + threadIdx.x;
#pragma unroll
    for (int h = 0; h < NH; ++h) v[h] = p[h * T];
  } else {
    const double c = kind == prog::kConst ? consts[idx] : params[idx];
#pragma unroll
    for (int h = 0; h < NH; ++h) v[h] = c;
  }
}

template <int NH>
__device__ __forceinline__ double fetch1(uint32_t kind, uint32_t idx, int h, const double* S, const double* X,
                                         const double* consts, const double* params) {
  if (kind <= prog::kVar) return (kind == prog::kSlot ? S : X)[(idx * NH + h) * T + threadIdx.x];
  return kind == prog::kConst ? consts[idx] : params[idx];
}

// The DSL's exp (dev::mcb_exp, shared with the specialised kernels so both
// paths stay bit-identical), called rather than inlined into the dispatch.
__device__ __noinline__ double interp_exp(double a) { return dev::mcb_exp(a); }

// One libm-class operation on one sample.
__device__ __forceinline__ double call_op(uint32_t op, double a, double b) {
  switch (op) {
    case prog::kDiv: return __ddiv_rn(a, b);
    case prog::kPow: return pow(a, b);
    case prog::kSin: return sin(a);
    case prog::kCos: return cos(a);
    case prog::kTan: return tan(a);
    case prog::kAsin: return asin(a);
    case prog::kAcos: return acos(a);
    case prog::kAtan: return atan(a);
    case prog::kExp: return interp_exp(a);
    case prog::kLog: return log(a);
    case prog::kCosPlusSin: return dev::cos_plus_sin(a);
    default: return __longlong_as_double(0x7FF8000000000000ll);
  }
}

// The interpreter: every instruction is dispatched once for NH samples (the
// two samples of each of NH/2 pairs), so the fetch / decode / warp-uniform
// branch of an instruction is shared by NH evaluations.  Element-wise
// operations run on NH register operands (NH independent FP64 chains in
// flight); libm-class calls take the samples one at a time straight from and
// to shared memory (code size, and no dynamically indexed register arrays).
// Operations and their order per sample are the same for any NH.
template <int NH>
__device__ __forceinline__ void interp(const uint32_t* __restrict__ code, uint32_t len,
                                       const double* __restrict__ consts, const double* __restrict__ params,
                                       double* S, const double* X) {
  const int tid = threadIdx.x;
  // the next instruction's words are loaded while this one executes (the
  // shared code area carries two zero words past the program for the last
  // look-ahead): +1.6 % on C2 as programs against loading at the top of the
  // iteration (profiles/r02_interp_variants.txt)
  uint32_t nw0 = code[0], nw1 = code[1];
  for (uint32_t pc = 0; pc < len; ++pc) {
    const uint32_t w0 = nw0, w1 = nw1;
    nw0 = code[2 * pc + 2];
    nw1 = code[2 * pc + 3];
    const uint32_t op = w0 & 0xFFu;
    const uint32_t ka = (w0 >> 18) & 3u, ia = w1 & 0xFFFFu, kb = (w0 >> 20) & 3u, ib = w1 >> 16;
    double* d = S + ((w0 >> 8) & 31u) * NH * T + tid;
    double a[NH], b[NH], r[NH];
    // one warp-uniform switch per instruction (a jump table), the NH samples'
    // work inside each case
#define MCB_UNARY(EXPR)                                       \
  fetch<NH>(ka, ia, S, X, consts, params, a);                 \
  _Pragma("unroll") for (int h = 0; h < NH; ++h) r[h] = (EXPR); \
  break
#define MCB_BINARY(EXPR)                                      \
  fetch<NH>(ka, ia, S, X, consts, params, a);                 \
  fetch<NH>(kb, ib, S, X, consts, params, b);                 \
  _Pragma("unroll") for (int h = 0; h < NH; ++h) r[h] = (EXPR); \
  break
    switch (op) {
      case prog::kCopy: MCB_UNARY(a[h]);
      case prog::kNeg: MCB_UNARY(-a[h]);
      case prog::kAdd: MCB_BINARY(__dadd_rn(a[h], b[h]));
      case prog::kSub: MCB_BINARY(__dsub_rn(a[h], b[h]));
      case prog::kMul: MCB_BINARY(__dmul_rn(a[h], b[h]));
      case prog::kSqrt: MCB_UNARY(__dsqrt_rn(a[h]));
      case prog::kAbs: MCB_UNARY(fabs(a[h]));
      case prog::kFloor: MCB_UNARY(floor(a[h]));
      case prog::kMin: MCB_BINARY(fmin(a[h], b[h]));
      case prog::kMax: MCB_BINARY(fmax(a[h], b[h]));
      case prog::kCosPlusSin: {  // the table form for NH samples at once, libm for the rare rest
        fetch<NH>(ka, ia, S, X, consts, params, a);
        uint32_t in_range = 0;
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          const bool in = dev::cos_plus_sin_in_range(a[h]);
          r[h] = dev::cos_plus_sin_table(in ? a[h] : 0.0);
          in_range |= in ? 1u << h : 0u;
        }
        if (in_range != (1u << NH) - 1u) {  // operands still intact: nothing stored yet
#pragma unroll 1
          for (int h = 0; h < NH; ++h)
            if (!(in_range >> h & 1u)) d[h * T] = dev::cos_plus_sin_libm(fetch1<NH>(ka, ia, h, S, X, consts, params));
        }
#pragma unroll
        for (int h = 0; h < NH; ++h)
          if (in_range >> h & 1u) d[h * T] = r[h];
        continue;
      }
      case prog::kSinCos: {
        double* d2 = S + ((w0 >> 13) & 31u) * NH * T + tid;
#pragma unroll 1
        for (int h = 0; h < NH; ++h) {
          double sn, cs;
          sincos(fetch1<NH>(ka, ia, h, S, X, consts, params), &sn, &cs);
          d[h * T] = sn;
          d2[h * T] = cs;
        }
        continue;
      }
      case prog::kDiv: case prog::kPow: case prog::kSin: case prog::kCos: case prog::kTan:
      case prog::kAsin: case prog::kAcos: case prog::kAtan: case prog::kExp: case prog::kLog: {
        const bool binary = op == prog::kDiv || op == prog::kPow;
#pragma unroll 1
        for (int h = 0; h < NH; ++h) {
          const double x = fetch1<NH>(ka, ia, h, S, X, consts, params);
          const double y = binary ? fetch1<NH>(kb, ib, h, S, X, consts, params) : 0.0;
          d[h * T] = call_op(op, x, y);
        }
        continue;
      }
      default:
#pragma unroll
        for (int h = 0; h < NH; ++h) r[h] = __longlong_as_double(0x7FF8000000000000ll);
        break;
    }
#undef MCB_UNARY
#undef MCB_BINARY
#pragma unroll
    for (int h = 0; h < NH; ++h) d[h * T] = r[h];
  }
}

__device__ __forceinline__ void interp_pair(const uint32_t* __restrict__ code, uint32_t len,
                                            const double* __restrict__ consts,
                                            const double* __restrict__ params, double* S,
                                            const double* X) {
  interp<2>(code, len, consts, params, S, X);
}

// Coordinates of the two samples of each of the NP pairs q0 + i*stride
// (i < NP) into X[j][2i + h][tid] (NH = 2 NP samples per dispatch).
template <int D, bool UNIT_DOM, int NP = 1>
__device__ __forceinline__ void gen_points(const FnDesc& f, const PhiloxPrefix& P, uint32_t q0,
                                           double* X, uint32_t stride = 0) {
  constexpr int NH = 2 * NP;
#pragma unroll
  for (int pi = 0; pi < NP; ++pi) {
    const uint64_t pbase = uint64_t(dev::kM0) * uint64_t((q0 + uint32_t(pi) * stride) * uint32_t(D));
#pragma unroll
    for (int i = 0; i < D; ++i) {
      uint32_t o[4];
      dev::philox_block_p(P, pbase + uint64_t(i) * dev::kM0, o);
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int t = 2 * i + hh, h = t / D, j = t % D;
        const double u = __dmul_rn(hh ? dev::u_scaled(o[2], o[3]) : dev::u_scaled(o[0], o[1]),
                                   dev::kTwoM64);
        const double x = UNIT_DOM ? u : __dadd_rn(f.low[j], __dmul_rn(f.width[j], u));
        X[(j * NH + 2 * pi + h) * T + threadIdx.x] = x;
      }
    }
  }
}

// Shared memory: S[slots][NH][T] | X[D][NH][T] | consts[kMaxConsts] | code[2 * kMaxCode + 2]
// (NH = 2 NP samples per dispatch)
__host__ __device__ constexpr size_t program_smem_bytes(uint32_t slots, int dim, int np = 1) {
  return (size_t(slots) + size_t(dim)) * 2 * size_t(np) * T * sizeof(double) + prog::kMaxConsts * sizeof(double) +
         (2 * prog::kMaxCode + 2) * sizeof(uint32_t);
}

struct ProgramSmem {
  double* S;
  double* X;
  double* consts;
  uint32_t* code;
};

template <int D, int NP = 1>
__device__ __forceinline__ ProgramSmem stage_program(const FnDesc& f, const uint32_t* __restrict__ code,
                                                     const double* __restrict__ consts, uint32_t slots,
                                                     double* params) {
  extern __shared__ double dyn[];
  ProgramSmem m;
  m.S = dyn;
  m.X = dyn + size_t(slots) * 2 * NP * T;
  m.consts = m.X + size_t(D) * 2 * NP * T;
  m.code = reinterpret_cast<uint32_t*>(m.consts + prog::kMaxConsts);
  for (uint32_t i = threadIdx.x; i < 2 * f.prog_len; i += T) m.code[i] = code[f.prog_off + i];
  if (threadIdx.x < 2) m.code[2 * f.prog_len + threadIdx.x] = 0u;  // interp's look-ahead words
  for (uint32_t i = threadIdx.x; i < f.n_consts; i += T) m.consts[i] = consts[f.const_off + i];
  // static indices only: a dynamic f.k[threadIdx.x] would demote the whole
  // descriptor copy to local memory
#pragma unroll
  for (int i = 0; i < int(prog::kMaxParams); ++i)
    if (threadIdx.x == i) params[i] = f.k[i];
  __syncthreads();
  return m;
}

// NP pairs per thread per dispatch (NH = 2 NP samples): thread tid takes the
// pairs q = tid + i T in ascending i exactly as with NP = 1, so its sums (and
// the results) do not depend on NP.
template <int D, int V, int NP>
__global__ void __launch_bounds__(T) k_program(const FnDesc* __restrict__ fns,
                                               const uint32_t* __restrict__ tile_fn, uint64_t tile0,
                                               TilePartial* __restrict__ part,
                                               const uint32_t* __restrict__ code,
                                               const double* __restrict__ consts, uint32_t slots) {
  constexpr bool UNIT_DOM = (V & kUnitDomain) != 0;
  constexpr bool STRAT = (V & kStrat) != 0;
  const uint64_t tile = tile0 + blockIdx.x;
  const uint32_t fi = __ldg(tile_fn + tile);
  FnDesc f = fns[fi];
  const uint32_t rem = uint32_t(tile - f.tile_base);
  const uint32_t trial = rem / f.n_chunks;
  const uint32_t chunk = rem - trial * f.n_chunks;  // STRAT: cell * cpc + chunk in cell
  uint32_t count;
  if (STRAT) {  // see k_direct: cells of stratified_mc (ref src/batch.cpp:255-275)
    const uint32_t cell = chunk / f.cpc, cc = chunk - cell * f.cpc;
    count = (cc + 1 == f.cpc) ? f.spc - cc * MCB_CHUNK_SIZE : MCB_CHUNK_SIZE;
    dev::cell_rect<D>(f, cell, 1.0);
  } else {
    count = (chunk + 1 == f.n_chunks) ? uint32_t(f.n_samples - uint64_t(chunk) * MCB_CHUNK_SIZE)
                                      : MCB_CHUNK_SIZE;
  }
  const uint32_t pairs = (count + 1) >> 1;
  const PhiloxPrefix P =
      dev::make_prefix(f.key0, f.key1, f.chunk_base + chunk, f.trial_base + trial);
  __shared__ double params[prog::kMaxParams];
  const ProgramSmem m = stage_program<D, NP>(f, code, consts, slots, params);
  constexpr int NH = 2 * NP;
  if (STRAT) {  // per-tile shift = f(first sample of the tile)
    __shared__ double s_shift;
    if (threadIdx.x == 0) {
      gen_points<D, false, NP>(f, P, 0, m.X, T);
      interp<NH>(m.code, f.prog_len, m.consts, params, m.S, m.X);
      const double f0 = m.S[0];
      s_shift = finite64(f0) ? f0 : 0.0;
    }
    __syncthreads();
    f.shift = s_shift;
  }

  double s1 = 0.0, s2 = 0.0;
  uint32_t nbad = 0;
  for (uint32_t q0 = threadIdx.x; q0 < pairs; q0 += NP * T) {
    gen_points<D, UNIT_DOM, NP>(f, P, q0, m.X, T);
    interp<NH>(m.code, f.prog_len, m.consts, params, m.S, m.X);
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const uint32_t q = q0 + uint32_t(i) * T;
      if (q >= pairs) break;
      const double f0 = m.S[2 * i * T + threadIdx.x], f1 = m.S[(2 * i + 1) * T + threadIdx.x];
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
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    s1 = __dadd_rn(s1, __shfl_xor_sync(0xFFFFFFFFu, s1, o));
    s2 = __dadd_rn(s2, __shfl_xor_sync(0xFFFFFFFFu, s2, o));
    nbad += __shfl_xor_sync(0xFFFFFFFFu, nbad, o);
  }
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

// Small cells (kStrat | kWarpTile): the CTA covers kProgThreads/32 tiles of
// one (integrand, trial) — the host pads per-trial tile ranges to multiples
// of kTileAlign — so the staged program stays CTA-uniform while each warp
// runs one tile: per-warp shift, lane-strided pairs, warp butterfly.
template <int D, int V, int NP>
__global__ void __launch_bounds__(T) k_program_warp(const FnDesc* __restrict__ fns,
                                                    const uint32_t* __restrict__ tile_fn, uint64_t tile0,
                                                    TilePartial* __restrict__ part,
                                                    const uint32_t* __restrict__ code,
                                                    const double* __restrict__ consts, uint32_t slots) {
  static_assert((V & kStrat) && (V & kWarpTile), "cell-structured warp-tile variant");
  constexpr uint32_t kTilesPerCta = T / 32;
  const uint64_t group = tile0 + uint64_t(blockIdx.x) * kTilesPerCta;
  const uint32_t fi = __ldg(tile_fn + group);
  FnDesc f = fns[fi];
  __shared__ double params[prog::kMaxParams];
  const ProgramSmem m = stage_program<D, NP>(f, code, consts, slots, params);
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
  const PhiloxPrefix P = dev::make_prefix(f.key0, f.key1, f.chunk_base + chunk, f.trial_base + trial);
  double s1 = 0.0, s2 = 0.0;
  uint32_t nbad = 0;
  auto add = [&](uint32_t q, double f0, double f1) {
    const bool has1 = 2 * q + 1 < count;
    const bool ok0 = finite64(f0), ok1 = has1 && finite64(f1);
    nbad += (ok0 ? 0u : 1u) + ((has1 && !ok1) ? 1u : 0u);
    const double g0 = ok0 ? __dsub_rn(f0, f.shift) : 0.0;
    const double g1 = ok1 ? __dsub_rn(f1, f.shift) : 0.0;
    s1 = __dadd_rn(s1, g0);
    s2 = fma(g0, g0, s2);
    s1 = __dadd_rn(s1, g1);
    s2 = fma(g1, g1, s2);
  };
  // each lane's pairs q = lane + 32 k in ascending k, NP of them per dispatch
  // (results do not depend on NP); lane 0's sample 0 is the per-tile shift
  constexpr int NH = 2 * NP;
  for (uint32_t q0 = lane; q0 < pairs || q0 == uint32_t(lane); q0 += 32 * NP) {
    gen_points<D, false, NP>(f, P, q0, m.X, 32);
    interp<NH>(m.code, f.prog_len, m.consts, params, m.S, m.X);
    if (q0 == uint32_t(lane)) {  // first dispatch of every lane (warp-uniform)
      const double c = __shfl_sync(0xFFFFFFFFu, m.S[threadIdx.x], 0);
      f.shift = finite64(c) ? c : 0.0;
    }
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const uint32_t q = q0 + 32u * uint32_t(i);
      if (q < pairs) add(q, m.S[2 * i * T + threadIdx.x], m.S[(2 * i + 1) * T + threadIdx.x]);
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    s1 = __dadd_rn(s1, __shfl_xor_sync(0xFFFFFFFFu, s1, o));
    s2 = __dadd_rn(s2, __shfl_xor_sync(0xFFFFFFFFu, s2, o));
    nbad += __shfl_xor_sync(0xFFFFFFFFu, nbad, o);
  }
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

// Small cells of a large grid (kStrat | kLaneCell): the CTA covers
// kProgThreads consecutive cells of one (integrand, trial) (ranges padded /
// aligned to kProgThreads by the host), one THREAD per cell (one chunk per
// cell): sample 0 is the cell's shift, the pairs in ascending order, the
// cell's TilePartial written by its thread — no reduction.
template <int D, int V, int NP>
__global__ void __launch_bounds__(T) k_program_lane(const FnDesc* __restrict__ fns,
                                                    const uint32_t* __restrict__ tile_fn, uint64_t tile0,
                                                    TilePartial* __restrict__ part,
                                                    const uint32_t* __restrict__ code,
                                                    const double* __restrict__ consts, uint32_t slots) {
  static_assert((V & kStrat) && (V & kLaneCell) && !(V & kWarpTile), "cell-per-lane variant");
  const uint64_t group = tile0 + uint64_t(blockIdx.x) * T;
  const uint32_t fi = __ldg(tile_fn + group);
  FnDesc f = fns[fi];
  __shared__ double params[prog::kMaxParams];
  const ProgramSmem m = stage_program<D, NP>(f, code, consts, slots, params);
  const uint64_t tile = group + threadIdx.x;
  const uint32_t rem = uint32_t(tile - f.tile_base);
  const uint32_t trial = rem / f.n_chunks;
  const uint32_t cell = rem - trial * f.n_chunks;
  if (cell >= f.n_cells) return;  // padding thread of the aligned range
  const uint32_t count = f.spc;
  dev::cell_rect<D>(f, cell, 1.0);
  const uint32_t pairs = (count + 1) >> 1;
  const PhiloxPrefix P = dev::make_prefix(f.key0, f.key1, f.chunk_base + cell, f.trial_base + trial);
  constexpr int NH = 2 * NP;
  double s1 = 0.0, s2 = 0.0;
  uint32_t nbad = 0;
  // NP consecutive pairs of the cell per dispatch, taken in ascending order
  // (so the sums, and the results, do not depend on NP)
  for (uint32_t q0 = 0; q0 < pairs; q0 += NP) {
    gen_points<D, false, NP>(f, P, q0, m.X, 1);
    interp<NH>(m.code, f.prog_len, m.consts, params, m.S, m.X);
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      const uint32_t q = q0 + uint32_t(i);
      if (q >= pairs) break;
      const double f0 = m.S[2 * i * T + threadIdx.x], f1 = m.S[(2 * i + 1) * T + threadIdx.x];
      if (q == 0) f.shift = finite64(f0) ? f0 : 0.0;
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
  }
  TilePartial p;
  p.s1 = s1;
  p.s2 = s2;
  p.shift = f.shift;
  p.n_nonfinite = nbad;
  p.n_finite = count - nbad;
  part[tile] = p;
}

// Per-sample values of pairs [first_pair, first_pair + n_pairs) of one chunk
// (test hook): exactly the gen_points/interp_pair of k_program.
template <int D, int V>
__global__ void __launch_bounds__(T) k_program_eval(const FnDesc* __restrict__ fn,
                                                    const uint32_t* __restrict__ code,
                                                    const double* __restrict__ consts, uint32_t slots,
                                                    uint32_t trial, uint32_t chunk,
                                                    uint32_t first_pair, uint32_t n_pairs,
                                                    double* __restrict__ out) {
  const FnDesc f = *fn;
  const PhiloxPrefix P = dev::make_prefix(f.key0, f.key1, chunk, trial);
  __shared__ double params[prog::kMaxParams];
  const ProgramSmem m = stage_program<D>(f, code, consts, slots, params);
  const uint32_t i = blockIdx.x * T + threadIdx.x;
  gen_points<D, (V & kUnitDomain) != 0>(f, P, first_pair + i, m.X);
  interp_pair(m.code, f.prog_len, m.consts, params, m.S, m.X);
  if (i < n_pairs) {
    out[2 * uint64_t(i)] = m.S[threadIdx.x];
    out[2 * uint64_t(i) + 1] = m.S[T + threadIdx.x];
  }
}

// CompiledProgram::evaluate at caller-given points (mcb_program_eval_points):
// the interpreter above on coordinates read from global memory, two points
// per thread as in the sampling kernels.  No sampler, no reduction.
template <int D>
__global__ void __launch_bounds__(T) k_program_points(const FnDesc* __restrict__ fn,
                                                      const uint32_t* __restrict__ code,
                                                      const double* __restrict__ consts, uint32_t slots,
                                                      const double* __restrict__ pts, uint64_t n,
                                                      double* __restrict__ out) {
  const FnDesc f = *fn;
  __shared__ double params[prog::kMaxParams];
  const ProgramSmem m = stage_program<D>(f, code, consts, slots, params);
  const uint64_t first = 2 * (uint64_t(blockIdx.x) * T + threadIdx.x);
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int j = 0; j < D; ++j)
      m.X[(j * 2 + h) * T + threadIdx.x] = first + h < n ? pts[(first + h) * D + j] : 0.0;
  interp_pair(m.code, f.prog_len, m.consts, params, m.S, m.X);
#pragma unroll
  for (int h = 0; h < 2; ++h)
    if (first + h < n) out[first + h] = m.S[h * T + threadIdx.x];
}

// ---- dispatch ------------------------------------------------------------------

using ProgFn = void (*)(const FnDesc*, const uint32_t*, uint64_t, TilePartial*, const uint32_t*,
                        const double*, uint32_t);
using ProgEvalFn = void (*)(const FnDesc*, const uint32_t*, const double*, uint32_t, uint32_t,
                            uint32_t, uint32_t, uint32_t, double*);

// Pairs per dispatch of the interpreter kernels (every mode): index of
// NP = 1, 2, 4.
constexpr int kNpVariants = 3;
constexpr int np_of(int i) { return 1 << i; }

struct ProgEntry {
  ProgFn run = nullptr;               // NP = 1 (every mode)
  ProgFn run_np[kNpVariants] = {};    // by NP index
  ProgEvalFn eval = nullptr;
};

struct ProgTable {
  ProgEntry e[MCB_MAX_DIM + 1][5];  // by program_kernel_mode: general / unit domain, cells, small cells (warp, lane)
  template <int D, int V>
  static ProgEntry tile_entry(ProgEvalFn eval) {
    ProgEntry p;
    p.run = k_program<D, V, 1>;
    p.run_np[0] = k_program<D, V, 1>;
    p.run_np[1] = k_program<D, V, 2>;
    p.run_np[2] = k_program<D, V, 4>;
    p.eval = eval;
    return p;
  }
  template <int D>
  void put() {
    e[D][0] = tile_entry<D, kSafe>(k_program_eval<D, kSafe>);
    e[D][1] = tile_entry<D, kSafe | kUnitDomain>(k_program_eval<D, kSafe | kUnitDomain>);
    e[D][2] = tile_entry<D, kSafe | kStrat>(k_program_eval<D, kSafe>);
    ProgEntry warp;
    warp.run = k_program_warp<D, kSafe | kStrat | kWarpTile, 1>;
    warp.run_np[0] = k_program_warp<D, kSafe | kStrat | kWarpTile, 1>;
    warp.run_np[1] = k_program_warp<D, kSafe | kStrat | kWarpTile, 2>;
    warp.run_np[2] = k_program_warp<D, kSafe | kStrat | kWarpTile, 4>;
    warp.eval = k_program_eval<D, kSafe>;
    e[D][3] = warp;
    ProgEntry lane;
    lane.run = k_program_lane<D, kSafe | kStrat | kLaneCell, 1>;
    lane.run_np[0] = k_program_lane<D, kSafe | kStrat | kLaneCell, 1>;
    lane.run_np[1] = k_program_lane<D, kSafe | kStrat | kLaneCell, 2>;
    lane.run_np[2] = k_program_lane<D, kSafe | kStrat | kLaneCell, 4>;
    lane.eval = k_program_eval<D, kSafe>;
    e[D][4] = lane;
  }
  ProgTable() {
    put<1>();
    put<2>();
    put<3>();
    put<4>();
    put<5>();
    put<6>();
    put<7>();
    put<8>();
  }
};

static const ProgTable& prog_table() {
  static const ProgTable t;
  return t;
}

// The >48 KB dynamic shared memory opt-in is per device: done once per
// device on first use (the caller has the device current).
static cudaError_t ensure_smem_optin() {
  static std::mutex mu;
  static std::set<int> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count(dev)) return cudaSuccess;
  const ProgTable& t = prog_table();
  for (int d = 1; d <= int(MCB_MAX_DIM); ++d)
    for (int v = 0; v < 5; ++v) {
      const int smem = int(program_smem_bytes(prog::kMaxDepth, d));
      if ((e = cudaFuncSetAttribute(t.e[d][v].run, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem)) != cudaSuccess)
        return e;
      for (int i = 0; i < kNpVariants; ++i)
        if (t.e[d][v].run_np[i] &&
            (e = cudaFuncSetAttribute(t.e[d][v].run_np[i], cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(program_smem_bytes(prog::kMaxDepth, d, np_of(i))))) != cudaSuccess)
          return e;
      if ((e = cudaFuncSetAttribute(t.e[d][v].eval, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem)) != cudaSuccess)
        return e;
    }
  done.insert(dev);
  return cudaSuccess;
}

// Pairs per dispatch for a group (CTA-per-tile modes 0-2): the largest NP
// whose stack + coordinates fit kInterpSmemBudget, so a few CTAs stay
// resident per SM; MCB_INTERP_NP=1|2|4 forces it (ablation).
constexpr size_t kInterpSmemBudget = 56 * 1024;
static int interp_np_index(uint32_t slots, int dim, int mode) {
  static const int forced = [] {
    const char* v = std::getenv("MCB_INTERP_NP");
    return v ? std::atoi(v) : 0;
  }();
  for (int i = kNpVariants - 1; i > 0; --i) {
    if (forced) {
      if (np_of(i) == forced) return i;
      continue;
    }
    if (program_smem_bytes(slots, dim, np_of(i)) <= kInterpSmemBudget) return i;
  }
  return 0;
}

static const ProgEntry* prog_entry(int dim, int variant) {
  if (dim < 1 || dim > int(MCB_MAX_DIM)) return nullptr;
  return &prog_table().e[dim][program_kernel_mode(variant)];
}

cudaError_t launch_program_group(const GroupLaunch& g, const FnDesc* fns, const uint32_t* tile_fn,
                                 TilePartial* part, const uint32_t* code, const double* consts,
                                 cudaStream_t s) {
  const ProgEntry* e = prog_entry(g.dim, g.variant);
  if (!e) return cudaErrorInvalidValue;
  const uint64_t per_cta = tiles_per_cta(g.variant, true);
  const uint64_t n_ctas = g.n_tiles / per_cta;
  const uint64_t kMaxGrid = 0x7FFFFFF8ull;
  if (g.prog && n_ctas <= kMaxGrid) {  // runtime-specialised kernel of this program (jit.hpp)
    const int mode = program_kernel_mode(g.variant);
    cudaError_t err = cudaSuccess;
    if (jit::launch(*g.prog, mode, uint32_t(n_ctas), g.n_tiles * g.tile_samples, fns, tile_fn, g.tile0, part, s,
                    &err))
      return err;
  }
  if (cudaError_t err = ensure_smem_optin(); err != cudaSuccess) return err;
  const int npi = interp_np_index(g.slots, g.dim, program_kernel_mode(g.variant));
  const ProgFn run = e->run_np[npi] ? e->run_np[npi] : e->run;
  const size_t smem = program_smem_bytes(g.slots, g.dim, e->run_np[npi] ? np_of(npi) : 1);
  for (uint64_t off = 0; off < n_ctas; off += kMaxGrid) {
    const uint64_t n = n_ctas - off < kMaxGrid ? n_ctas - off : kMaxGrid;
    run<<<dim3(uint32_t(n)), dim3(T), smem, s>>>(fns, tile_fn, g.tile0 + off * per_cta, part, code,
                                                   consts, g.slots);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
  }
  return cudaSuccess;
}

cudaError_t launch_program_eval(int dim, int variant, const FnDesc* fn, const uint32_t* code,
                                const double* consts, uint32_t slots, uint32_t trial, uint32_t chunk,
                                uint32_t first_pair, uint32_t n_pairs, double* out, cudaStream_t s) {
  const ProgEntry* e = prog_entry(dim, variant);
  if (!e) return cudaErrorInvalidValue;
  if (n_pairs == 0) return cudaSuccess;
  if (cudaError_t err = ensure_smem_optin(); err != cudaSuccess) return err;
  e->eval<<<(n_pairs + T - 1) / T, T, program_smem_bytes(slots, dim), s>>>(
      fn, code, consts, slots, trial, chunk, first_pair, n_pairs, out);
  return cudaGetLastError();
}

template <int D>
static cudaError_t program_points_d(const FnDesc* fn, const uint32_t* code, const double* consts,
                                    uint32_t slots, const double* pts, uint64_t n, double* out, cudaStream_t s) {
  const size_t smem = program_smem_bytes(slots, D);
  cudaError_t e = cudaFuncSetAttribute(k_program_points<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  const uint64_t pairs = (n + 1) / 2;
  k_program_points<D><<<dim3(uint32_t((pairs + T - 1) / T)), dim3(T), smem, s>>>(fn, code, consts, slots, pts, n,
                                                                                 out);
  return cudaGetLastError();
}

cudaError_t launch_program_points(int dim, const FnDesc* fn, const uint32_t* code, const double* consts,
                                  uint32_t slots, const double* pts, uint64_t n, double* out, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  switch (dim) {
    case 1: return program_points_d<1>(fn, code, consts, slots, pts, n, out, s);
    case 2: return program_points_d<2>(fn, code, consts, slots, pts, n, out, s);
    case 3: return program_points_d<3>(fn, code, consts, slots, pts, n, out, s);
    case 4: return program_points_d<4>(fn, code, consts, slots, pts, n, out, s);
    case 5: return program_points_d<5>(fn, code, consts, slots, pts, n, out, s);
    case 6: return program_points_d<6>(fn, code, consts, slots, pts, n, out, s);
    case 7: return program_points_d<7>(fn, code, consts, slots, pts, n, out, s);
    case 8: return program_points_d<8>(fn, code, consts, slots, pts, n, out, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace detail
}  // namespace mcb
