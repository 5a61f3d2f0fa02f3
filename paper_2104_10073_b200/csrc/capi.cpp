// capi.cpp — the C-ABI layer (include/mcb/mcb.h): validation, descriptor
// lowering, device plans and the multi-GPU host scheduler.
//
// Reference correspondence (file:line under /root/reference/proj):
//   mcb_validate        validate                 src/batch.cpp:62-120
//   mcb_run_direct      run_batch (Direct)       src/batch.cpp:195-333
//   mcb_direct_mc       direct_mc                src/estimator.cpp:75-92
//   mcb_tree_refine     tree_refine              src/estimator.cpp:212-318 (tree.cpp)
//   mcb_stratified_mc   stratified_mc            src/estimator.cpp:161-182
//   mcb_summarize_trials summarize_trials        src/estimator.cpp:320-337
//   mcb_stream_key      UniformStream key        src/sampling.cpp:84-87
//   mcb_volume          HyperRect::volume        src/sampling.cpp:16-20
//   mcb_debug_points    sample_uniform           src/sampling.cpp:102-112
// There is no CPU fallback: every numeric result comes from the sm_100a
// kernels in direct.cu; without a device the compute entry points return
// MCB_ERR_NO_DEVICE.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "mcb/mcb.h"
#include "mcb_internal.hpp"
#include "jit.hpp"
#include "program.hpp"
#include "tree.hpp"
#include "tree_device.cuh"

// Opaque compiled program of the C-ABI.
struct mcb_program {
  mcb::prog::Program p;
  std::vector<uint32_t> words;
};

using mcb::detail::GroupLaunch;
using mcb::dev::FnDesc;
using mcb::dev::TilePartial;

namespace {

thread_local std::string g_last_error;

mcb_status fail(mcb_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

mcb_status cuda_fail(cudaError_t e, const char* what) {
  return fail(MCB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define MCB_CUDA(call)                                   \
  do {                                                   \
    cudaError_t e_ = (call);                             \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);  \
  } while (0)

uint64_t splitmix64(uint64_t z) {  // src/sampling.cpp:44-49
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t chunk_count(uint64_t n) { return (n + MCB_CHUNK_SIZE - 1) / MCB_CHUNK_SIZE; }

template <class T>
T round_up(T v, T m) { return (v + m - 1) / m * m; }

// ---- stratified plan (ref src/batch.cpp:41-54, src/estimator.cpp:94-122) ----

// cell_grid_size: k^d, failing past the cap (CellBudgetExceeded).
bool cell_grid_size(uint32_t k, uint32_t d, uint64_t cap, uint64_t& cells) {
  if (k == 0) return false;
  cells = 1;
  for (uint32_t i = 0; i < d; ++i) {
    if (cells > cap / k + 1) return false;
    cells *= k;
  }
  return cells <= cap;
}

// auto_cells_per_dim: the largest k with k^d <= limit (at least 1).
uint32_t auto_cells_per_dim(uint32_t d, uint64_t limit) {
  uint32_t k = 1;
  for (;;) {
    uint64_t cells = 1;
    for (uint32_t i = 0; i < d; ++i) {
      cells *= uint64_t(k) + 1;
      if (cells > limit) return k;
    }
    ++k;
  }
}

struct StratPlan {
  uint32_t k = 1, spc = 2;
  uint64_t n_cells = 1;
  bool ok = false;
};

StratPlan stratified_plan(const mcb_integrand& f) {
  StratPlan p;
  const uint64_t cap = f.cell_cap ? f.cell_cap : 1000000ull;
  if (f.cells_per_dim > 0) {
    p.k = f.cells_per_dim;
  } else {
    const uint64_t limit = std::min<uint64_t>(4096, f.n_samples / 2);
    p.k = auto_cells_per_dim(f.dim, std::max<uint64_t>(limit, 1));
  }
  p.ok = cell_grid_size(p.k, f.dim, cap, p.n_cells);
  if (p.ok) p.spc = uint32_t(std::max<uint64_t>(2, f.n_samples / p.n_cells));  // as the reference
  return p;
}

bool stratified(const mcb_integrand& f) { return f.method == MCB_METHOD_STRATIFIED; }

// Samples one trial of an integrand really draws.
uint64_t trial_samples(const mcb_integrand& f) {
  if (!stratified(f)) return f.n_samples;
  const StratPlan p = stratified_plan(f);
  return p.n_cells * uint64_t(p.spc);
}

uint32_t min_dim(uint32_t family) {
  return family == MCB_FAMILY_ABS2 ? 2u : (family == MCB_FAMILY_ABS3 ? 3u : 1u);
}

bool family_known(uint32_t f) { return f <= MCB_FAMILY_PROGRAM; }

// Per-sample cost estimate (relative units) for LPT sharding: Philox blocks
// dominate (d/2 per sample), a sincos costs about one block.
double sample_cost(const mcb_integrand& f) {
  double blocks = 0.5 * double(std::max(f.dim, 1u));
  if (f.family == MCB_FAMILY_ABS2) blocks = std::min(blocks, 1.0);
  if (f.family == MCB_FAMILY_ABS3) blocks = std::min(blocks, 1.5);
  const bool harm = f.family == MCB_FAMILY_HARMONIC || f.family == MCB_FAMILY_HARMONIC_VEC;
  if (f.family == MCB_FAMILY_PROGRAM)  // interpreter: ~1 block-equivalent per 2 instructions
    return blocks + (f.program ? 0.5 * double(f.program->p.code.size()) : 1.0);
  return blocks + (harm ? 1.0 : 0.2);
}

// Reference-order evaluation on the host, used only for the shift constant
// c = f(domain midpoint) (any finite c is correct; a c near the mean keeps
// sum (f-c)^2 well conditioned, and for a constant f it makes the variance
// exactly 0 as in the reference, tests/test_estimator.cpp:44-52).
double host_eval(const mcb_integrand& f, const double* x) {
  switch (f.family) {
    case MCB_FAMILY_HARMONIC: {
      double s = x[0];
      for (uint32_t j = 1; j < f.dim; ++j) s = s + x[j];
      const double t = f.k[0] * s;
      if (f.flags & MCB_FLAG_UNIT_COEFFS) return std::cos(t) + std::sin(t);
      const double c = f.a * std::cos(t), sn = f.b * std::sin(t);
      return c + sn;
    }
    case MCB_FAMILY_HARMONIC_VEC: {
      double t = f.k[0] * x[0];
      for (uint32_t j = 1; j < f.dim; ++j) {
        const double p = f.k[j] * x[j];
        t = t + p;
      }
      const double c = f.a * std::cos(t), sn = f.b * std::sin(t);
      return c + sn;
    }
    case MCB_FAMILY_ABS2:
      return f.a * std::fabs(x[0] + x[1]);
    case MCB_FAMILY_ABS3: {
      const double s = x[0] + x[1];
      return f.a * std::fabs(s - x[2]);
    }
    case MCB_FAMILY_PROGRAM:
      return f.program ? mcb::prog::evaluate(f.program->p, x, f.k) : 0.0;
  }
  return 0.0;
}

void append_sum(std::string& s, uint32_t dim) {
  for (uint32_t j = 0; j < dim; ++j) {
    if (j) s += "+";
    s += "x" + std::to_string(j + 1);
  }
}

std::string to_dsl(const mcb_integrand& f) {
  std::string s;
  switch (f.family) {
    case MCB_FAMILY_HARMONIC: {
      std::string arg = "k*(";
      append_sum(arg, f.dim);
      arg += ")";
      if (f.flags & MCB_FLAG_UNIT_COEFFS)
        s = "cos(" + arg + ") + sin(" + arg + ")";  // src/job_io.cpp:367
      else
        s = "a*cos(" + arg + ") + b*sin(" + arg + ")";
      break;
    }
    case MCB_FAMILY_HARMONIC_VEC: {
      std::string arg;
      for (uint32_t j = 0; j < f.dim; ++j) {
        if (j) arg += "+";
        arg += "k" + std::to_string(j + 1) + "*x" + std::to_string(j + 1);
      }
      s = "a*cos(" + arg + ") + b*sin(" + arg + ")";
      break;
    }
    case MCB_FAMILY_ABS2:
      s = f.a == 1.0 ? "abs(x1+x2)" : "a*abs(x1+x2)";  // tests/test_batch.cpp:49
      break;
    case MCB_FAMILY_ABS3:
      s = f.a == 1.0 ? "abs(x1+x2-x3)" : "a*abs(x1+x2-x3)";  // tests/test_batch.cpp:51
      break;
    case MCB_FAMILY_PROGRAM:
      s = f.program ? f.program->p.source : "";
      break;
    default:
      s = "";
  }
  return s;
}

bool rect_valid(const mcb_integrand& f) {  // HyperRect::valid, src/sampling.cpp:7-14
  if (f.dim < 1 || f.dim > MCB_MAX_DIM) return false;
  for (uint32_t j = 0; j < f.dim; ++j) {
    if (!(f.low[j] < f.high[j])) return false;
    if (!std::isfinite(f.low[j]) || !std::isfinite(f.high[j])) return false;
  }
  return true;
}

double volume(const mcb_integrand& f) {  // src/sampling.cpp:16-20
  double v = 1.0;
  for (uint32_t j = 0; j < f.dim && j < MCB_MAX_DIM; ++j) v *= f.high[j] - f.low[j];
  return v;
}

void violations_of(const mcb_integrand& f, uint32_t trials,
                   std::vector<std::string>& out) {
  if (!family_known(f.family)) {
    out.push_back("unknown integrand family " + std::to_string(f.family));
    return;
  }
  if (f.family == MCB_FAMILY_PROGRAM) {
    if (!f.program) out.push_back("program family needs a compiled program");
    else if (f.program->p.dim != f.dim)
      out.push_back("program compiled for dim=" + std::to_string(f.program->p.dim) +
                    " but the integrand has dim=" + std::to_string(f.dim));
  }
  if (f.dim < 1) out.push_back("dim must be >= 1");
  if (f.dim > MCB_MAX_DIM)
    out.push_back("dim " + std::to_string(f.dim) + " exceeds the supported maximum " +
                  std::to_string(MCB_MAX_DIM));
  if (f.dim >= 1 && f.dim < min_dim(f.family))
    out.push_back("x" + std::to_string(min_dim(f.family)) +
                  " exceeds dim=" + std::to_string(f.dim));  // batch.cpp:102-105 wording
  if (f.dim >= 1 && f.dim <= MCB_MAX_DIM && !rect_valid(f))
    out.push_back("domain is invalid (need low[i] < high[i], finite, dim >= 1)");
  if (f.n_samples < 2) out.push_back("samples must be >= 2");
  if ((f.flags & MCB_FLAG_UNIT_COEFFS) &&
      !(f.family == MCB_FAMILY_HARMONIC && f.a == 1.0 && f.b == 1.0))
    out.push_back("unit-coefficient flag needs the harmonic family with a = b = 1");
  if (f.flags & ~(MCB_FLAG_UNIT_COEFFS | MCB_FLAG_REFINE_CONFIG)) out.push_back("unknown flag bits");
  if (f.method > MCB_METHOD_TREE) {
    out.push_back("unknown method " + std::to_string(f.method));
    return;
  }
  if (f.method == MCB_METHOD_TREE) {  // src/batch.cpp:94-106
    const mcb::tree::Config rc = mcb::tree::config_of(f);
    uint64_t cells;
    if (rc.init_cells_per_dim > 0 && f.dim >= 1 && f.dim <= MCB_MAX_DIM &&
        !cell_grid_size(rc.init_cells_per_dim, f.dim, rc.cell_cap, cells))
      out.push_back("cell grid exceeds configured cap");
    if (!(rc.sigma_multiplier == rc.sigma_multiplier)) out.push_back("sigma_multiplier is NaN");
    return;  // chunk indices are checked per cell at run time (MCB_TRIAL_CHUNK_RANGE)
  }
  uint64_t nc = chunk_count(f.n_samples);
  if (stratified(f) && f.dim >= 1 && f.dim <= MCB_MAX_DIM) {
    const StratPlan sp = stratified_plan(f);
    if (!sp.ok) {
      out.push_back(f.cells_per_dim == 0 && f.cell_cap == 0 ? "cells_per_dim must be >= 1"
                                                            : "cell grid exceeds configured cap");
      return;
    }
    nc = sp.n_cells * chunk_count(sp.spc);
  }
  if (nc > 0xFFFFFFFFull) out.push_back("samples exceed 2^32 chunks (chunk_index is 32-bit)");
  else if (nc * uint64_t(std::max(trials, 1u)) > 0xFFFFFFFFull)
    out.push_back("chunks x trials exceeds 2^32 work units for one integrand");
}

// ---- variant selection -----------------------------------------------------

constexpr double kTwoM64 = 0x1p-64;
constexpr double kMinFold = 0x1p-958;  // |p| * 2^-64 stays a normal double

bool foldable(double p) { return p == 0.0 || std::fabs(p) >= kMinFold; }

struct Prepared {
  FnDesc d;
  int variant;
};

// Decide the kernel variant and fill the device descriptor.  FAST variants
// need (host-proven, for every point of the domain): finite parameters,
// |t| < 2^20 for the table reduction, no overflow of f, and exact 2^-64
// folding.  Anything else runs the SAFE variant (libdevice sincos, counted
// non-finite samples) — still on the GPU.
// tree_cells: the descriptor of one tree's cells in a refinement round (the
// caller sets n_cells / spc / cpc / cell_rects / cell_est); cells are at
// least width / (k0 * 2^depth) wide, which bounds the 2^-64 fold.
Prepared prepare(const mcb_integrand& f, uint64_t seed, uint32_t chunk_base,
                 uint32_t trial_base, bool tree_cells = false) {
  using namespace mcb::detail;
  Prepared p;
  FnDesc& d = p.d;
  std::memset(&d, 0, sizeof d);
  uint32_t key[2];
  mcb_stream_key(seed, f.integrand_index, key);
  d.key0 = key[0];
  d.key1 = key[1];
  d.n_chunks = uint32_t(chunk_count(f.n_samples));
  d.dim = f.dim;
  const bool strat = stratified(f) || tree_cells;
  double cell_k = 1.0;
  if (tree_cells) {
    const mcb::tree::Config rc = mcb::tree::config_of(f);
    const uint32_t k0 = rc.init_cells_per_dim ? rc.init_cells_per_dim : auto_cells_per_dim(f.dim, 4096);
    const uint64_t splits = f.n_samples / (2ull * std::max<uint32_t>(rc.samples_per_cell, 2)) + 1;
    cell_k = double(k0) * std::ldexp(1.0, int(std::min<uint64_t>({uint64_t(rc.max_depth), splits, 2000ull})));
  } else if (strat) {  // tiles per trial = cells x chunks per cell
    const StratPlan sp = stratified_plan(f);
    d.strat_k = sp.k;
    d.n_cells = uint32_t(sp.n_cells);
    d.spc = sp.spc;
    d.cpc = uint32_t(chunk_count(sp.spc));
    d.n_chunks = d.n_cells * d.cpc;
    if (sp.spc <= kWarpTileMaxSpc) d.n_chunks = round_up(d.n_chunks, kTileAlign);  // warp per tile
    cell_k = double(sp.k);
  }
  d.chunk_base = chunk_base;
  d.trial_base = trial_base;
  d.n_samples = f.n_samples;
  d.a = f.a;
  d.b = f.b;
  d.volume = volume(f);
  bool unit_dom = true;
  double xmax = 0.0;  // bound on sum_j |x_j| (or |k_j x_j|)
  bool finite = std::isfinite(f.a) && std::isfinite(f.b);
  for (uint32_t j = 0; j < f.dim; ++j) {
    d.low[j] = f.low[j];
    d.high[j] = f.high[j];
    d.width[j] = f.high[j] - f.low[j];
    d.k[j] = f.k[j];
    if (strat || !(f.low[j] == 0.0 && f.high[j] == 1.0)) unit_dom = false;
    const double m = std::max(std::fabs(f.low[j]), std::fabs(f.high[j]));
    if (f.family == MCB_FAMILY_HARMONIC_VEC) {
      finite = finite && std::isfinite(f.k[j]);
      xmax += std::fabs(f.k[j]) * m;
    } else {
      xmax += m;
    }
  }
  if (f.family == MCB_FAMILY_HARMONIC) finite = finite && std::isfinite(f.k[0]);
  const bool unit_coef = (f.flags & MCB_FLAG_UNIT_COEFFS) != 0;
  if (f.family == MCB_FAMILY_PROGRAM) {
    // interpreter: plain parameters, unscaled draws, non-finite counting
    for (uint32_t j = 0; j < MCB_MAX_DIM; ++j) d.k[j] = f.k[j];
    p.variant = kSafe | (unit_dom ? kUnitDomain : 0) | (strat ? kStrat : 0);
    if (stratified(f) && d.spc <= kWarpTileMaxSpc) p.variant |= kWarpTile;
    if (!strat) {  // cells use a per-tile shift computed on the device
      double mid[MCB_MAX_DIM];
      for (uint32_t j = 0; j < f.dim; ++j) mid[j] = f.low[j] + 0.5 * (f.high[j] - f.low[j]);
      const double c = host_eval(f, mid);
      d.shift = std::isfinite(c) && std::fabs(c) < 1e300 ? c : 0.0;
    }
    return p;
  }
  const bool harm = f.family == MCB_FAMILY_HARMONIC || f.family == MCB_FAMILY_HARMONIC_VEC;

  bool fast = finite && std::isfinite(xmax);
  if (fast && harm) {
    const double tmax = f.family == MCB_FAMILY_HARMONIC ? std::fabs(f.k[0]) * xmax * 1.0000001
                                                        : xmax * 1.0000001;
    fast = tmax < 0x1p20 && std::fabs(f.a) + std::fabs(f.b) < 1e300;
  }
  if (fast && !harm) fast = std::fabs(f.a) * xmax < 1e300;
  // 2^-64 folding: onto the factor that multiplies the raw draw
  if (fast) {
    if (unit_dom) {
      if (f.family == MCB_FAMILY_HARMONIC) fast = foldable(f.k[0]);
      else if (f.family == MCB_FAMILY_HARMONIC_VEC)
        for (uint32_t j = 0; j < f.dim; ++j) fast = fast && foldable(f.k[j]);
      else fast = foldable(f.a);
    } else {
      // cells are >= width/k wide (the device folds each cell's width)
      for (uint32_t j = 0; j < f.dim; ++j) {
        const double w = 0.5 * d.width[j] / cell_k;
        fast = fast && w >= kMinFold && std::isfinite(w);
      }
    }
  }
  if (fast) {
    if (unit_dom) {
      if (f.family == MCB_FAMILY_HARMONIC) d.k[0] = f.k[0] * kTwoM64;
      else if (f.family == MCB_FAMILY_HARMONIC_VEC)
        for (uint32_t j = 0; j < f.dim; ++j) d.k[j] = f.k[j] * kTwoM64;
      else d.a = f.a * kTwoM64;
    } else if (!strat) {
      for (uint32_t j = 0; j < f.dim; ++j) d.width[j] = d.width[j] * kTwoM64;
    }
    p.variant = (unit_dom ? kUnitDomain : 0) | (unit_coef ? kUnitCoef : 0);
    // NOSHIFT: the argument sweeps >= 0.05 rad over the domain, so the
    // integrand is far from constant and sum f^2 - (sum f)^2/n does not
    // cancel; a (near-)constant integrand keeps the shift (exact 0 variance).
    if (harm) {
      double sweep = 0.0;
      for (uint32_t j = 0; j < f.dim; ++j)  // over one cell when stratified
        sweep += std::fabs(f.family == MCB_FAMILY_HARMONIC ? f.k[0] : f.k[j]) *
                 (f.high[j] - f.low[j]) / cell_k;
      if (sweep >= 0.05 && std::fabs(f.a) + std::fabs(f.b) > 0.0) p.variant |= kNoShift;
    }
  } else {
    p.variant = kSafe;
  }
  if (!harm) p.variant &= ~kUnitCoef;
  if (strat) p.variant |= kStrat;
  if (tree_cells) p.variant &= ~kNoShift;  // cells shrink: keep the per-tile shift
  if (stratified(f) && d.spc <= kWarpTileMaxSpc) p.variant |= kWarpTile;
  // shift constant: f at the domain midpoint (reference op order, libm);
  // cells use a per-tile shift computed on the device instead
  if (!strat) {
    double mid[MCB_MAX_DIM];
    for (uint32_t j = 0; j < f.dim; ++j) mid[j] = f.low[j] + 0.5 * (f.high[j] - f.low[j]);
    const double c = host_eval(f, mid);
    d.shift = std::isfinite(c) && std::fabs(c) < 1e300 ? c : 0.0;
  }
  if (p.variant & kNoShift) d.shift = 0.0;  // the kernel accumulates f itself
  return p;
}

}  // namespace

// ---- plans -------------------------------------------------------------------

namespace {

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

// Device checks are cached: cudaGetDeviceProperties is slow and this runs
// on every call.
mcb_status check_device(int device) {
  static std::mutex mu;
  static int count = -1;
  static std::map<int, int> major;
  std::lock_guard<std::mutex> lock(mu);
  if (count < 0) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    count = n;
  }
  if (count == 0)
    return fail(MCB_ERR_NO_DEVICE, "no CUDA device visible (the mcb path has no CPU fallback)");
  if (device < 0 || device >= count)
    return fail(MCB_ERR_INVALID_ARGUMENT, "device ordinal " + std::to_string(device) +
                                              " out of range (" + std::to_string(count) + " visible)");
  auto it = major.find(device);
  if (it == major.end()) {
    int m = 0;
    if (cudaDeviceGetAttribute(&m, cudaDevAttrComputeCapabilityMajor, device) != cudaSuccess)
      return fail(MCB_ERR_NO_DEVICE, "cannot query device");
    it = major.emplace(device, m).first;
  }
  if (it->second != 10)
    return fail(MCB_ERR_NO_DEVICE, "device " + std::to_string(device) +
                                       " is not sm_100 (this build targets sm_100a only)");
  return MCB_OK;
}

mcb_status validate_for_run(const mcb_integrand* fns, size_t n_fns, uint32_t trials) {
  if (!fns && n_fns) return fail(MCB_ERR_INVALID_ARGUMENT, "fns is NULL");
  std::vector<mcb_violation> v(16);
  size_t n = 0;
  mcb_validate(fns, n_fns, nullptr, trials, v.data(), v.size(), &n);
  if (n == 0) return MCB_OK;
  std::string msg = "job validation failed (" + std::to_string(n) + " problem(s)):";
  for (size_t i = 0; i < std::min(n, v.size()); ++i) {
    msg += "\n  ";
    if (v[i].integrand >= 0) msg += "f" + std::to_string(v[i].integrand) + ": ";
    msg += v[i].message;
  }
  return fail(MCB_ERR_VALIDATION, msg);
}

// Philox blocks one sample pair really needs (blocks holding only draws of
// coordinates a family never reads are skipped by eval_pair).
uint64_t blocks_per_pair(uint32_t family, uint32_t dim) {
  const uint32_t used = family == MCB_FAMILY_ABS2 ? 2u : (family == MCB_FAMILY_ABS3 ? 3u : dim);
  uint64_t n = 0;
  for (uint32_t i = 0; i < dim; ++i)
    if ((2 * i) % dim < used || (2 * i + 1) % dim < used) ++n;
  return n;
}

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

// chunk_bases / trial_bases (may be NULL): per-integrand key bases overriding
// chunk_base / trial_base (the tree driver's cell batches).
mcb_status build_host_plan(const mcb_integrand* fns, size_t n_fns, uint64_t seed, uint32_t trials,
                           uint32_t chunk_base, uint32_t trial_base, HostPlan& hp,
                           const uint32_t* chunk_bases = nullptr, const uint32_t* trial_bases = nullptr) {
  std::vector<Prepared> prep(n_fns);
  for (size_t i = 0; i < n_fns; ++i)
    prep[i] = prepare(fns[i], seed, chunk_bases ? chunk_bases[i] : chunk_base,
                      trial_bases ? trial_bases[i] : trial_base);
  std::vector<size_t> order(n_fns);
  std::iota(order.begin(), order.end(), size_t(0));
  // groups: (family, dim, variant), and one group per program for PROGRAM
  // integrands (each program launches its own specialised kernel)
  auto prog_key = [&](size_t i) {
    return fns[i].family == MCB_FAMILY_PROGRAM ? reinterpret_cast<uintptr_t>(fns[i].program) : uintptr_t(0);
  };
  std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) {
    auto kx = std::make_tuple(fns[x].family, fns[x].dim, prep[x].variant, prog_key(x));
    auto ky = std::make_tuple(fns[y].family, fns[y].dim, prep[y].variant, prog_key(y));
    return kx < ky;
  });
  hp.descs.resize(n_fns);
  hp.bounds_off.assign(n_fns, -1);
  std::map<const mcb_program*, std::pair<uint32_t, uint32_t>> prog_at;  // code, const offsets
  uint64_t tile = 0;
  for (size_t r = 0; r < n_fns; ++r) {
    const size_t i = order[r];
    FnDesc d = prep[i].d;
    const int fam = int(fns[i].family), dim = int(fns[i].dim), var = prep[i].variant;
    if (var & mcb::detail::kWarpTile) tile = round_up<uint64_t>(tile, mcb::detail::kTileAlign);
    d.tile_base = tile;
    d.out_slot = i;
    const uint64_t nt = uint64_t(d.n_chunks) * trials;
    uint32_t slots = 0;
    if (fam == MCB_FAMILY_PROGRAM) {
      const mcb_program* pg = fns[i].program;
      auto it = prog_at.find(pg);
      if (it == prog_at.end()) {
        it = prog_at.emplace(pg, std::make_pair(uint32_t(hp.code.size()), uint32_t(hp.consts.size()))).first;
        hp.code.insert(hp.code.end(), pg->words.begin(), pg->words.end());
        hp.consts.insert(hp.consts.end(), pg->p.consts.begin(), pg->p.consts.end());
      }
      d.prog_off = it->second.first;
      d.prog_len = uint32_t(pg->p.code.size());
      d.const_off = it->second.second;
      d.n_consts = uint32_t(pg->p.consts.size());
      slots = pg->p.depth;
    }
    const mcb::prog::Program* gp = fam == MCB_FAMILY_PROGRAM ? &fns[i].program->p : nullptr;
    if (hp.groups.empty() || hp.groups.back().family != fam || hp.groups.back().dim != dim ||
        hp.groups.back().variant != var || hp.groups.back().prog != gp)
      hp.groups.push_back(GroupLaunch{fam, dim, var, tile, 0, 0, gp});
    hp.groups.back().n_tiles += nt;
    hp.groups.back().slots = std::max(hp.groups.back().slots, slots);
    tile += nt;
    if (d.strat_k > 0) {  // grid_cell boundaries, ref src/estimator.cpp:124-143 arithmetic
      hp.bounds_off[r] = int64_t(hp.bounds.size());
      const uint32_t k = d.strat_k;
      for (uint32_t j = 0; j < fns[i].dim; ++j) {
        const double lo = fns[i].low[j], width = fns[i].high[j] - fns[i].low[j];
        for (uint32_t dg = 0; dg <= k; ++dg)
          hp.bounds.push_back(dg == 0 ? lo : (dg == k ? fns[i].high[j] : lo + width * (double(dg) / k)));
      }
    }
    hp.descs[r] = d;
    hp.total_samples += trial_samples(fns[i]) * trials;
    uint64_t pairs;
    if (d.strat_k > 0) {
      const uint64_t full = d.spc / MCB_CHUNK_SIZE, last = d.spc % MCB_CHUNK_SIZE;
      pairs = (full * (MCB_CHUNK_SIZE / 2) + (last + 1) / 2) * d.n_cells;
    } else {
      const uint64_t full = fns[i].n_samples / MCB_CHUNK_SIZE, last = fns[i].n_samples % MCB_CHUNK_SIZE;
      pairs = full * (MCB_CHUNK_SIZE / 2) + (last + 1) / 2;
    }
    hp.philox_blocks += pairs * blocks_per_pair(fns[i].family, fns[i].dim) * trials;
  }
  for (const auto& g : hp.groups)
    if (g.family != MCB_FAMILY_PROGRAM && !mcb::detail::variant_supported(g.family, g.dim, g.variant))
      return fail(MCB_ERR_INVALID_ARGUMENT, "unsupported (family, dim) combination");
  hp.n_tiles = tile;
  return MCB_OK;
}

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

// Enqueue: descriptor upload (from `staged`, pinned or not) + tile table +
// fused kernels + ordered combine, all on `s`.
// Runtime-specialised kernels of the plan's programs (jit.hpp): cache
// look-ups, and with `compile` (plans, which are relaunched) parallel
// compiles of the missing ones before the first launch.
void prepare_programs(const HostPlan& hp, bool compile) {
  using mcb::detail::kStrat;
  using mcb::detail::kUnitDomain;
  using mcb::detail::kWarpTile;
  std::vector<std::pair<const mcb::prog::Program*, int>> kernels;
  for (const auto& g : hp.groups) {
    if (!g.prog) continue;
    const int km = (g.variant & kWarpTile) ? 3 : (g.variant & kStrat) ? 2 : (g.variant & kUnitDomain) ? 1 : 0;
    const auto k = std::make_pair(g.prog, km);
    if (std::find(kernels.begin(), kernels.end(), k) == kernels.end()) kernels.push_back(k);
  }
  mcb::jit::prepare(kernels, compile);
}

mcb_status enqueue_run(const HostPlan& hp, DevBuf& buf, uint32_t trials, const FnDesc* staged,
                       bool upload, cudaStream_t s) {
  cudaError_t e;
  if (upload) prepare_programs(hp, false);
  const uint32_t n_fns = uint32_t(hp.descs.size());
  if (upload) {
    if ((e = cudaMemcpyAsync(buf.fns, staged, sizeof(FnDesc) * n_fns, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return cuda_fail(e, "cudaMemcpyAsync(descriptors)");
    if (!hp.bounds.empty() &&
        (e = cudaMemcpyAsync(buf.bounds, hp.bounds.data(), sizeof(double) * hp.bounds.size(),
                             cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return cuda_fail(e, "cudaMemcpyAsync(grid bounds)");
    if (!hp.code.empty() &&
        ((e = cudaMemcpyAsync(buf.code, hp.code.data(), sizeof(uint32_t) * hp.code.size(),
                              cudaMemcpyHostToDevice, s)) != cudaSuccess ||
         (!hp.consts.empty() &&
          (e = cudaMemcpyAsync(buf.consts, hp.consts.data(), sizeof(double) * hp.consts.size(),
                               cudaMemcpyHostToDevice, s)) != cudaSuccess)))
      return cuda_fail(e, "cudaMemcpyAsync(programs)");
    if ((e = mcb::detail::launch_expand_tiles(buf.fns, n_fns, trials, buf.tile_fn, s)) != cudaSuccess)
      return cuda_fail(e, "launch k_expand_tiles");
  }
  for (const auto& g : hp.groups) {
    if (g.family == MCB_FAMILY_PROGRAM)
      e = mcb::detail::launch_program_group(g, buf.fns, buf.tile_fn, buf.part, buf.code, buf.consts, s);
    else
      e = mcb::detail::launch_direct_group(g, buf.fns, buf.tile_fn, buf.part, s);
    if (e != cudaSuccess) return cuda_fail(e, "launch k_direct");
  }
  if ((e = mcb::detail::launch_combine(buf.fns, n_fns, trials, buf.part, buf.out, s)) != cudaSuccess)
    return cuda_fail(e, "launch k_combine");
  return MCB_OK;
}

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

DeviceCtx& device_ctx(int device) {
  static std::mutex mu;
  static std::map<int, DeviceCtx*> ctxs;  // never freed: lives for the process
  std::lock_guard<std::mutex> lock(mu);
  DeviceCtx*& c = ctxs[device];
  if (!c) c = new DeviceCtx();
  return *c;
}

template <class T>
cudaError_t grow_pinned(T*& p, size_t& cap, size_t need) {
  if (need <= cap && p) return cudaSuccess;
  if (p) cudaFreeHost(p);
  p = nullptr;
  cap = 0;
  const size_t n = std::max<size_t>(need, 1);
  cudaError_t e = cudaMallocHost(&p, sizeof(T) * n);
  if (e == cudaSuccess) cap = n;
  return e;
}

// One shard of mcb_run_direct on one device (synchronous).
mcb_status run_shard(const mcb_integrand* fns, size_t n_fns, uint64_t seed, uint32_t trials,
                     int device, mcb_trial_stats* out, const uint32_t* chunk_bases = nullptr,
                     const uint32_t* trial_bases = nullptr) {
  HostPlan hp;
  const auto tb0 = std::chrono::steady_clock::now();
  mcb_status st = build_host_plan(fns, n_fns, seed, trials, 0, 0, hp, chunk_bases, trial_bases);
  if (st != MCB_OK) return st;
  static const bool trace = [] {
    const char* e = std::getenv("MCB_TREE_TRACE");
    return e && *e && *e != '0';
  }();
  if (trace)
    std::fprintf(stderr, "[mcb shard] dev %d: %zu fns, %llu tiles, host plan %.3f ms\n", device, n_fns,
                 (unsigned long long)hp.n_tiles,
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tb0).count());
  DeviceCtx& c = device_ctx(device);
  std::lock_guard<std::mutex> lock(c.mu);
  DeviceGuard guard(device);
  cudaError_t e;
  if (!c.ready) {
    if ((e = cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamCreate");
    c.ready = true;
  }
  const size_t n_out = n_fns * trials;
  if ((e = c.buf.reserve(n_fns, hp.n_tiles, n_out, hp.code.size(), hp.consts.size())) != cudaSuccess)
    return cuda_fail(e, "cudaMalloc");
  if ((e = grow_pinned(c.h_descs, c.h_descs_cap, n_fns)) != cudaSuccess) return cuda_fail(e, "cudaMallocHost");
  if ((e = grow_pinned(c.h_out, c.h_out_cap, n_out)) != cudaSuccess) return cuda_fail(e, "cudaMallocHost");
  if ((e = DevBuf::grow(c.buf.bounds, c.buf.cap_bounds, hp.bounds.size())) != cudaSuccess)
    return cuda_fail(e, "cudaMalloc");
  std::memcpy(c.h_descs, hp.descs.data(), sizeof(FnDesc) * n_fns);
  for (size_t r = 0; r < n_fns; ++r)
    if (hp.bounds_off[r] >= 0) c.h_descs[r].grid_bounds = c.buf.bounds + hp.bounds_off[r];
  if ((st = enqueue_run(hp, c.buf, trials, c.h_descs, true, c.stream)) != MCB_OK) return st;
  if ((e = cudaMemcpyAsync(c.h_out, c.buf.out, sizeof(mcb_trial_stats) * n_out, cudaMemcpyDeviceToHost,
                           c.stream)) != cudaSuccess)
    return cuda_fail(e, "cudaMemcpyAsync(results)");
  if ((e = cudaStreamSynchronize(c.stream)) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  std::memcpy(out, c.h_out, sizeof(mcb_trial_stats) * n_out);
  return MCB_OK;
}

// One device's share of a tree round: a cell-list descriptor per batch
// (prepared as the tree's integrand, cells from the rectangle table), the
// fused kernels in cell-list mode, per-cell estimates back to the batches.
mcb_status run_cell_shard(const std::vector<const mcb::tree::CellBatch*>& batches, uint64_t seed,
                          int device) {
  const size_t n = batches.size();
  using clk = std::chrono::steady_clock;
  const auto t_start = clk::now();
  HostPlan hp;
  std::vector<Prepared> prep(n);
  size_t n_rects = 0, n_cells = 0;
  std::map<const mcb_integrand*, Prepared> base;  // one prepare per integrand (its trials share it)
  for (size_t i = 0; i < n; ++i) {
    const mcb::tree::CellBatch& b = *batches[i];
    auto it = base.find(b.fn);
    if (it == base.end()) it = base.emplace(b.fn, prepare(*b.fn, seed, 0, 0, true)).first;
    prep[i] = it->second;
    prep[i].d.chunk_base = uint32_t(b.chunk_base);
    prep[i].d.trial_base = b.trial;
    if (b.spc <= mcb::detail::kWarpTileMaxSpc) prep[i].variant |= mcb::detail::kWarpTile;
    n_rects += size_t(b.n_cells) * 2 * b.fn->dim;
    n_cells += b.n_cells;
  }
  std::vector<size_t> order(n);
  std::iota(order.begin(), order.end(), size_t(0));
  auto prog_key = [&](size_t i) {
    return batches[i]->fn->family == MCB_FAMILY_PROGRAM ? reinterpret_cast<uintptr_t>(batches[i]->fn->program)
                                                        : uintptr_t(0);
  };
  std::stable_sort(order.begin(), order.end(), [&](size_t x, size_t y) {
    return std::make_tuple(batches[x]->fn->family, batches[x]->fn->dim, prep[x].variant, prog_key(x)) <
           std::make_tuple(batches[y]->fn->family, batches[y]->fn->dim, prep[y].variant, prog_key(y));
  });
  uint64_t tiles = 0;  // upper bound incl. warp-tile padding and alignment
  for (size_t i = 0; i < n; ++i)
    tiles += uint64_t(batches[i]->n_cells) * chunk_count(batches[i]->spc) + 2 * mcb::detail::kTileAlign;

  DeviceCtx& c = device_ctx(device);
  std::lock_guard<std::mutex> lock(c.mu);
  DeviceGuard guard(device);
  cudaError_t e;
  if (!c.ready) {
    if ((e = cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamCreate");
    c.ready = true;
  }
  // program tables first (sizes), then buffers, then descriptors with device addresses
  std::map<const mcb_program*, std::pair<uint32_t, uint32_t>> prog_at;
  for (size_t i = 0; i < n; ++i) {
    const mcb_program* pg = batches[i]->fn->program;
    if (batches[i]->fn->family != MCB_FAMILY_PROGRAM || prog_at.count(pg)) continue;
    prog_at.emplace(pg, std::make_pair(uint32_t(hp.code.size()), uint32_t(hp.consts.size())));
    hp.code.insert(hp.code.end(), pg->words.begin(), pg->words.end());
    hp.consts.insert(hp.consts.end(), pg->p.consts.begin(), pg->p.consts.end());
  }
  if ((e = c.buf.reserve(n, tiles, n, hp.code.size(), hp.consts.size())) != cudaSuccess ||
      (e = DevBuf::grow(c.buf.rects, c.buf.cap_rects, n_rects)) != cudaSuccess ||
      (e = DevBuf::grow(c.buf.cell_est, c.buf.cap_cell_est, n_cells)) != cudaSuccess)
    return cuda_fail(e, "cudaMalloc");
  if ((e = grow_pinned(c.h_descs, c.h_descs_cap, n)) != cudaSuccess ||
      (e = grow_pinned(c.h_rects, c.h_rects_cap, n_rects)) != cudaSuccess ||
      (e = grow_pinned(c.h_cell_est, c.h_cell_est_cap, n_cells)) != cudaSuccess)
    return cuda_fail(e, "cudaMallocHost");
  hp.descs.resize(n);
  std::vector<size_t> est_at(n);
  uint64_t tile = 0;
  size_t rect_at = 0, cell_at = 0;
  for (size_t r = 0; r < n; ++r) {
    const size_t i = order[r];
    const mcb::tree::CellBatch& b = *batches[i];
    FnDesc d = prep[i].d;
    d.strat_k = 0;
    d.n_cells = b.n_cells;
    d.spc = b.spc;
    d.cpc = uint32_t(chunk_count(b.spc));
    d.n_chunks = d.n_cells * d.cpc;
    d.n_samples = uint64_t(b.n_cells) * b.spc;
    if (prep[i].variant & mcb::detail::kWarpTile) {
      d.n_chunks = round_up<uint32_t>(d.n_chunks, mcb::detail::kTileAlign);
      tile = round_up<uint64_t>(tile, mcb::detail::kTileAlign);
    }
    d.tile_base = tile;
    d.out_slot = r;
    d.cell_rects = c.buf.rects + rect_at;
    d.cell_est = c.buf.cell_est + cell_at;
    const size_t nr = size_t(b.n_cells) * 2 * b.fn->dim;
    std::memcpy(c.h_rects + rect_at, b.rects, sizeof(double) * nr);
    est_at[i] = cell_at;
    rect_at += nr;
    cell_at += b.n_cells;
    const int fam = int(b.fn->family), dim = int(b.fn->dim), var = prep[i].variant;
    uint32_t slots = 0;
    if (fam == MCB_FAMILY_PROGRAM) {
      const auto& at = prog_at.at(b.fn->program);
      d.prog_off = at.first;
      d.prog_len = uint32_t(b.fn->program->p.code.size());
      d.const_off = at.second;
      d.n_consts = uint32_t(b.fn->program->p.consts.size());
      slots = b.fn->program->p.depth;
    }
    const mcb::prog::Program* gp = fam == MCB_FAMILY_PROGRAM ? &b.fn->program->p : nullptr;
    if (hp.groups.empty() || hp.groups.back().family != fam || hp.groups.back().dim != dim ||
        hp.groups.back().variant != var || hp.groups.back().prog != gp)
      hp.groups.push_back(GroupLaunch{fam, dim, var, tile, 0, 0, gp});
    hp.groups.back().n_tiles += d.n_chunks;
    hp.groups.back().slots = std::max(hp.groups.back().slots, slots);
    tile += d.n_chunks;
    hp.descs[r] = d;
  }
  hp.n_tiles = tile;
  for (const auto& g : hp.groups)
    if (g.family != MCB_FAMILY_PROGRAM && !mcb::detail::variant_supported(g.family, g.dim, g.variant))
      return fail(MCB_ERR_INVALID_ARGUMENT, "unsupported (family, dim) combination");
  std::memcpy(c.h_descs, hp.descs.data(), sizeof(FnDesc) * n);
  const auto t_host = clk::now();
  if (n_rects &&
      (e = cudaMemcpyAsync(c.buf.rects, c.h_rects, sizeof(double) * n_rects, cudaMemcpyHostToDevice,
                           c.stream)) != cudaSuccess)
    return cuda_fail(e, "cudaMemcpyAsync(cells)");
  mcb_status st = enqueue_run(hp, c.buf, 1, c.h_descs, true, c.stream);
  if (st != MCB_OK) return st;
  if ((e = cudaMemcpyAsync(c.h_cell_est, c.buf.cell_est, sizeof(mcb::CellEst) * n_cells,
                           cudaMemcpyDeviceToHost, c.stream)) != cudaSuccess)
    return cuda_fail(e, "cudaMemcpyAsync(cell estimates)");
  if ((e = cudaStreamSynchronize(c.stream)) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  const auto t_gpu = clk::now();
  for (size_t i = 0; i < n; ++i)
    std::memcpy(batches[i]->est, c.h_cell_est + est_at[i], sizeof(mcb::CellEst) * batches[i]->n_cells);
  static const bool trace = [] {
    const char* env = std::getenv("MCB_TREE_TRACE");
    return env && *env && *env != '0';
  }();
  if (trace) {
    auto ms = [](clk::time_point a, clk::time_point b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[mcb cells] dev %d: %zu batches, %zu cells: host %.3f ms, H2D+kernels+D2H %.3f ms, scatter %.3f ms\n",
                 device, n, n_cells, ms(t_start, t_host), ms(t_host, t_gpu), ms(t_gpu, clk::now()));
  }
  return MCB_OK;
}

// tree_refine's first-pass grid (src/estimator.cpp:219-231): cells per dim
// and cell count; false = CellBudgetExceeded.
bool tree_first_pass(const mcb_integrand& f, const mcb::tree::Config& cfg, uint32_t spc, uint32_t& k,
                     uint64_t& n0) {
  k = cfg.init_cells_per_dim;
  if (k == 0) {
    k = auto_cells_per_dim(f.dim, 4096);
    while (k > 1) {
      uint64_t cells;
      if (!cell_grid_size(k, f.dim, cfg.cell_cap, cells)) return false;
      if (cells * spc <= cfg.total_budget / 2) break;
      --k;
    }
  }
  return cell_grid_size(k, f.dim, cfg.cell_cap, n0);
}

// Most leaves a tree can reach: one per split the budget allows past the
// first pass, and at most 2^max_depth per first-pass cell.
uint64_t tree_leaf_bound(uint64_t n0, uint32_t spc, const mcb::tree::Config& cfg) {
  const uint64_t first = n0 * spc;
  const uint64_t splits = cfg.total_budget >= first ? (cfg.total_budget - first) / (2ull * spc) : 0;
  const uint64_t by_depth = cfg.max_depth >= 40 ? ~0ull : n0 << cfg.max_depth;
  return std::min(n0 + splits, std::max(n0, by_depth));
}

// Device-resident tree_refine for `tasks` on one device (tree_device.cuh):
// the host builds each tree's first-pass grid and constants once; every
// round then runs on the GPU with one small read-back (the launch groups'
// tile ranges).  Results are those of the host driver (tree.cpp).
mcb_status run_trees_device(std::vector<mcb::tree::TreeTask*>& tasks, uint64_t seed, int device) {
  using namespace mcb::detail;
  using mcb::tdev::TreeConst;
  using mcb::tdev::TreeState;
  const size_t T = tasks.size();
  if (T == 0) return MCB_OK;
  // ---- host: configs, first-pass grids, descriptors, launch groups ----
  struct HostTree {
    mcb::tree::Config cfg;
    uint32_t k = 0, spc = 0, cpc = 0, fail = 0;
    uint64_t n0 = 0, cap = 0;
    Prepared prep;
  };
  std::vector<HostTree> ht(T);
  for (size_t i = 0; i < T; ++i) {
    const mcb_integrand& f = *tasks[i]->fn;
    HostTree& h = ht[i];
    h.cfg = mcb::tree::config_of(f);
    h.spc = std::max<uint32_t>(h.cfg.samples_per_cell, 2);
    h.cpc = uint32_t(chunk_count(h.spc));
    uint32_t k = 0;
    if (!tree_first_pass(f, h.cfg, h.spc, k, h.n0)) {
      h.fail = MCB_TRIAL_CELL_BUDGET;
      h.n0 = 0;
    } else if (tasks[i]->chunk_base + h.n0 * h.cpc - 1 > 0xFFFFFFFFull) {
      h.fail = MCB_TRIAL_CHUNK_RANGE;
      h.n0 = 0;
    }
    h.k = k;
    h.cap = tree_leaf_bound(h.n0, h.spc, h.cfg) + 1;
    if (h.cap > 0xFFFFFFFFull) return fail(MCB_ERR_INVALID_ARGUMENT, "tree budget too large for one device run");
    h.prep = prepare(f, seed, 0, tasks[i]->trial, true);
    if (h.spc <= kWarpTileMaxSpc) h.prep.variant |= kWarpTile;
  }
  std::vector<size_t> order(T);  // launch groups: (family, dim, variant, program)
  std::iota(order.begin(), order.end(), size_t(0));
  auto key = [&](size_t i) {
    const mcb_integrand& f = *tasks[i]->fn;
    return std::make_tuple(f.family, f.dim, ht[i].prep.variant,
                           f.family == MCB_FAMILY_PROGRAM ? reinterpret_cast<uintptr_t>(f.program) : uintptr_t(0));
  };
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return key(a) < key(b); });
  HostPlan hp;
  std::vector<TreeConst> tc(T);
  std::vector<TreeState> tst(T);
  std::map<const mcb_program*, std::pair<uint32_t, uint32_t>> prog_at;
  uint64_t leaves = 0, rect_doubles = 0, max_tiles = 0;
  hp.descs.resize(T);
  for (size_t r = 0; r < T; ++r) {
    const size_t i = order[r];
    const mcb_integrand& f = *tasks[i]->fn;
    HostTree& h = ht[i];
    const int fam = int(f.family), dim = int(f.dim), var = h.prep.variant;
    const mcb::prog::Program* gp = fam == MCB_FAMILY_PROGRAM ? &f.program->p : nullptr;
    if (hp.groups.empty() || hp.groups.back().family != fam || hp.groups.back().dim != dim ||
        hp.groups.back().variant != var || hp.groups.back().prog != gp)
      hp.groups.push_back(GroupLaunch{fam, dim, var, 0, 0, 0, gp});
    FnDesc d = h.prep.d;
    d.strat_k = 0;
    d.spc = h.spc;
    d.cpc = h.cpc;
    d.out_slot = r;
    if (fam == MCB_FAMILY_PROGRAM) {
      auto it = prog_at.find(f.program);
      if (it == prog_at.end()) {
        it = prog_at.emplace(f.program, std::make_pair(uint32_t(hp.code.size()), uint32_t(hp.consts.size()))).first;
        hp.code.insert(hp.code.end(), f.program->words.begin(), f.program->words.end());
        hp.consts.insert(hp.consts.end(), f.program->p.consts.begin(), f.program->p.consts.end());
      }
      d.prog_off = it->second.first;
      d.prog_len = uint32_t(f.program->p.code.size());
      d.const_off = it->second.second;
      d.n_consts = uint32_t(f.program->p.consts.size());
      hp.groups.back().slots = std::max(hp.groups.back().slots, f.program->p.depth);
    }
    hp.descs[r] = d;
    TreeConst& c = tc[r];
    c.leaf_off = leaves;
    c.rect_off = rect_doubles;
    c.budget = h.cfg.total_budget;
    c.sigma = h.cfg.sigma_multiplier;
    c.leaf_cap = uint32_t(h.cap);
    c.dim = f.dim;
    c.spc = h.spc;
    c.cpc = h.cpc;
    c.max_depth = h.cfg.max_depth;
    c.warp_tiles = (var & kWarpTile) ? 1u : 0u;
    c.group = uint32_t(hp.groups.size() - 1);
    c.reserved = 0;
    TreeState& st = tst[r];
    std::memset(&st, 0, sizeof st);
    st.fail = h.fail;
    st.n_leaves = uint32_t(h.n0);
    st.n_new = uint32_t(h.n0);
    st.active = h.fail ? 0u : 1u;
    st.chunk0 = tasks[i]->chunk_base;
    st.next_chunk = tasks[i]->chunk_base + h.n0 * h.cpc;
    st.used = h.n0 * h.spc;
    leaves += h.cap;
    rect_doubles += h.cap * 2 * f.dim;
    max_tiles += (h.cap * h.cpc + kTileAlign - 1) / kTileAlign * kTileAlign;
  }
  max_tiles += kTileAlign * hp.groups.size();
  if (hp.groups.size() > 256) return fail(MCB_ERR_INVALID_ARGUMENT, "too many distinct tree kernels in one run");
  for (const auto& g : hp.groups)
    if (g.family != MCB_FAMILY_PROGRAM && !variant_supported(g.family, g.dim, g.variant))
      return fail(MCB_ERR_INVALID_ARGUMENT, "unsupported (family, dim) combination");
  // first-pass grids (grid_cell, src/estimator.cpp:124-143) = the initial
  // leaves and round-0 cells, packed tree after tree (k_tree_init spreads them)
  uint64_t packed_doubles = 0;
  for (size_t r = 0; r < T; ++r) {
    tc[r].init_off = packed_doubles;
    packed_doubles += uint64_t(tst[r].n_leaves) * 2 * tc[r].dim;
  }
  DeviceCtx& c = device_ctx(device);
  std::lock_guard<std::mutex> lock(c.mu);
  DeviceGuard guard(device);
  cudaError_t e;
  if ((e = grow_pinned(c.h_rects, c.h_rects_cap, packed_doubles)) != cudaSuccess)
    return cuda_fail(e, "cudaMallocHost");
  for (size_t r = 0; r < T; ++r) {
    const size_t i = order[r];
    const mcb_integrand& f = *tasks[i]->fn;
    const uint32_t k = ht[i].k, D = f.dim;
    for (uint64_t cell = 0; cell < ht[i].n0; ++cell) {
      double* lo = c.h_rects + tc[r].init_off + 2 * D * cell;
      double* hi = lo + D;
      uint64_t rem = cell;
      for (uint32_t j = D; j-- > 0;) {
        const uint32_t digit = uint32_t(rem % k);
        rem /= k;
        const double width = f.high[j] - f.low[j];
        lo[j] = digit == 0 ? f.low[j] : f.low[j] + width * (double(digit) / k);
        hi[j] = digit + 1 == k ? f.high[j] : f.low[j] + width * (double(digit + 1) / k);
      }
    }
  }
  // ---- device ----
  if (!c.ready) {
    if ((e = cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "cudaStreamCreate");
    c.ready = true;
  }
  const cudaStream_t s = c.stream;
  if ((e = c.buf.reserve(T, max_tiles, T, hp.code.size(), hp.consts.size())) != cudaSuccess ||
      (e = DevBuf::grow(c.t_const, c.cap_trees, T)) != cudaSuccess ||
      (e = DevBuf::grow(c.t_state, c.cap_tstate, T)) != cudaSuccess)
    return cuda_fail(e, "cudaMalloc");
  if ((e = DevBuf::grow(c.t_groups, c.cap_tgroups, 2 * hp.groups.size())) != cudaSuccess ||
      (e = DevBuf::grow(c.l_rect, c.cap_rect, rect_doubles)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_new_rect, c.cap_new_rect, rect_doubles)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_se, c.cap_se, leaves)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_val, c.cap_val, leaves)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_nn, c.cap_nn, leaves)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_depth, c.cap_depth, leaves)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_dead, c.cap_dead, leaves)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_new_leaf, c.cap_new_leaf, leaves)) != cudaSuccess ||
      (e = DevBuf::grow(c.l_est, c.cap_est, leaves)) != cudaSuccess)
    return cuda_fail(e, "cudaMalloc");
  mcb::tdev::Leaves L{c.l_rect, c.l_se, c.l_val, c.l_nn, c.l_depth, c.l_dead, c.l_new_leaf, c.l_new_rect, c.l_est};
  auto up = [&](void* dst, const void* src, size_t bytes) {
    return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s) : cudaSuccess;
  };
  if ((e = up(c.t_const, tc.data(), sizeof(TreeConst) * T)) != cudaSuccess ||
      (e = up(c.t_state, tst.data(), sizeof(TreeState) * T)) != cudaSuccess ||
      (e = up(c.buf.fns, hp.descs.data(), sizeof(FnDesc) * T)) != cudaSuccess ||
      (e = DevBuf::grow(c.buf.rects, c.buf.cap_rects, packed_doubles)) != cudaSuccess ||
      (e = up(c.buf.rects, c.h_rects, sizeof(double) * packed_doubles)) != cudaSuccess ||
      (e = launch_tree_init(c.t_const, c.t_state, L, c.buf.rects, uint32_t(T), s)) != cudaSuccess ||
      (!hp.code.empty() && (e = up(c.buf.code, hp.code.data(), sizeof(uint32_t) * hp.code.size())) != cudaSuccess) ||
      (!hp.consts.empty() && (e = up(c.buf.consts, hp.consts.data(), sizeof(double) * hp.consts.size())) != cudaSuccess))
    return cuda_fail(e, "cudaMemcpyAsync(tree setup)");
  prepare_programs(hp, false);
  std::vector<uint64_t> gt(2 * hp.groups.size());
  for (int round = 0;; ++round) {
    if (round > 0 && (e = launch_tree_select(c.t_const, c.t_state, L, uint32_t(T), s)) != cudaSuccess)
      return cuda_fail(e, "launch k_tree_select");
    if ((e = launch_tree_layout(c.t_const, c.t_state, c.buf.fns, L, uint32_t(T), c.t_groups,
                                uint32_t(hp.groups.size()), s)) != cudaSuccess)
      return cuda_fail(e, "launch k_tree_layout");
    if ((e = cudaMemcpyAsync(gt.data(), c.t_groups, sizeof(uint64_t) * gt.size(), cudaMemcpyDeviceToHost, s)) !=
            cudaSuccess ||
        (e = cudaStreamSynchronize(s)) != cudaSuccess)
      return cuda_fail(e, "tree round read-back");
    uint64_t tiles = 0;
    for (size_t g = 0; g < hp.groups.size(); ++g) tiles += gt[2 * g + 1];
    if (tiles == 0) break;
    if ((e = launch_expand_tiles(c.buf.fns, uint32_t(T), 1, c.buf.tile_fn, s)) != cudaSuccess)
      return cuda_fail(e, "launch k_expand_tiles");
    for (size_t g = 0; g < hp.groups.size(); ++g) {
      if (gt[2 * g + 1] == 0) continue;
      GroupLaunch gl = hp.groups[g];
      gl.tile0 = gt[2 * g];
      gl.n_tiles = gt[2 * g + 1];
      e = gl.family == MCB_FAMILY_PROGRAM
              ? launch_program_group(gl, c.buf.fns, c.buf.tile_fn, c.buf.part, c.buf.code, c.buf.consts, s)
              : launch_direct_group(gl, c.buf.fns, c.buf.tile_fn, c.buf.part, s);
      if (e != cudaSuccess) return cuda_fail(e, "launch tree cells");
    }
    if ((e = launch_combine(c.buf.fns, uint32_t(T), 1, c.buf.part, c.buf.out, s)) != cudaSuccess ||
        (e = launch_tree_scatter(c.t_const, c.t_state, L, uint32_t(T), s)) != cudaSuccess)
      return cuda_fail(e, "launch tree combine/scatter");
  }
  if ((e = launch_tree_finish(c.t_const, c.t_state, L, uint32_t(T), c.buf.out, s)) != cudaSuccess)
    return cuda_fail(e, "launch k_tree_finish");
  std::vector<mcb_trial_stats> out(T);
  if ((e = cudaMemcpyAsync(out.data(), c.buf.out, sizeof(mcb_trial_stats) * T, cudaMemcpyDeviceToHost, s)) !=
      cudaSuccess)
    return cuda_fail(e, "cudaMemcpyAsync(tree results)");
  bool want_leaves = false;
  for (auto* t : tasks) want_leaves = want_leaves || t->leaves;
  std::vector<double> h_rect, h_se, h_val;
  std::vector<uint32_t> h_nn, h_depth, h_dead;
  if (want_leaves) {
    h_rect.resize(rect_doubles);
    h_se.resize(leaves);
    h_val.resize(leaves);
    h_nn.resize(leaves);
    h_depth.resize(leaves);
    h_dead.resize(leaves);
    if ((e = cudaMemcpyAsync(h_rect.data(), c.l_rect, sizeof(double) * rect_doubles, cudaMemcpyDeviceToHost, s)) !=
            cudaSuccess ||
        (e = cudaMemcpyAsync(h_se.data(), c.l_se, sizeof(double) * leaves, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaMemcpyAsync(h_val.data(), c.l_val, sizeof(double) * leaves, cudaMemcpyDeviceToHost, s)) !=
            cudaSuccess ||
        (e = cudaMemcpyAsync(h_nn.data(), c.l_nn, sizeof(uint32_t) * leaves, cudaMemcpyDeviceToHost, s)) !=
            cudaSuccess ||
        (e = cudaMemcpyAsync(h_depth.data(), c.l_depth, sizeof(uint32_t) * leaves, cudaMemcpyDeviceToHost, s)) !=
            cudaSuccess ||
        (e = cudaMemcpyAsync(h_dead.data(), c.l_dead, sizeof(uint32_t) * leaves, cudaMemcpyDeviceToHost, s)) !=
            cudaSuccess)
      return cuda_fail(e, "cudaMemcpyAsync(leaves)");
  }
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  for (size_t r = 0; r < T; ++r) {
    mcb::tree::TreeTask& task = *tasks[order[r]];
    *task.out = out[r];
    if (!task.leaves) continue;
    task.leaves->clear();
    if (out[r].status != MCB_TRIAL_OK) continue;  // leaves_out is written only when tree_refine returns
    const uint32_t D = task.fn->dim, spc = tc[r].spc;
    for (uint32_t i = 0; i < out[r].n_cells; ++i) {
      const uint64_t l = tc[r].leaf_off + i;
      mcb_leaf m;
      std::memset(&m, 0, sizeof m);
      std::memcpy(m.low, h_rect.data() + tc[r].rect_off + 2 * D * i, sizeof(double) * D);
      std::memcpy(m.high, h_rect.data() + tc[r].rect_off + 2 * D * i + D, sizeof(double) * D);
      m.depth = h_depth[l];
      mcb_trial_stats& est = m.estimate;
      est.n_samples = spc;
      est.n_nonfinite = h_nn[l];
      est.n_cells = 1;
      if (h_dead[l]) {
        est.status = MCB_TRIAL_ALL_NONFINITE;
        est.nonfinite_warning = 1;
      } else {
        est.value = h_val[l];
        est.std_error = h_se[l];
        est.nonfinite_warning = double(h_nn[l]) > MCB_NONFINITE_WARN_FRACTION * double(spc) ? 1u : 0u;
      }
      task.leaves->push_back(m);
    }
  }
  return MCB_OK;
}

}  // namespace

struct mcb_plan {
  int device = 0;
  uint64_t n_fns = 0;
  uint32_t trials = 0;
  HostPlan hp;
  DevBuf buf;
};

namespace {

mcb_status plan_create_impl(const mcb_integrand* fns, size_t n_fns, uint64_t seed,
                            uint32_t trials, int device, uint32_t chunk_base,
                            uint32_t trial_base, mcb_plan** out) {
  mcb_status st = validate_for_run(fns, n_fns, trials);
  if (st != MCB_OK) return st;
  for (size_t i = 0; i < n_fns; ++i)
    if (fns[i].method == MCB_METHOD_TREE)
      return fail(MCB_ERR_INVALID_ARGUMENT,
                  "method tree has no static plan (use mcb_run_direct or mcb_tree_refine)");
  if (chunk_base) {
    for (size_t i = 0; i < n_fns; ++i)
      if (uint64_t(chunk_base) + chunk_count(fns[i].n_samples) - 1 > 0xFFFFFFFFull)
        return fail(MCB_ERR_OUT_OF_RANGE, "chunk_index exceeds 32 bits");
  }
  if ((st = check_device(device)) != MCB_OK) return st;
  auto plan = new mcb_plan();
  plan->device = device;
  plan->n_fns = n_fns;
  plan->trials = trials;
  if ((st = build_host_plan(fns, n_fns, seed, trials, chunk_base, trial_base, plan->hp)) != MCB_OK) {
    delete plan;
    return st;
  }
  DeviceGuard guard(device);
  cudaError_t e = plan->buf.reserve(n_fns, plan->hp.n_tiles, n_fns * trials, plan->hp.code.size(),
                                    plan->hp.consts.size());
  if (e == cudaSuccess) e = DevBuf::grow(plan->buf.bounds, plan->buf.cap_bounds, plan->hp.bounds.size());
  if (e == cudaSuccess && !plan->hp.bounds.empty())
    e = cudaMemcpy(plan->buf.bounds, plan->hp.bounds.data(), sizeof(double) * plan->hp.bounds.size(),
                   cudaMemcpyHostToDevice);
  for (size_t r = 0; r < n_fns; ++r)
    if (plan->hp.bounds_off[r] >= 0) plan->hp.descs[r].grid_bounds = plan->buf.bounds + plan->hp.bounds_off[r];
  if (e == cudaSuccess)
    e = cudaMemcpy(plan->buf.fns, plan->hp.descs.data(), sizeof(FnDesc) * n_fns, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !plan->hp.code.empty())
    e = cudaMemcpy(plan->buf.code, plan->hp.code.data(), sizeof(uint32_t) * plan->hp.code.size(),
                   cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !plan->hp.consts.empty())
    e = cudaMemcpy(plan->buf.consts, plan->hp.consts.data(), sizeof(double) * plan->hp.consts.size(),
                   cudaMemcpyHostToDevice);
  if (e == cudaSuccess) prepare_programs(plan->hp, true);
  if (e == cudaSuccess)
    e = mcb::detail::launch_expand_tiles(plan->buf.fns, uint32_t(n_fns), trials, plan->buf.tile_fn, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    mcb_plan_destroy(plan);
    return cuda_fail(e, "plan setup");
  }
  *out = plan;
  return MCB_OK;
}

mcb_status plan_launch_impl(mcb_plan* plan, cudaStream_t s) {
  DeviceGuard guard(plan->device);
  return enqueue_run(plan->hp, plan->buf, plan->trials, nullptr, false, s);
}

mcb_status plan_download_impl(mcb_plan* plan, mcb_trial_stats* out, cudaStream_t s) {
  DeviceGuard guard(plan->device);
  MCB_CUDA(cudaMemcpyAsync(out, plan->buf.out, sizeof(mcb_trial_stats) * plan->n_fns * plan->trials,
                           cudaMemcpyDeviceToHost, s));
  MCB_CUDA(cudaStreamSynchronize(s));
  return MCB_OK;
}

// LPT: integrands by decreasing cost onto the least-loaded shard.
void lpt(const mcb_integrand* fns, size_t n, uint32_t trials, int shards, uint32_t* shard_of) {
  std::vector<size_t> order(n);
  std::iota(order.begin(), order.end(), size_t(0));
  std::vector<double> cost(n);
  for (size_t i = 0; i < n; ++i)
    cost[i] = double(trial_samples(fns[i])) * double(trials) * sample_cost(fns[i]);
  std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return cost[a] > cost[b]; });
  std::vector<double> load(size_t(shards), 0.0);
  for (size_t i : order) {
    size_t best = 0;
    for (size_t s = 1; s < load.size(); ++s)
      if (load[s] < load[best]) best = s;
    shard_of[i] = uint32_t(best);
    load[best] += cost[i];
  }
}

// Shards integrands over `devs` by LPT, one host thread per device; results
// land in `out` (n_fns * trials) by integrand.  Byte-identical for any list.
mcb_status run_sharded(const mcb_integrand* fns, size_t n_fns, uint64_t seed, uint32_t trials,
                       const std::vector<int>& devs, mcb_trial_stats* out, const uint32_t* chunk_bases,
                       const uint32_t* trial_bases) {
  std::vector<uint32_t> shard(n_fns, 0);
  lpt(fns, n_fns, trials, int(devs.size()), shard.data());
  std::vector<mcb_status> status(devs.size(), MCB_OK);
  std::vector<std::string> errors(devs.size());
  auto work = [&](size_t w) {
    std::vector<size_t> mine;
    for (size_t i = 0; i < n_fns; ++i)
      if (shard[i] == w) mine.push_back(i);
    if (mine.empty()) return;
    std::vector<mcb_integrand> sub(mine.size());
    std::vector<uint32_t> cb, tb;
    for (size_t r = 0; r < mine.size(); ++r) sub[r] = fns[mine[r]];
    if (chunk_bases)
      for (size_t i : mine) cb.push_back(chunk_bases[i]);
    if (trial_bases)
      for (size_t i : mine) tb.push_back(trial_bases[i]);
    std::vector<mcb_trial_stats> res(sub.size() * trials);
    const mcb_status s = run_shard(sub.data(), sub.size(), seed, trials, devs[w], res.data(),
                                   chunk_bases ? cb.data() : nullptr, trial_bases ? tb.data() : nullptr);
    status[w] = s;
    if (s != MCB_OK) {
      errors[w] = g_last_error;
      return;
    }
    for (size_t r = 0; r < mine.size(); ++r)
      std::memcpy(out + mine[r] * trials, res.data() + r * trials, sizeof(mcb_trial_stats) * trials);
  };
  if (devs.size() == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (size_t w = 0; w < devs.size(); ++w) pool.emplace_back(work, w);
    for (auto& th : pool) th.join();
  }
  for (size_t w = 0; w < devs.size(); ++w)
    if (status[w] != MCB_OK) return fail(status[w], "device " + std::to_string(devs[w]) + ": " + errors[w]);
  return MCB_OK;
}

// One tree round: batches sharded over `devs` by LPT on their sample cost.
mcb_status run_cells(const std::vector<mcb::tree::CellBatch>& batches, uint64_t seed,
                     const std::vector<int>& devs) {
  const size_t n = batches.size();
  std::vector<std::vector<const mcb::tree::CellBatch*>> shard(devs.size());
  if (devs.size() == 1) {
    for (const auto& b : batches) shard[0].push_back(&b);
  } else {
    std::vector<size_t> order(n);
    std::iota(order.begin(), order.end(), size_t(0));
    std::vector<double> cost(n);
    for (size_t i = 0; i < n; ++i)
      cost[i] = double(batches[i].n_cells) * double(batches[i].spc) * sample_cost(*batches[i].fn);
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return cost[a] > cost[b]; });
    std::vector<double> load(devs.size(), 0.0);
    for (size_t i : order) {
      size_t best = 0;
      for (size_t w = 1; w < load.size(); ++w)
        if (load[w] < load[best]) best = w;
      shard[best].push_back(&batches[i]);
      load[best] += cost[i];
    }
  }
  std::vector<mcb_status> status(devs.size(), MCB_OK);
  std::vector<std::string> errors(devs.size());
  auto work = [&](size_t w) {
    if (shard[w].empty()) return;
    status[w] = run_cell_shard(shard[w], seed, devs[w]);
    if (status[w] != MCB_OK) errors[w] = g_last_error;
  };
  if (devs.size() == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (size_t w = 0; w < devs.size(); ++w) pool.emplace_back(work, w);
    for (auto& th : pool) th.join();
  }
  for (size_t w = 0; w < devs.size(); ++w)
    if (status[w] != MCB_OK) return fail(status[w], "device " + std::to_string(devs[w]) + ": " + errors[w]);
  return MCB_OK;
}

// Every tree of `tasks`, on `devs`: device-resident rounds (default; trees
// sharded over the devices by budget, each device independent), or the host
// driver over batched cell launches (MCB_TREE_DEVICE=0, kept as the
// cross-check of the device rounds: both give identical trees).
mcb_status run_trees_on(std::vector<mcb::tree::TreeTask>& tasks, uint64_t seed, const std::vector<int>& devs) {
  static const bool host_driven = [] {
    const char* e = std::getenv("MCB_TREE_DEVICE");
    return e && e[0] == '0';
  }();
  if (host_driven) {
    std::mutex err_mu;
    std::string err;
    const mcb_status st = mcb::tree::run_trees(tasks, [&](const std::vector<mcb::tree::CellBatch>& batches) {
      const mcb_status r = run_cells(batches, seed, devs);
      if (r != MCB_OK) {
        std::lock_guard<std::mutex> lk(err_mu);
        err = g_last_error;
      }
      return r;
    });
    return st == MCB_OK ? st : fail(st, err);
  }
  // leaf storage is reserved up front on the device: very large trees (a
  // budget / depth allowing > 64 Mi leaves in one call) take the host driver
  uint64_t bound = 0;
  for (auto& t : tasks) {
    const mcb::tree::Config cfg = mcb::tree::config_of(*t.fn);
    const uint32_t spc = std::max<uint32_t>(cfg.samples_per_cell, 2);
    uint32_t k;
    uint64_t n0;
    if (tree_first_pass(*t.fn, cfg, spc, k, n0)) bound += tree_leaf_bound(n0, spc, cfg);
  }
  if (bound > (uint64_t(1) << 26)) {
    std::mutex err_mu;
    std::string err;
    const mcb_status st = mcb::tree::run_trees(tasks, [&](const std::vector<mcb::tree::CellBatch>& batches) {
      const mcb_status r = run_cells(batches, seed, devs);
      if (r != MCB_OK) {
        std::lock_guard<std::mutex> lk(err_mu);
        err = g_last_error;
      }
      return r;
    });
    return st == MCB_OK ? st : fail(st, err);
  }
  std::vector<std::vector<mcb::tree::TreeTask*>> shard(devs.size());
  std::vector<double> load(devs.size(), 0.0);
  for (auto& t : tasks) {  // greedy by budget (the trees' work bound)
    size_t best = 0;
    for (size_t w = 1; w < devs.size(); ++w)
      if (load[w] < load[best]) best = w;
    shard[best].push_back(&t);
    load[best] += double(t.fn->n_samples) * sample_cost(*t.fn);
  }
  std::vector<mcb_status> status(devs.size(), MCB_OK);
  std::vector<std::string> errors(devs.size());
  auto work = [&](size_t w) {
    status[w] = run_trees_device(shard[w], seed, devs[w]);
    if (status[w] != MCB_OK) errors[w] = g_last_error;
  };
  if (devs.size() == 1) {
    work(0);
  } else {
    std::vector<std::thread> pool;
    for (size_t w = 0; w < devs.size(); ++w) pool.emplace_back(work, w);
    for (auto& th : pool) th.join();
  }
  for (size_t w = 0; w < devs.size(); ++w)
    if (status[w] != MCB_OK) return fail(status[w], "device " + std::to_string(devs[w]) + ": " + errors[w]);
  return MCB_OK;
}

}  // namespace

extern "C" {

uint32_t mcb_abi_version(void) { return MCB_ABI_VERSION; }

const char* mcb_last_error(void) { return g_last_error.c_str(); }

int mcb_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void mcb_stream_key(uint64_t global_seed, uint32_t integrand_index, uint32_t key_out[2]) {
  uint64_t h = splitmix64(global_seed);
  h = splitmix64(h ^ (0x9E3779B97F4A7C15ull * (uint64_t(integrand_index) + 1)));
  key_out[0] = uint32_t(h);
  key_out[1] = uint32_t(h >> 32);
}

double mcb_volume(const mcb_integrand* fn) { return fn ? volume(*fn) : 0.0; }

size_t mcb_to_dsl(const mcb_integrand* fn, char* buf, size_t cap) {
  if (!fn) return 0;
  const std::string s = to_dsl(*fn);
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return s.size() + 1;
}

mcb_status mcb_validate(const mcb_integrand* fns, size_t n_fns, const char* const* names,
                        uint32_t trials, mcb_violation* out, size_t cap, size_t* n_out) {
  std::vector<std::pair<int64_t, std::string>> v;
  if (trials < 1) v.push_back({-1, "trials must be >= 1"});
  if (n_fns == 0) v.push_back({-1, "integrand list is empty"});
  if (n_fns && !fns) return fail(MCB_ERR_INVALID_ARGUMENT, "fns is NULL");
  std::map<std::string, int> name_count;
  if (names)
    for (size_t i = 0; i < n_fns; ++i) ++name_count[names[i] ? names[i] : ""];
  for (size_t i = 0; i < n_fns; ++i) {
    std::vector<std::string> msgs;
    if (names && (!names[i] || !names[i][0])) msgs.push_back("integrand name is empty");
    violations_of(fns[i], trials, msgs);
    for (auto& m : msgs) v.push_back({int64_t(i), m});
  }
  if (names)  // duplicate names, once per offending name (src/batch.cpp:113-118)
    for (const auto& [name, count] : name_count)
      if (count > 1) {
        int64_t first = -1;
        for (size_t i = 0; i < n_fns; ++i)
          if (names[i] && name == names[i]) { first = int64_t(i); break; }
        v.push_back({first, "duplicate integrand name (" + std::to_string(count) + " occurrences)"});
      }
  if (n_out) *n_out = v.size();
  for (size_t i = 0; i < v.size() && i < cap && out; ++i) {
    out[i].integrand = v[i].first;
    std::snprintf(out[i].message, sizeof out[i].message, "%s", v[i].second.c_str());
  }
  return MCB_OK;
}

mcb_status mcb_stratified_plan(const mcb_integrand* fn, uint32_t* cells_per_dim, uint64_t* n_cells,
                               uint32_t* samples_per_cell) {
  if (!fn) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL integrand");
  if (fn->dim < 1 || fn->dim > MCB_MAX_DIM) return fail(MCB_ERR_INVALID_ARGUMENT, "bad dim");
  const StratPlan p = stratified_plan(*fn);
  if (!p.ok) return fail(MCB_ERR_VALIDATION, "cell grid exceeds configured cap");
  if (cells_per_dim) *cells_per_dim = p.k;
  if (n_cells) *n_cells = p.n_cells;
  if (samples_per_cell) *samples_per_cell = p.spc;
  return MCB_OK;
}

mcb_status mcb_partition(const mcb_integrand* fns, size_t n_fns, uint32_t trials, int n_shards,
                         uint32_t* shard_of_fn) {
  if (n_shards < 1) return fail(MCB_ERR_INVALID_ARGUMENT, "n_shards must be >= 1");
  if (n_fns && (!fns || !shard_of_fn)) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL buffer");
  lpt(fns, n_fns, trials, n_shards, shard_of_fn);
  return MCB_OK;
}

mcb_status mcb_summarize_trials(const mcb_trial_stats* per_trial, uint32_t n_trials, double* mean,
                                double* trial_stddev, uint32_t* n_ok) {
  if (!per_trial || !mean || !trial_stddev) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL buffer");
  double sum = 0.0;
  uint32_t r = 0;
  for (uint32_t t = 0; t < n_trials; ++t)
    if (per_trial[t].status == MCB_TRIAL_OK) {
      sum += per_trial[t].value;
      ++r;
    }
  if (n_ok) *n_ok = r;
  if (r == 0) return fail(MCB_ERR_INVALID_ARGUMENT, "no successful trials");  // InsufficientTrials
  *mean = sum / double(r);
  *trial_stddev = 0.0;
  if (r >= 2) {
    double ss = 0.0;
    for (uint32_t t = 0; t < n_trials; ++t)
      if (per_trial[t].status == MCB_TRIAL_OK) {
        const double d = per_trial[t].value - *mean;
        ss += d * d;
      }
    *trial_stddev = std::sqrt(ss / double(r - 1));
  }
  return MCB_OK;
}

mcb_status mcb_plan_create(const mcb_integrand* fns, size_t n_fns, uint64_t seed, uint32_t trials,
                           int device, mcb_plan** plan_out) {
  if (!plan_out) return fail(MCB_ERR_INVALID_ARGUMENT, "plan_out is NULL");
  *plan_out = nullptr;
  return plan_create_impl(fns, n_fns, seed, trials, device, 0, 0, plan_out);
}

mcb_status mcb_plan_launch(mcb_plan* plan, void* stream) {
  if (!plan) return fail(MCB_ERR_INVALID_ARGUMENT, "plan is NULL");
  return plan_launch_impl(plan, static_cast<cudaStream_t>(stream));
}

mcb_status mcb_plan_download(mcb_plan* plan, mcb_trial_stats* out, void* stream) {
  if (!plan || !out) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  return plan_download_impl(plan, out, static_cast<cudaStream_t>(stream));
}

mcb_status mcb_plan_get_info(const mcb_plan* plan, mcb_plan_info* info) {
  if (!plan || !info) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  std::memset(info, 0, sizeof *info);
  info->n_fns = plan->n_fns;
  info->trials = plan->trials;
  info->n_groups = uint32_t(plan->hp.groups.size());
  info->n_tiles = plan->hp.n_tiles;
  info->total_samples = plan->hp.total_samples;
  info->philox_blocks = plan->hp.philox_blocks;
  uint32_t launches = 1;  // k_combine
  for (const auto& g : plan->hp.groups) {
    const uint64_t ctas = g.n_tiles / ((g.variant & mcb::detail::kWarpTile)
                                           ? (g.family == MCB_FAMILY_PROGRAM ? uint64_t(mcb::detail::kProgThreads / 32)
                                                                             : uint64_t(mcb::detail::kTileAlign))
                                           : 1u);
    launches += uint32_t((ctas + 0x7FFFFFF7ull) / 0x7FFFFFF8ull);
  }
  info->launches_per_run = launches;
  return MCB_OK;
}

void mcb_plan_destroy(mcb_plan* plan) {
  if (!plan) return;
  {
    DeviceGuard guard(plan->device);
    plan->buf.release();
  }
  delete plan;
}

mcb_status mcb_run_direct(const mcb_integrand* fns, size_t n_fns, uint64_t seed, uint32_t trials,
                          const int* devices, int n_devices, mcb_trial_stats* out,
                          double* seconds) {
  mcb_status st = validate_for_run(fns, n_fns, trials);
  if (st != MCB_OK) return st;
  if (!out) return fail(MCB_ERR_INVALID_ARGUMENT, "out is NULL");
  std::vector<int> devs;
  if (!devices || n_devices <= 0) devs.push_back(0);
  else devs.assign(devices, devices + n_devices);
  for (int d : devs)
    if ((st = check_device(d)) != MCB_OK) return st;

  const auto t0 = std::chrono::steady_clock::now();
  std::vector<size_t> plain, trees;
  for (size_t i = 0; i < n_fns; ++i) (fns[i].method == MCB_METHOD_TREE ? trees : plain).push_back(i);
  if (!plain.empty()) {  // direct + stratified: one sharded launch set
    std::vector<mcb_integrand> sub(plain.size());
    for (size_t r = 0; r < plain.size(); ++r) sub[r] = fns[plain[r]];
    std::vector<mcb_trial_stats> res(sub.size() * trials);
    if ((st = run_sharded(sub.data(), sub.size(), seed, trials, devs, res.data(), nullptr, nullptr)) != MCB_OK)
      return st;
    for (size_t r = 0; r < plain.size(); ++r)
      std::memcpy(out + plain[r] * trials, res.data() + r * trials, sizeof(mcb_trial_stats) * trials);
  }
  if (!trees.empty()) {  // tree: lock-step rounds over every (integrand, trial) tree
    std::vector<mcb::tree::TreeTask> tasks;
    tasks.reserve(trees.size() * trials);
    for (size_t i : trees)
      for (uint32_t t = 0; t < trials; ++t)
        tasks.push_back(mcb::tree::TreeTask{&fns[i], t, 0, out + i * trials + t, nullptr});
    if ((st = run_trees_on(tasks, seed, devs)) != MCB_OK) return st;
  }
  const auto t1 = std::chrono::steady_clock::now();
  if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
  return MCB_OK;
}

mcb_status mcb_tree_refine(const mcb_integrand* fn, uint64_t seed, uint32_t trial, uint64_t chunk_base,
                           int device, mcb_trial_stats* out, mcb_leaf* leaves, size_t leaf_cap,
                           size_t* n_leaves) {
  if (!fn || !out) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  // tree_refine itself has no validation step: a grid past the cap is a
  // CellBudgetExceeded result (MCB_TRIAL_CELL_BUDGET), not a job error.
  mcb_integrand f = *fn;
  f.method = MCB_METHOD_DIRECT;
  mcb_status st = validate_for_run(&f, 1, 1);
  if (st != MCB_OK) return st;
  f.method = MCB_METHOD_TREE;
  if ((st = check_device(device)) != MCB_OK) return st;
  std::vector<mcb_leaf> lv;
  std::vector<mcb::tree::TreeTask> tasks{mcb::tree::TreeTask{&f, trial, chunk_base, out, &lv}};
  const std::vector<int> devs{device};
  st = run_trees_on(tasks, seed, devs);
  if (st != MCB_OK) return st;
  if (n_leaves) *n_leaves = lv.size();
  if (leaves)
    std::memcpy(leaves, lv.data(), sizeof(mcb_leaf) * std::min(leaf_cap, lv.size()));
  return MCB_OK;
}

mcb_status mcb_stratified_mc(const mcb_integrand* fn, uint32_t cells_per_dim, uint32_t samples_per_cell,
                             uint64_t cell_cap, uint64_t seed, uint32_t trial, uint64_t chunk_base, int device,
                             mcb_trial_stats* out, mcb_leaf* leaves, size_t leaf_cap, size_t* n_leaves) {
  if (!fn || !out) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  if (cells_per_dim == 0) return fail(MCB_ERR_INVALID_ARGUMENT, "cells_per_dim must be >= 1");
  if (samples_per_cell < 2) return fail(MCB_ERR_INVALID_ARGUMENT, "n_samples must be >= 2");
  mcb_integrand f = *fn;
  f.method = MCB_METHOD_DIRECT;
  mcb_status st = validate_for_run(&f, 1, 1);
  if (st != MCB_OK) return st;
  if ((st = check_device(device)) != MCB_OK) return st;
  // = the first pass of tree_refine with the grid given and no refinement
  f.method = MCB_METHOD_TREE;
  f.flags |= MCB_FLAG_REFINE_CONFIG;
  f.cells_per_dim = cells_per_dim;
  f.samples_per_cell = samples_per_cell;
  f.max_depth = 0;
  f.cell_cap = cell_cap;
  std::vector<mcb_leaf> lv;
  std::vector<mcb::tree::TreeTask> tasks{mcb::tree::TreeTask{&f, trial, chunk_base, out, &lv}};
  const std::vector<int> devs{device};
  st = run_trees_on(tasks, seed, devs);
  if (st != MCB_OK) return st;
  if (out->status == MCB_TRIAL_ALL_NONFINITE) {  // every cell dead: the first one throws
    out->status = MCB_TRIAL_DEAD_CELL;
    out->detail = 0;
  } else if (out->status == MCB_TRIAL_OK) {
    for (size_t i = 0; i < lv.size(); ++i)
      if (lv[i].estimate.status != MCB_TRIAL_OK) {  // direct_mc of cell i threw
        out->status = MCB_TRIAL_DEAD_CELL;
        out->detail = uint32_t(i);
        out->value = out->std_error = 0.0;
        lv.clear();
        break;
      }
  }
  if (n_leaves) *n_leaves = lv.size();
  if (leaves) std::memcpy(leaves, lv.data(), sizeof(mcb_leaf) * std::min(leaf_cap, lv.size()));
  return MCB_OK;
}

mcb_status mcb_direct_mc(const mcb_integrand* fn, uint64_t seed, uint32_t trial, uint64_t chunk_base,
                         int device, mcb_trial_stats* out) {
  if (!fn || !out) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  if (fn->n_samples < 2) return fail(MCB_ERR_INVALID_ARGUMENT, "n_samples must be >= 2");
  if (chunk_base + chunk_count(fn->n_samples) - 1 > 0xFFFFFFFFull)
    return fail(MCB_ERR_OUT_OF_RANGE, "chunk_index exceeds 32 bits");
  // One (integrand, trial) unit: a 1-trial plan whose key base is
  // {seed, integrand_index, trial, chunk_base}.
  mcb_integrand f = *fn;  // direct_mc ignores the spec's method
  f.method = MCB_METHOD_DIRECT;
  mcb_plan* plan = nullptr;
  mcb_status st = plan_create_impl(&f, 1, seed, 1, device, uint32_t(chunk_base), trial, &plan);
  if (st != MCB_OK) return st;
  st = plan_launch_impl(plan, nullptr);
  if (st == MCB_OK) st = plan_download_impl(plan, out, nullptr);
  mcb_plan_destroy(plan);
  return st;
}

mcb_status mcb_debug_points(uint64_t seed, uint32_t integrand_index, uint32_t trial, uint64_t chunk,
                            uint64_t first_point, uint64_t count, uint32_t dim, const double* low,
                            const double* high, int device, double* out) {
  if (dim < 1 || dim > MCB_MAX_DIM || !low || !high || (count && !out))
    return fail(MCB_ERR_INVALID_ARGUMENT, "bad arguments");
  if (chunk > 0xFFFFFFFFull) return fail(MCB_ERR_OUT_OF_RANGE, "chunk_index exceeds 32 bits");
  if ((first_point + count) * dim / 2 > 0xFFFFFFFFull)
    return fail(MCB_ERR_OUT_OF_RANGE, "block index exceeds 32 bits");
  mcb_status st = check_device(device);
  if (st != MCB_OK) return st;
  if (count == 0) return MCB_OK;
  DeviceGuard guard(device);
  uint32_t key[2];
  mcb_stream_key(seed, integrand_index, key);
  double hw[2 * MCB_MAX_DIM];
  for (uint32_t j = 0; j < dim; ++j) {
    hw[j] = low[j];
    hw[MCB_MAX_DIM + j] = high[j] - low[j];
  }
  double* d_lw = nullptr;
  double* d_out = nullptr;
  MCB_CUDA(cudaMalloc(&d_lw, sizeof hw));
  cudaError_t e = cudaMalloc(&d_out, sizeof(double) * count * dim);
  if (e == cudaSuccess) e = cudaMemcpy(d_lw, hw, sizeof hw, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = mcb::detail::launch_debug_points(key[0], key[1], trial, uint32_t(chunk), first_point, count,
                                         dim, d_lw, d_lw + MCB_MAX_DIM, d_out, nullptr);
  if (e == cudaSuccess)
    e = cudaMemcpy(out, d_out, sizeof(double) * count * dim, cudaMemcpyDeviceToHost);
  cudaFree(d_lw);
  if (d_out) cudaFree(d_out);
  if (e != cudaSuccess) return cuda_fail(e, "debug_points");
  return MCB_OK;
}

mcb_status mcb_debug_eval(const mcb_integrand* fn, uint64_t seed, uint32_t trial, uint64_t chunk,
                          uint64_t first_point, uint64_t count, int device, double* out) {
  if (!fn || (count && !out)) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  std::vector<std::string> msgs;
  violations_of(*fn, 1, msgs);
  if (!msgs.empty()) return fail(MCB_ERR_VALIDATION, msgs.front());
  if (chunk > 0xFFFFFFFFull) return fail(MCB_ERR_OUT_OF_RANGE, "chunk_index exceeds 32 bits");
  if (first_point + count > MCB_CHUNK_SIZE)
    return fail(MCB_ERR_OUT_OF_RANGE, "points must lie inside one chunk");
  mcb_status st = check_device(device);
  if (st != MCB_OK) return st;
  if (count == 0) return MCB_OK;
  DeviceGuard guard(device);
  mcb_integrand direct = *fn;  // per-sample values on the integrand's own domain
  direct.method = MCB_METHOD_DIRECT;
  Prepared p = prepare(direct, seed, 0, 0);
  const uint64_t first_pair = first_point / 2;
  const uint64_t n_pairs = (first_point + count - 1) / 2 - first_pair + 1;
  const bool is_prog = fn->family == MCB_FAMILY_PROGRAM;
  FnDesc* d_fn = nullptr;
  double* d_out = nullptr;
  uint32_t* d_code = nullptr;
  double* d_consts = nullptr;
  if (is_prog) {
    p.d.prog_off = 0;
    p.d.prog_len = uint32_t(fn->program->p.code.size());
    p.d.const_off = 0;
    p.d.n_consts = uint32_t(fn->program->p.consts.size());
  }
  MCB_CUDA(cudaMalloc(&d_fn, sizeof(FnDesc)));
  cudaError_t e = cudaMalloc(&d_out, sizeof(double) * 2 * n_pairs);
  if (e == cudaSuccess) e = cudaMemcpy(d_fn, &p.d, sizeof(FnDesc), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && is_prog) {
    const auto& w = fn->program->words;
    const auto& c = fn->program->p.consts;
    e = cudaMalloc(&d_code, sizeof(uint32_t) * std::max<size_t>(w.size(), 1));
    if (e == cudaSuccess) e = cudaMalloc(&d_consts, sizeof(double) * std::max<size_t>(c.size(), 1));
    if (e == cudaSuccess) e = cudaMemcpy(d_code, w.data(), sizeof(uint32_t) * w.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !c.empty())
      e = cudaMemcpy(d_consts, c.data(), sizeof(double) * c.size(), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess) {
    if (is_prog)
      e = mcb::detail::launch_program_eval(int(fn->dim), p.variant, d_fn, d_code, d_consts,
                                           fn->program->p.depth, trial, uint32_t(chunk),
                                           uint32_t(first_pair), uint32_t(n_pairs), d_out, nullptr);
    else
      e = mcb::detail::launch_debug_eval_impl(int(fn->family), int(fn->dim), p.variant, d_fn, trial,
                                              uint32_t(chunk), uint32_t(first_pair),
                                              uint32_t(n_pairs), d_out, nullptr);
  }
  std::vector<double> tmp(2 * n_pairs);
  if (e == cudaSuccess)
    e = cudaMemcpy(tmp.data(), d_out, sizeof(double) * 2 * n_pairs, cudaMemcpyDeviceToHost);
  cudaFree(d_fn);
  if (d_out) cudaFree(d_out);
  if (d_code) cudaFree(d_code);
  if (d_consts) cudaFree(d_consts);
  if (e != cudaSuccess) return cuda_fail(e, "debug_eval");
  std::memcpy(out, tmp.data() + (first_point - 2 * first_pair), sizeof(double) * count);
  return MCB_OK;
}

int mcb_program_jit(int mode) {
  if (mode >= 0) mcb::jit::set_mode(mode);
  return mcb::jit::mode();
}

uint64_t mcb_program_jit_compiles(void) { return mcb::jit::compile_count(); }

mcb_status mcb_program_jit_build(const mcb_program* program) {
  if (!program) return fail(MCB_ERR_INVALID_ARGUMENT, "program is NULL");
  std::string err;
  if (!mcb::jit::compile_only(program->p, &err)) return fail(MCB_ERR_INVALID_ARGUMENT, "JIT build failed: " + err);
  return MCB_OK;
}

size_t mcb_program_jit_error(char* buf, size_t cap) {
  const std::string s = mcb::jit::last_error();
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return s.size() + 1;
}

mcb_status mcb_probe_philox_peak(int device, double ms, double* blocks_per_s) {
  if (!blocks_per_s) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  mcb_status st = check_device(device);
  if (st != MCB_OK) return st;
  DeviceGuard guard(device);
  int sms = 0;
  MCB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const int ctas = sms * 8;
  uint32_t* buf = nullptr;
  MCB_CUDA(cudaMalloc(&buf, sizeof(uint32_t) * (ctas + 2)));
  const uint32_t key[2] = {0x37BA30CAu, 0xCCC782D2u};  // (seed 20200814, integrand 0)
  cudaError_t e = cudaMemcpy(buf, key, sizeof key, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int iters = 256;
  float elapsed = 0.f;
  for (int round = 0; round < 14 && e == cudaSuccess; ++round) {  // grow until ~ms
    cudaEventRecord(a);
    e = mcb::detail::launch_philox_probe(buf, buf + 2, ctas, iters, nullptr);
    cudaEventRecord(b);
    if (e == cudaSuccess) e = cudaEventSynchronize(b);
    if (e != cudaSuccess) break;
    cudaEventElapsedTime(&elapsed, a, b);
    if (elapsed >= ms) break;
    iters *= 2;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  if (e != cudaSuccess) return cuda_fail(e, "philox_probe");
  *blocks_per_s = double(ctas) * 256.0 * 4.0 * double(iters) / (double(elapsed) * 1e-3);
  return MCB_OK;
}

mcb_status mcb_program_compile(const char* source, uint32_t dim, const char* const* param_names,
                               size_t n_params, mcb_program** out) {
  if (!source || !out || (n_params && !param_names))
    return fail(MCB_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  std::vector<std::string> names;
  for (size_t i = 0; i < n_params; ++i) {
    if (!param_names[i]) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL parameter name");
    names.emplace_back(param_names[i]);
  }
  std::sort(names.begin(), names.end());
  names.erase(std::unique(names.begin(), names.end()), names.end());
  try {
    auto* p = new mcb_program();
    try {
      p->p = mcb::prog::compile(source, dim, names);
    } catch (...) {
      delete p;
      throw;
    }
    p->words = p->p.words();
    *out = p;
    return MCB_OK;
  } catch (const mcb::prog::ParseError& e) {
    return fail(MCB_ERR_VALIDATION, std::string("expression does not parse: ") + e.what());
  } catch (const mcb::prog::CompileError& e) {
    return fail(MCB_ERR_VALIDATION, e.what());
  } catch (const std::exception& e) {
    return fail(MCB_ERR_INVALID_ARGUMENT, e.what());
  }
}

void mcb_program_destroy(mcb_program* program) { delete program; }

mcb_status mcb_program_info(const mcb_program* program, uint32_t* n_instr, uint32_t* depth,
                            uint32_t* n_params) {
  if (!program) return fail(MCB_ERR_INVALID_ARGUMENT, "NULL program");
  if (n_instr) *n_instr = uint32_t(program->p.code.size());
  if (depth) *depth = program->p.depth;
  if (n_params) *n_params = uint32_t(program->p.param_names.size());
  return MCB_OK;
}

size_t mcb_program_param_name(const mcb_program* program, uint32_t i, char* buf, size_t cap) {
  if (!program || i >= program->p.param_names.size()) return 0;
  const std::string& s = program->p.param_names[i];
  if (buf && cap) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return s.size() + 1;
}

}  // extern "C"
