// capi_plan.cpp — the C-ABI layer's descriptor lowering and validation
// (reference helpers, variant selection under the FAST preconditions, host
// plans, device buffers, per-device contexts, one device shard of a run).
//
// Reference correspondence (file:line under /root/reference/proj):
//   validate (violations_of)        src/batch.cpp:62-120
//   stratified_plan                 src/batch.cpp:41-54
//   cell_grid_size / auto_cells     src/estimator.cpp:94-122
//   HyperRect::valid / volume       src/sampling.cpp:7-20
//   UniformStream key (splitmix64)  src/sampling.cpp:44-49, 84-87
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <numeric>
#include <thread>
#include <tuple>

#include "capi_internal.hpp"
#include "jit.hpp"

namespace mcb::capi {

thread_local std::string g_last_error;

mcb_status fail(mcb_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

mcb_status cuda_fail(cudaError_t e, const char* what) {
  return fail(MCB_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}


uint64_t splitmix64(uint64_t z) {  // src/sampling.cpp:44-49
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

uint64_t chunk_count(uint64_t n) { return (n + MCB_CHUNK_SIZE - 1) / MCB_CHUNK_SIZE; }


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

// k^d, saturating at UINT64_MAX.
static uint64_t sat_pow(uint64_t k, uint32_t d) {
  uint64_t r = 1;
  for (uint32_t i = 0; i < d; ++i) {
    if (k && r > UINT64_MAX / k) return UINT64_MAX;
    r *= k;
  }
  return r;
}

// The largest k >= 1 with k^d <= x (1 when there is none): a floating-point
// guess corrected with exact integer powers.
uint32_t int_root_floor(uint64_t x, uint32_t d) {
  if (d == 0 || x <= 1) return 1;
  uint64_t k = uint64_t(std::pow(double(x), 1.0 / d));
  k = std::min<uint64_t>(std::max<uint64_t>(k, 1), 0xFFFFFFFFull);
  while (k > 1 && sat_pow(k, d) > x) --k;
  while (k < 0xFFFFFFFFull && sat_pow(k + 1, d) <= x) ++k;
  return uint32_t(k);
}

// auto_cells_per_dim (src/estimator.cpp:107-122): the largest k with
// k^d <= limit (at least 1) — the reference's k = 1, 2, ... search, closed form.
uint32_t auto_cells_per_dim(uint32_t d, uint64_t limit) { return int_root_floor(limit, d); }

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


// Decide the kernel variant and fill the device descriptor.  FAST variants
// need (host-proven, for every point of the domain): finite parameters,
// |t| < 2^20 for the table reduction, no overflow of f, and exact 2^-64
// folding.  Anything else runs the SAFE variant (libdevice sincos, counted
// non-finite samples) — still on the GPU.
// tree_cells: the descriptor of one tree's cells in a refinement round (the
// caller sets n_cells / spc / cpc / cell_rects / cell_est); cells are at
// least width / (k0 * 2^depth) wide, which bounds the 2^-64 fold.
Prepared prepare(const mcb_integrand& f, uint64_t seed, uint32_t chunk_base,
                 uint32_t trial_base, bool tree_cells) {
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
    if (stratified(f) && d.spc <= kWarpTileMaxSpc) {  // small cells: lane per cell on large grids
      if (d.n_cells >= kProgLaneMinCells) {
        p.variant |= kLaneCell;
        d.n_chunks = round_up(d.n_cells * d.cpc, uint32_t(kProgThreads));
      } else {
        p.variant |= kWarpTile;
      }
    }
    if (!strat) {  // cells use a per-tile shift computed on the device
      double mid[MCB_MAX_DIM];
      for (uint32_t j = 0; j < f.dim; ++j) mid[j] = f.low[j] + 0.5 * (f.high[j] - f.low[j]);
      const double c = host_eval(f, mid);
      d.shift = std::isfinite(c) && std::fabs(c) < 1e300 ? c : 0.0;
    }
    return p;
  }
  const bool harm = f.family == MCB_FAMILY_HARMONIC || f.family == MCB_FAMILY_HARMONIC_VEC;

  // MCB_FAMILY_SAFE=1 (measurement knob): every family
  // integrand runs the SAFE variant — libdevice sincos instead of the table
  // form, plain parameters, per-sample non-finite counting — the ablation
  // point "accurate sincos" of DESIGN.md §3.
  static const bool force_safe = [] {
    const char* e = std::getenv("MCB_FAMILY_SAFE");
    return e && *e == '1';
  }();
  bool fast = finite && std::isfinite(xmax) && !force_safe;
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
    // direct harmonic: the shift rides in the CTA's table (kFoldShift), so
    // g = f - c costs nothing extra; cells use a per-tile shift instead
    if (harm && !strat) p.variant |= kFoldShift;
  } else {
    p.variant = kSafe;
  }
  if (!harm) p.variant &= ~kUnitCoef;
  if (strat) p.variant |= kStrat;
  if (stratified(f) && d.spc <= kWarpTileMaxSpc) {
    // small cells: a lane per cell on large grids (unit-coefficient or no
    // table), else a warp per cell
    const bool general_table = harm && !(p.variant & kSafe) && !(p.variant & kUnitCoef);
    if (d.n_cells >= kLaneCellMinCells && !general_table) {
      p.variant |= kLaneCell;
      d.n_chunks = round_up(d.n_cells * d.cpc, kLaneAlign);
    } else {
      p.variant |= kWarpTile;
    }
  }
  // shift constant: f at the domain midpoint (reference op order, libm);
  // cells use a per-tile shift computed on the device instead
  if (!strat) {
    double mid[MCB_MAX_DIM];
    for (uint32_t j = 0; j < f.dim; ++j) mid[j] = f.low[j] + 0.5 * (f.high[j] - f.low[j]);
    const double c = host_eval(f, mid);
    d.shift = std::isfinite(c) && std::fabs(c) < 1e300 ? c : 0.0;
  }
  return p;
}

}  // namespace mcb::capi

// ---- plans -------------------------------------------------------------------

namespace mcb::capi {


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


// chunk_bases / trial_bases (may be NULL): per-integrand key bases overriding
// chunk_base / trial_base (the tree driver's cell batches).
mcb_status build_host_plan(const mcb_integrand* fns, size_t n_fns, uint64_t seed, uint32_t trials,
                           uint32_t chunk_base, uint32_t trial_base, HostPlan& hp,
                           const uint32_t* chunk_bases, const uint32_t* trial_bases) {
  hp.descs.clear();
  hp.groups.clear();
  hp.code.clear();
  hp.consts.clear();
  hp.bounds.clear();
  hp.bounds_off.clear();
  hp.n_tiles = hp.total_samples = hp.philox_blocks = 0;
  // per-thread scratch: a call reuses the previous call's pages (fresh
  // vectors of this size are mmap'ed and page-faulted in on every call)
  thread_local std::vector<Prepared> prep;
  prep.resize(n_fns);
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
    tile = round_up<uint64_t>(tile, mcb::detail::tile_align(var, fam == MCB_FAMILY_PROGRAM));
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
        hp.groups.back().variant != var || hp.groups.back().prog != gp) {
      hp.groups.push_back(GroupLaunch{fam, dim, var, tile, 0, 0, gp});
      hp.groups.back().tile_samples = 0;
    }
    const uint64_t per_tile = d.strat_k > 0 ? d.spc : fns[i].n_samples;
    hp.groups.back().tile_samples =
        std::max(hp.groups.back().tile_samples, uint32_t(std::min<uint64_t>(per_tile, MCB_CHUNK_SIZE)));
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


// Enqueue: descriptor upload (from `staged`, pinned or not) + tile table +
// fused kernels + ordered combine, all on `s`.
// Runtime-specialised kernels of the plan's programs (jit.hpp): cache
// look-ups, and with `compile` (plans, which are relaunched) parallel
// compiles of the missing ones before the first launch.
void prepare_programs(const HostPlan& hp, bool compile) {
  std::vector<std::pair<const mcb::prog::Program*, int>> kernels;
  for (const auto& g : hp.groups) {
    if (!g.prog) continue;
    const int km = mcb::detail::program_kernel_mode(g.variant);
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


DeviceCtx& device_ctx(int device) {
  static std::mutex mu;
  static std::map<int, DeviceCtx*> ctxs;  // never freed: lives for the process
  std::lock_guard<std::mutex> lock(mu);
  DeviceCtx*& c = ctxs[device];
  if (!c) c = new DeviceCtx();
  return *c;
}


// One shard of mcb_run_direct on one device (synchronous).
// Tiles one trial of an integrand occupies (an upper bound for padded cell
// grids).
uint64_t tiles_per_trial(const mcb_integrand& f) {
  if (!stratified(f)) return chunk_count(f.n_samples);
  const StratPlan p = stratified_plan(f);
  return p.n_cells * chunk_count(p.spc) + mcb::detail::kLaneAlign;
}

// tile_out (may be NULL): also returns the first tile_cap raw tile partials
// (the chunk accumulators of mcb_accumulate_chunk).  A job whose tiles exceed
// one wave (MCB_WAVE_TILES, default 2^29 tiles = 19 GB of partials and tile
// table) runs as consecutive waves of whole integrands on the device, each a
// shard of its own: results are those of one launch set (every (integrand,
// trial) depends only on its own tiles), memory stays bounded.
mcb_status run_shard(const mcb_integrand* fns, size_t n_fns, uint64_t seed, uint32_t trials,
                     int device, mcb_trial_stats* out, const uint32_t* chunk_bases,
                     const uint32_t* trial_bases, TilePartial* tile_out, size_t tile_cap) {
  static const uint64_t wave = [] {
    const char* e = std::getenv("MCB_WAVE_TILES");
    const unsigned long long v = e && *e ? std::strtoull(e, nullptr, 10) : 0ull;
    return v ? uint64_t(v) : (uint64_t(1) << 29);
  }();
  if (n_fns > 1 && !tile_out) {
    uint64_t total = 0;
    for (size_t i = 0; i < n_fns && total <= wave; ++i) total += tiles_per_trial(fns[i]) * trials;
    if (total > wave) {
      for (size_t i0 = 0; i0 < n_fns;) {
        size_t i1 = i0 + 1;
        uint64_t acc = tiles_per_trial(fns[i0]) * trials;
        while (i1 < n_fns && acc + tiles_per_trial(fns[i1]) * trials <= wave) acc += tiles_per_trial(fns[i1++]) * trials;
        const mcb_status st = run_shard(fns + i0, i1 - i0, seed, trials, device, out + i0 * trials,
                                        chunk_bases ? chunk_bases + i0 : nullptr,
                                        trial_bases ? trial_bases + i0 : nullptr);
        if (st != MCB_OK) return st;
        i0 = i1;
      }
      return MCB_OK;
    }
  }
  thread_local HostPlan hp;  // reused capacity (see build_host_plan)
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
  const auto tq0 = std::chrono::steady_clock::now();
  std::memcpy(c.h_descs, hp.descs.data(), sizeof(FnDesc) * n_fns);
  for (size_t r = 0; r < n_fns; ++r)
    if (hp.bounds_off[r] >= 0) c.h_descs[r].grid_bounds = c.buf.bounds + hp.bounds_off[r];
  if ((st = enqueue_run(hp, c.buf, trials, c.h_descs, true, c.stream)) != MCB_OK) return st;
  if ((e = cudaMemcpyAsync(c.h_out, c.buf.out, sizeof(mcb_trial_stats) * n_out, cudaMemcpyDeviceToHost,
                           c.stream)) != cudaSuccess)
    return cuda_fail(e, "cudaMemcpyAsync(results)");
  if (tile_out && tile_cap &&
      (e = cudaMemcpyAsync(tile_out, c.buf.part, sizeof(TilePartial) * std::min<size_t>(tile_cap, hp.n_tiles),
                           cudaMemcpyDeviceToHost, c.stream)) != cudaSuccess)
    return cuda_fail(e, "cudaMemcpyAsync(tile partials)");
  const auto tq1 = std::chrono::steady_clock::now();
  if ((e = cudaStreamSynchronize(c.stream)) != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize");
  const auto tq2 = std::chrono::steady_clock::now();
  std::memcpy(out, c.h_out, sizeof(mcb_trial_stats) * n_out);
  const auto tq3 = std::chrono::steady_clock::now();
  if (trace)
    std::fprintf(stderr, "[mcb shard] enqueue %.3f ms, sync %.3f ms, copy-out %.3f ms\n",
                 std::chrono::duration<double, std::milli>(tq1 - tq0).count(),
                 std::chrono::duration<double, std::milli>(tq2 - tq1).count(),
                 std::chrono::duration<double, std::milli>(tq3 - tq2).count());
  return MCB_OK;
}


}  // namespace mcb::capi
