// mcbatch.cpp — C++ host API (include/mcb/mcbatch.hpp) over the C-ABI.
// Each function names the reference function whose contract it keeps
// (file:line under /root/reference/proj).
#include "mcb/mcbatch.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <complex>
#include <cstdio>
#include <numbers>
#include <sstream>

namespace mcb {

namespace {

void check(mcb_status st) {
  if (st == MCB_OK) return;
  if (st == MCB_ERR_INVALID_ARGUMENT) throw std::invalid_argument(mcb_last_error());
  if (st == MCB_ERR_OUT_OF_RANGE) throw std::out_of_range(mcb_last_error());
  throw DeviceError(mcb_last_error());
}

std::string strip(const std::string& s) {
  std::string o;
  for (char c : s)
    if (!std::isspace(static_cast<unsigned char>(c))) o += c;
  return o;
}

// Parameter names each family binds (mcb_to_dsl sources).
std::vector<std::string> required_params(const IntegrandSpec& s) {
  switch (s.family) {
    case Family::Harmonic:
      return s.unit_coeffs ? std::vector<std::string>{"k"} : std::vector<std::string>{"a", "b", "k"};
    case Family::HarmonicVec: {
      std::vector<std::string> p{"a", "b"};
      for (std::size_t j = 0; j < s.dim; ++j) p.push_back("k" + std::to_string(j + 1));
      return p;
    }
    case Family::Abs2:
    case Family::Abs3:
      return {};  // "a" defaults to 1 ("abs(x1+x2)" has no parameter)
    case Family::Program:
      return {};  // bound at compile time (compile_program)
  }
  return {};
}

// Programs of one job, compiled once per distinct (source, dim, params).
struct ProgramCache {
  std::map<std::string, CompiledSource> by_key;
  const mcb_program* get(const IntegrandSpec& s) {
    std::string key = s.program_source + '\x1f' + std::to_string(s.dim);
    for (const auto& [n, v] : s.params) key += '\x1f' + n;
    auto it = by_key.find(key);
    if (it == by_key.end())
      it = by_key.emplace(key, compile_program(s.program_source, s.dim, s.params)).first;
    return it->second.handle;
  }
};

double param_or(const IntegrandSpec& s, const char* name, double dflt) {
  auto it = s.params.find(name);
  return it == s.params.end() ? dflt : it->second;
}

}  // namespace

// ---- sampling (src/sampling.cpp) ---------------------------------------------

bool HyperRect::valid() const {  // src/sampling.cpp:7-14
  if (low.size() != high.size() || low.empty()) return false;
  for (std::size_t i = 0; i < low.size(); ++i) {
    if (!(low[i] < high[i])) return false;
    if (!std::isfinite(low[i]) || !std::isfinite(high[i])) return false;
  }
  return true;
}

double HyperRect::volume() const {  // src/sampling.cpp:16-20
  double v = 1.0;
  for (std::size_t i = 0; i < low.size(); ++i) v *= high[i] - low[i];
  return v;
}

HyperRect HyperRect::unit(std::size_t d) {
  HyperRect r;
  r.low.assign(d, 0.0);
  r.high.assign(d, 1.0);
  return r;
}

HyperRect HyperRect::box(std::vector<double> lo, std::vector<double> hi) {
  HyperRect r;
  r.low = std::move(lo);
  r.high = std::move(hi);
  if (!r.valid()) throw InvalidDomain("invalid hyperrectangle bounds");
  return r;
}

std::vector<double> sample_uniform(const HyperRect& rect, const StreamKey& key, std::size_t count,
                                   int device) {
  if (!rect.valid() || rect.dim() > MCB_MAX_DIM) throw InvalidDomain("invalid hyperrectangle");
  std::vector<double> out(count * rect.dim());
  check(mcb_debug_points(key.global_seed, key.integrand_index, key.trial_index, key.chunk_index, 0,
                         count, uint32_t(rect.dim()), rect.low.data(), rect.high.data(), device,
                         out.data()));
  return out;
}

// ---- integrand specs --------------------------------------------------------

const char* method_name(Method m) {
  return m == Method::Stratified ? "stratified" : (m == Method::Tree ? "tree" : "direct");
}

std::vector<int> devices_for_workers(std::uint32_t workers) {
  int n = mcb_device_count();
  if (workers > 0 && int(workers) < n) n = int(workers);
  std::vector<int> d;
  for (int i = 0; i < std::max(n, 1); ++i) d.push_back(i);
  return d;
}

CompiledSource compile_program(const std::string& source, std::size_t dim,
                               const std::map<std::string, double>& params) {
  std::vector<const char*> names;
  for (const auto& [n, v] : params) names.push_back(n.c_str());
  CompiledSource c;
  const mcb_status st =
      mcb_program_compile(source.c_str(), uint32_t(dim), names.data(), names.size(), &c.handle);
  if (st != MCB_OK) throw std::invalid_argument(mcb_last_error());
  return c;
}

mcb_integrand to_descriptor(const IntegrandSpec& s, std::uint32_t integrand_index,
                            const mcb_program* program) {
  mcb_integrand d{};
  d.family = uint32_t(s.family);
  d.dim = uint32_t(s.dim);
  d.integrand_index = integrand_index;
  d.n_samples = s.n_samples;
  d.flags = (s.family == Family::Harmonic && s.unit_coeffs) ? MCB_FLAG_UNIT_COEFFS : 0u;
  switch (s.family) {
    case Family::Harmonic:
      d.a = s.unit_coeffs ? 1.0 : param_or(s, "a", NAN);
      d.b = s.unit_coeffs ? 1.0 : param_or(s, "b", NAN);
      d.k[0] = param_or(s, "k", NAN);
      break;
    case Family::HarmonicVec:
      d.a = param_or(s, "a", NAN);
      d.b = param_or(s, "b", NAN);
      for (std::size_t j = 0; j < s.dim && j < MCB_MAX_DIM; ++j)
        d.k[j] = param_or(s, ("k" + std::to_string(j + 1)).c_str(), NAN);
      break;
    case Family::Abs2:
    case Family::Abs3:
      d.a = param_or(s, "a", 1.0);
      break;
    case Family::Program: {
      std::size_t j = 0;
      for (const auto& [n, v] : s.params)  // sorted, the binding order
        if (j < MCB_MAX_PARAMS) d.k[j++] = v;
      d.program = program;
      break;
    }
  }
  for (std::size_t j = 0; j < s.domain.dim() && j < MCB_MAX_DIM; ++j) {
    d.low[j] = s.domain.low[j];
    d.high[j] = s.domain.high[j];
  }
  if (s.method == Method::Stratified || s.method == Method::Tree) {
    const RefineConfig rc = s.method_config.value_or(RefineConfig{});
    d.method = s.method == Method::Tree ? MCB_METHOD_TREE : MCB_METHOD_STRATIFIED;
    d.cells_per_dim = rc.init_cells_per_dim;
    d.cell_cap = rc.cell_cap;
    if (s.method == Method::Tree) {  // total_budget = n_samples (src/batch.cpp:278)
      d.flags |= MCB_FLAG_REFINE_CONFIG;
      d.samples_per_cell = rc.samples_per_cell;
      d.max_depth = rc.max_depth;
      d.sigma_multiplier = rc.sigma_multiplier;
    }
  }
  return d;
}

StratifiedPlan stratified_plan(const IntegrandSpec& spec) {
  IntegrandSpec s = spec;
  s.method = Method::Stratified;
  mcb_integrand d = to_descriptor(s, 0);
  StratifiedPlan p;
  uint64_t n = 0;
  if (mcb_stratified_plan(&d, &p.cells_per_dim, &n, &p.samples_per_cell) != MCB_OK)
    throw std::invalid_argument(mcb_last_error());  // reference: CellBudgetExceeded
  p.n_cells = n;
  return p;
}

std::string IntegrandSpec::source() const {
  if (family == Family::Program || !program_source.empty()) return program_source;
  mcb_integrand d = to_descriptor(*this, 0);
  std::string s(mcb_to_dsl(&d, nullptr, 0), '\0');
  mcb_to_dsl(&d, s.data(), s.size());
  s.pop_back();
  return s;
}

IntegrandSpec IntegrandSpec::from_source(std::string name, const std::string& source,
                                         std::size_t dim, HyperRect domain,
                                         std::map<std::string, double> params,
                                         std::uint64_t n_samples) {
  IntegrandSpec s;
  s.name = std::move(name);
  s.dim = dim;
  s.domain = std::move(domain);
  s.params = std::move(params);
  s.n_samples = n_samples;
  const std::string want = strip(source);
  struct Cand {
    Family f;
    bool unit;
    bool a1;
  };
  const Cand cands[] = {{Family::Harmonic, true, false}, {Family::Harmonic, false, false},
                        {Family::HarmonicVec, false, false}, {Family::Abs2, false, true},
                        {Family::Abs2, false, false}, {Family::Abs3, false, true},
                        {Family::Abs3, false, false}};
  for (const Cand& c : cands) {
    IntegrandSpec t = s;
    t.family = c.f;
    t.unit_coeffs = c.unit;
    t.params["a"] = c.a1 ? 1.0 : 2.0;  // only selects the printed form
    if (c.f == Family::Abs2 && dim < 2) continue;
    if (c.f == Family::Abs3 && dim < 3) continue;
    t.program_source.clear();
    if (strip(t.source()) == want) {
      s.family = c.f;
      s.unit_coeffs = c.unit;
      s.program_source = source;  // keep the caller's text (job-file round trips)
      return s;
    }
  }
  s.family = Family::Program;  // any other source: the GPU interpreter
  s.program_source = source;
  return s;
}

// ---- validation (src/batch.cpp:62-120) --------------------------------------

ValidationError::ValidationError(std::vector<Violation> v)
    : std::runtime_error([&v] {
        std::ostringstream os;
        os << "job validation failed (" << v.size() << " problem(s)):";
        for (const Violation& viol : v) {
          os << "\n  ";
          if (!viol.integrand.empty()) os << viol.integrand << ": ";
          os << viol.message;
        }
        return os.str();
      }()),
      violations(std::move(v)) {}

std::vector<Violation> validate(const JobSpec& job) {
  std::vector<Violation> out;
  std::vector<mcb_integrand> descs;
  std::vector<const char*> names;
  ProgramCache programs;
  for (std::size_t i = 0; i < job.integrands.size(); ++i) {
    const IntegrandSpec& s = job.integrands[i];
    const mcb_program* prog = nullptr;
    if (s.family == Family::Program) {
      try {
        prog = programs.get(s);
      } catch (const std::invalid_argument& e) {
        out.push_back({s.name, e.what()});
      }
    }
    if (s.dim >= 1 && s.domain.dim() != s.dim && s.domain.valid())
      out.push_back({s.name, "domain dimension " + std::to_string(s.domain.dim()) +
                                 " does not match dim=" + std::to_string(s.dim)});
    if (s.domain.dim() > MCB_MAX_DIM || !s.domain.valid())
      out.push_back({s.name, "domain is invalid (need low[i] < high[i], finite, dim >= 1)"});
    for (const std::string& p : required_params(s))
      if (!s.params.count(p)) out.push_back({s.name, "unbound parameter '" + p + "'"});
    descs.push_back(to_descriptor(s, uint32_t(i), prog));
    names.push_back(s.name.c_str());
  }
  std::vector<mcb_violation> v(descs.size() * 8 + 8);
  std::size_t n = 0;
  check(mcb_validate(descs.data(), descs.size(), names.data(), job.trials, v.data(), v.size(), &n));
  for (std::size_t i = 0; i < std::min(n, v.size()); ++i) {
    std::string who = v[i].integrand >= 0 ? job.integrands[std::size_t(v[i].integrand)].name : "";
    std::string msg = v[i].message;
    // the domain check above already reported these with the reference wording
    if (msg.rfind("domain is invalid", 0) == 0) continue;
    if (msg.rfind("program family needs", 0) == 0) continue;  // reported by compile_program
    out.push_back({who, msg});
  }
  return out;
}

// ---- estimator (src/estimator.cpp) ------------------------------------------

std::uint64_t chunk_count(std::uint64_t n) { return (n + kChunkSize - 1) / kChunkSize; }

static McEstimate to_estimate(const mcb_trial_stats& t) {
  McEstimate e;
  e.value = t.value;
  e.std_error = t.std_error;
  e.n_samples = t.n_samples;
  e.n_nonfinite = t.n_nonfinite;
  e.nonfinite_warning = t.nonfinite_warning != 0;
  e.budget_exhausted = t.budget_exhausted != 0;
  return e;
}

// The reference's exception text of a failed trial (src/batch.cpp:172-190).
static std::string trial_error(const mcb_trial_stats& st) {
  switch (st.status) {
    case MCB_TRIAL_DEAD_CELL: return "cell " + std::to_string(st.detail) + " produced no finite sample";
    case MCB_TRIAL_CELL_BUDGET: return "cell grid exceeds configured cap";
    case MCB_TRIAL_CHUNK_RANGE: return "chunk_index exceeds 32 bits";
    default: return "every sample evaluated to NaN or infinity";
  }
}

// ---- per-chunk layer (src/estimator.cpp:9-73) ---------------------------------

void ChunkAccum::add(double x) {
  if (!std::isfinite(x)) {
    n_nonfinite += 1;
    return;
  }
  n += 1;
  const double d = x - mean;  // deviation from the old mean
  mean = mean + d / double(n);
  m2 = m2 + d * (x - mean);   // times the deviation from the new one
}

void ChunkAccum::merge(const ChunkAccum& b) {
  n_nonfinite += b.n_nonfinite;
  if (b.n == 0) return;
  if (n == 0) {
    n = b.n;
    mean = b.mean;
    m2 = b.m2;
    return;
  }
  const std::uint64_t both = n + b.n;
  const double d = b.mean - mean;
  mean = mean + d * (double(b.n) / double(both));
  m2 = m2 + (b.m2 + d * d * (double(n) * double(b.n) / double(both)));
  n = both;
}

ChunkAccum accumulate_chunk(const IntegrandSpec& spec, const StreamKey& key, std::size_t count, int device) {
  if (spec.domain.dim() != spec.dim) throw std::invalid_argument("program/domain dimension mismatch");
  if (key.chunk_index > 0xFFFFFFFFull) throw std::out_of_range("chunk_index exceeds 32 bits");
  if (count > kChunkSize) throw std::invalid_argument("count exceeds the chunk size");
  ProgramCache programs;
  const mcb_program* prog = spec.family == Family::Program ? programs.get(spec) : nullptr;
  const mcb_integrand d = to_descriptor(spec, key.integrand_index, prog);
  mcb_chunk_accum a{};
  check(mcb_accumulate_chunk(&d, key.global_seed, key.trial_index, key.chunk_index, std::uint32_t(count), device,
                             &a));
  return ChunkAccum{a.n, a.n_nonfinite, a.mean, a.m2};
}

McEstimate reduce_chunks(double volume, std::span<const ChunkAccum> chunks) {
  ChunkAccum all;
  for (const ChunkAccum& c : chunks) all.merge(c);
  if (all.n == 0) throw AllSamplesNonFinite("every sample evaluated to NaN or infinity");
  McEstimate e;
  e.n_samples = all.n + all.n_nonfinite;
  e.n_nonfinite = all.n_nonfinite;
  e.value = volume * all.mean;
  e.std_error = all.n >= 2 ? volume * std::sqrt((all.m2 / double(all.n - 1)) / double(all.n))
                           : std::numeric_limits<double>::infinity();
  e.nonfinite_warning = double(all.n_nonfinite) > kNonFiniteWarnFraction * double(e.n_samples);
  return e;
}

McEstimate direct_mc(const IntegrandSpec& spec, std::uint64_t n_samples, const StreamKey& key_base,
                     int device) {
  if (n_samples < 2) throw std::invalid_argument("n_samples must be >= 2");
  if (spec.domain.dim() != spec.dim)
    throw std::invalid_argument("program/domain dimension mismatch");
  ProgramCache programs;
  const mcb_program* prog = spec.family == Family::Program ? programs.get(spec) : nullptr;
  mcb_integrand d = to_descriptor(spec, key_base.integrand_index, prog);
  d.n_samples = n_samples;
  mcb_trial_stats st{};
  check(mcb_direct_mc(&d, key_base.global_seed, key_base.trial_index, key_base.chunk_index, device,
                      &st));
  if (st.status == MCB_TRIAL_ALL_NONFINITE)
    throw AllSamplesNonFinite("every sample evaluated to NaN or infinity");
  if (st.status == MCB_TRIAL_DEAD_CELL)
    throw AllSamplesNonFinite("cell " + std::to_string(st.detail) + " produced no finite sample");
  return to_estimate(st);
}

McEstimate tree_refine(const IntegrandSpec& spec, const RefineConfig& config, const StreamKey& key_base,
                       std::vector<StratumNode>* leaves_out, int device) {  // :212-318
  if (spec.domain.dim() != spec.dim) throw std::invalid_argument("program/domain dimension mismatch");
  IntegrandSpec s = spec;
  s.method = Method::Tree;
  s.method_config = config;
  ProgramCache programs;
  const mcb_program* prog = s.family == Family::Program ? programs.get(s) : nullptr;
  mcb_integrand d = to_descriptor(s, key_base.integrand_index, prog);
  d.n_samples = config.total_budget;
  mcb_trial_stats st{};
  size_t n = 0;
  std::vector<mcb_leaf> lv;
  if (leaves_out) {  // leaf bound: first pass (<= 4096 cells, or the given grid) + one per split
    double grid = 4096.0;
    if (config.init_cells_per_dim) grid = std::pow(double(config.init_cells_per_dim), double(s.dim));
    lv.resize(size_t(std::min(double(1 << 22),
                              grid + double(config.total_budget / std::max<uint32_t>(config.samples_per_cell, 2)) + 1)));
  }
  check(mcb_tree_refine(&d, key_base.global_seed, key_base.trial_index, key_base.chunk_index, device, &st,
                        lv.empty() ? nullptr : lv.data(), lv.size(), &n));
  if (leaves_out && n > lv.size()) {  // past the bound: run again with room for every leaf
    lv.resize(n);
    check(mcb_tree_refine(&d, key_base.global_seed, key_base.trial_index, key_base.chunk_index, device, &st,
                          lv.data(), lv.size(), &n));
  }
  lv.resize(std::min(lv.size(), n));
  if (st.status == MCB_TRIAL_CELL_BUDGET) throw CellBudgetExceeded("cell grid exceeds configured cap");
  if (st.status == MCB_TRIAL_CHUNK_RANGE) throw std::out_of_range("chunk_index exceeds 32 bits");
  if (st.status == MCB_TRIAL_ALL_NONFINITE)
    throw AllSamplesNonFinite("every sample evaluated to NaN or infinity");
  if (leaves_out) {
    leaves_out->clear();
    for (const mcb_leaf& l : lv) {
      StratumNode node;
      node.cell.low.assign(l.low, l.low + s.dim);
      node.cell.high.assign(l.high, l.high + s.dim);
      node.estimate = to_estimate(l.estimate);
      node.depth = l.depth;
      leaves_out->push_back(std::move(node));
    }
  }
  return to_estimate(st);
}

std::pair<McEstimate, std::vector<StratumNode>> stratified_mc(const IntegrandSpec& spec,
                                                              std::uint32_t cells_per_dim,
                                                              std::uint32_t samples_per_cell,
                                                              const StreamKey& key_base, std::uint64_t cell_cap,
                                                              int device) {  // :161-182
  if (spec.domain.dim() != spec.dim) throw std::invalid_argument("program/domain dimension mismatch");
  if (cells_per_dim == 0) throw std::invalid_argument("cells_per_dim must be >= 1");
  IntegrandSpec s = spec;
  s.method = Method::Direct;
  ProgramCache programs;
  const mcb_program* prog = s.family == Family::Program ? programs.get(s) : nullptr;
  mcb_integrand d = to_descriptor(s, key_base.integrand_index, prog);
  mcb_trial_stats st{};
  size_t n = 0;
  std::vector<mcb_leaf> lv(size_t(std::min(double(1 << 22), std::pow(double(cells_per_dim), double(s.dim)))));
  check(mcb_stratified_mc(&d, cells_per_dim, samples_per_cell, cell_cap, key_base.global_seed,
                          key_base.trial_index, key_base.chunk_index, device, &st, lv.data(), lv.size(), &n));
  if (n > lv.size()) {
    lv.resize(n);
    check(mcb_stratified_mc(&d, cells_per_dim, samples_per_cell, cell_cap, key_base.global_seed,
                            key_base.trial_index, key_base.chunk_index, device, &st, lv.data(), lv.size(), &n));
  }
  lv.resize(std::min(lv.size(), n));
  if (st.status == MCB_TRIAL_CELL_BUDGET) throw CellBudgetExceeded("cell grid exceeds configured cap");
  if (st.status == MCB_TRIAL_CHUNK_RANGE) throw std::out_of_range("chunk_index exceeds 32 bits");
  if (st.status != MCB_TRIAL_OK) throw AllSamplesNonFinite("every sample evaluated to NaN or infinity");
  std::vector<StratumNode> leaves;
  leaves.reserve(lv.size());
  for (const mcb_leaf& l : lv) {
    StratumNode node;
    node.cell.low.assign(l.low, l.low + s.dim);
    node.cell.high.assign(l.high, l.high + s.dim);
    node.estimate = to_estimate(l.estimate);
    node.depth = l.depth;
    leaves.push_back(std::move(node));
  }
  return {to_estimate(st), std::move(leaves)};
}

std::uint64_t cell_grid_size(std::uint32_t k, std::size_t dim, std::uint64_t cap) {  // :94-105
  if (k == 0) throw std::invalid_argument("cells_per_dim must be >= 1");
  std::uint64_t cells = 1;
  for (std::size_t i = 0; i < dim; ++i) {
    if (cells > cap / k + 1) throw CellBudgetExceeded("cell grid exceeds configured cap");
    cells *= k;
  }
  if (cells > cap) throw CellBudgetExceeded("cell grid exceeds configured cap");
  return cells;
}

std::uint32_t auto_cells_per_dim(std::size_t dim, std::uint64_t limit) {  // :107-122
  std::uint32_t k = 1;
  for (;;) {
    std::uint64_t cells = 1;
    for (std::size_t i = 0; i < dim; ++i) {
      cells *= std::uint64_t(k) + 1;
      if (cells > limit) return k;
    }
    ++k;
  }
}

HyperRect grid_cell(const HyperRect& rect, std::uint32_t k, std::uint64_t index) {  // :124-143
  const std::size_t d = rect.dim();
  HyperRect cell;
  cell.low.resize(d);
  cell.high.resize(d);
  std::uint64_t rem = index;
  for (std::size_t j = d; j-- > 0;) {  // axis 0 is the most significant digit
    const std::uint32_t digit = std::uint32_t(rem % k);
    rem /= k;
    const double width = rect.high[j] - rect.low[j];
    cell.low[j] = digit == 0 ? rect.low[j] : rect.low[j] + width * (double(digit) / k);
    cell.high[j] = digit + 1 == k ? rect.high[j] : rect.low[j] + width * (double(digit + 1) / k);
  }
  return cell;
}

McEstimate combine_cells(std::span<const McEstimate> cells) {  // :145-159
  McEstimate total;
  double var = 0.0;
  for (const McEstimate& c : cells) {
    total.value += c.value;
    var += c.std_error * c.std_error;
    total.n_samples += c.n_samples;
    total.n_nonfinite += c.n_nonfinite;
    total.budget_exhausted |= c.budget_exhausted;
  }
  total.std_error = std::sqrt(var);
  total.nonfinite_warning = double(total.n_nonfinite) > kNonFiniteWarnFraction * double(total.n_samples);
  return total;
}

TrialSummary summarize_trials(std::vector<McEstimate> per_trial) {  // :320-337
  TrialSummary s;
  s.per_trial = std::move(per_trial);
  const std::size_t r = s.per_trial.size();
  if (r == 0) throw InsufficientTrials("no successful trials");
  double sum = 0.0;
  for (const McEstimate& e : s.per_trial) sum += e.value;
  s.mean = sum / double(r);
  if (r >= 2) {
    double ss = 0.0;
    for (const McEstimate& e : s.per_trial) {
      const double d = e.value - s.mean;
      ss += d * d;
    }
    s.trial_stddev = std::sqrt(ss / double(r - 1));
  }
  return s;
}

TrialSummary repeated_trials(const std::function<McEstimate(std::uint32_t)>& run,
                             std::uint32_t trials) {  // :339-355
  if (trials < 2) throw std::invalid_argument("repeated_trials requires R >= 2");
  std::vector<McEstimate> ok;
  for (std::uint32_t t = 0; t < trials; ++t) {
    try {
      ok.push_back(run(t));
    } catch (const AllSamplesNonFinite&) {
    }
  }
  if (ok.size() < 2) throw InsufficientTrials("fewer than 2 trials produced a finite estimate");
  return summarize_trials(std::move(ok));
}

// ---- batch (src/batch.cpp:195-367) ------------------------------------------

BatchResult run_batch(const JobSpec& job) {
  {
    std::vector<Violation> v = validate(job);
    if (!v.empty()) throw ValidationError(std::move(v));
  }
  const std::size_t n = job.integrands.size();
  const std::uint32_t trials = job.trials;
  std::vector<mcb_integrand> descs(n);
  ProgramCache programs;
  for (std::size_t i = 0; i < n; ++i) {
    const IntegrandSpec& s = job.integrands[i];
    descs[i] = to_descriptor(s, uint32_t(i), s.family == Family::Program ? programs.get(s) : nullptr);
  }
  std::vector<mcb_trial_stats> out(n * trials);
  double seconds = 0.0;
  const std::vector<int> devices = job.devices.empty() ? devices_for_workers(job.workers) : job.devices;
  check(mcb_run_direct(descs.data(), n, job.seed, trials, devices.data(), int(devices.size()), out.data(),
                       &seconds));

  BatchResult result;
  result.total_seconds = seconds;
  double total_cost = 0.0;
  std::vector<double> cost(n);
  for (std::size_t i = 0; i < n; ++i) {
    cost[i] = double(out[i * trials].n_samples) * double(descs[i].dim);
    total_cost += cost[i];
  }
  for (std::size_t i = 0; i < n; ++i) {
    IntegrandResult r;
    r.name = job.integrands[i].name;
    r.seconds = total_cost > 0 ? seconds * cost[i] / total_cost : 0.0;
    std::vector<McEstimate> ok;
    std::string first_error;
    for (std::uint32_t t = 0; t < trials; ++t) {
      const mcb_trial_stats& st = out[i * trials + t];
      if (st.status == MCB_TRIAL_OK) {
        McEstimate e = to_estimate(st);
        r.nonfinite_warning |= e.nonfinite_warning;
        r.budget_exhausted |= e.budget_exhausted;
        ok.push_back(e);
      } else if (first_error.empty()) {
        first_error = "trial " + std::to_string(t) + ": " + trial_error(st);
      }
    }
    const std::size_t need = trials >= 2 ? 2 : 1;  // src/batch.cpp:320
    if (ok.size() >= need) {
      r.ok = true;
      r.summary = summarize_trials(std::move(ok));
      if (!first_error.empty()) r.error = "partial: " + first_error;
    } else {
      r.ok = false;
      r.error = first_error.empty() ? "no successful trials" : first_error;
    }
    result.per_integrand.push_back(std::move(r));
  }
  return result;
}

std::vector<TrialSummary> parameter_scan(const IntegrandSpec& tmpl, const std::string& param_name,
                                         std::span<const double> values, std::uint32_t trials,
                                         std::uint64_t seed, std::vector<int> devices) {
  if (!tmpl.params.count(param_name))
    throw std::invalid_argument("parameter '" + param_name + "' is not bound in the template");
  if (values.empty()) throw std::invalid_argument("parameter_scan needs at least one value");
  JobSpec job;
  job.seed = seed;
  job.trials = trials;
  job.devices = std::move(devices);
  job.integrands.reserve(values.size());
  for (std::size_t i = 0; i < values.size(); ++i) {
    IntegrandSpec s = tmpl;
    s.name = tmpl.name + "#" + std::to_string(i);
    s.params[param_name] = values[i];
    job.integrands.push_back(std::move(s));
  }
  BatchResult br = run_batch(job);
  std::vector<TrialSummary> out;
  out.reserve(br.per_integrand.size());
  for (IntegrandResult& r : br.per_integrand) {
    if (!r.ok) throw std::runtime_error("parameter_scan: " + r.name + " failed: " + r.error);
    out.push_back(std::move(r.summary));
  }
  return out;
}

// ---- harmonic benchmark (src/job_io.cpp:336-376) -----------------------------

double harmonic_k(std::uint32_t n) { return (double(n) + 50.0) / (2.0 * std::numbers::pi); }

double harmonic_closed_form(double k, std::size_t dim) {
  if (k == 0.0) return 1.0;
  std::complex<double> ik(0.0, k);
  std::complex<double> phi = (std::exp(ik) - 1.0) / ik;
  std::complex<double> p = phi;
  for (std::size_t j = 1; j < dim; ++j) p = p * phi;
  return p.real() + p.imag();
}

double analytic_harmonic(std::uint32_t n) {
  if (n < 1) throw std::invalid_argument("n must be >= 1");
  return harmonic_closed_form(harmonic_k(n), 4);
}

JobSpec make_harmonic_job(std::uint32_t n_count, std::uint64_t samples) {
  if (n_count < 1) throw std::invalid_argument("n_count must be >= 1");
  JobSpec job;
  job.seed = 20200814;
  job.trials = 10;
  const int width = int(std::to_string(n_count).size());
  for (std::uint32_t n = 1; n <= n_count; ++n) {
    IntegrandSpec s;
    char name[32];
    std::snprintf(name, sizeof name, "f%0*u", width, n);
    s.name = name;
    s.family = Family::Harmonic;
    s.unit_coeffs = true;
    s.dim = 4;
    s.domain = HyperRect::unit(4);
    s.params["k"] = harmonic_k(n);
    s.n_samples = samples;
    job.integrands.push_back(std::move(s));
  }
  return job;
}

}  // namespace mcb
