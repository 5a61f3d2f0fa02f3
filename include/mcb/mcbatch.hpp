// mcbatch.hpp — C++ host API mirroring the reference `mcbatch` direct path
// (/root/reference/proj/include/mcbatch/{sampling,estimator,batch,job_io}.hpp),
// implemented over the C-ABI in mcb.h and executed by the sm_100a kernels.
//
// Differences from the reference, all deliberate:
//  * IntegrandSpec carries a family descriptor (`family` + `params` map using
//    the DSL parameter names a, b, k, k1..kd); `source()` returns the exact
//    DSL the reference would parse.  Any other DSL source runs as
//    Family::Program (GPU interpreter, same sampler and reduction);
//    `IntegrandSpec::from_source()` picks the family when the source is one
//    of them and Program otherwise, so reference IntegrandSpecs port as-is.
//  * JobSpec::workers (CPU threads) becomes JobSpec::devices (CUDA ordinals).
//    Results are byte-identical for any device list, the analogue of the
//    reference's worker invariance (tests/test_batch.cpp:91-121).
//  * Every method runs on the GPU: Direct and Stratified as fused launches,
//    Tree as host-driven refinement rounds whose cells (of every tree in the
//    batch) are estimated by the same fused kernels (csrc/tree.cpp).
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mcb/mcb.h"

namespace mcb {

inline constexpr std::size_t kChunkSize = MCB_CHUNK_SIZE;             // sampling.hpp:11
inline constexpr double kNonFiniteWarnFraction = MCB_NONFINITE_WARN_FRACTION;  // estimator.hpp:16

// include/mcbatch/sampling.hpp:14-24
struct HyperRect {
  std::vector<double> low;
  std::vector<double> high;

  std::size_t dim() const { return low.size(); }
  bool valid() const;
  double volume() const;

  static HyperRect unit(std::size_t d);
  static HyperRect box(std::vector<double> lo, std::vector<double> hi);
};

struct InvalidDomain : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// include/mcbatch/sampling.hpp:33-44
struct StreamKey {
  std::uint64_t global_seed = 0;
  std::uint32_t integrand_index = 0;
  std::uint32_t trial_index = 0;
  std::uint64_t chunk_index = 0;

  StreamKey with_chunk(std::uint64_t c) const {
    StreamKey k = *this;
    k.chunk_index = c;
    return k;
  }
};

// sample_uniform (src/sampling.cpp:102-112), computed on the GPU.
std::vector<double> sample_uniform(const HyperRect& rect, const StreamKey& key, std::size_t count,
                                   int device = 0);

enum class Family {
  Harmonic = MCB_FAMILY_HARMONIC,         // a*cos(k*(x1+..+xd)) + b*sin(k*(x1+..+xd))
  HarmonicVec = MCB_FAMILY_HARMONIC_VEC,  // a*cos(k1*x1+..+kd*xd) + b*sin(...)
  Abs2 = MCB_FAMILY_ABS2,                 // a*abs(x1+x2)
  Abs3 = MCB_FAMILY_ABS3,                 // a*abs(x1+x2-x3)
  Program = MCB_FAMILY_PROGRAM            // any DSL source (`program_source`)
};

enum class Method { Direct, Stratified, Tree };
const char* method_name(Method m);

// include/mcbatch/estimator.hpp:40-47 (stratified uses init_cells_per_dim
// and cell_cap; run_batch sets a tree's total_budget to n_samples)
struct RefineConfig {
  std::uint32_t init_cells_per_dim = 0;  // 0 = auto (k^d <= min(4096, n/2))
  std::uint32_t samples_per_cell = 2048;
  std::uint32_t max_depth = 6;
  double sigma_multiplier = 1.0;
  std::uint64_t total_budget = 100000;
  std::uint64_t cell_cap = 1000000;
};

// include/mcbatch/batch.hpp:22-31 with a family descriptor.
struct IntegrandSpec {
  std::string name;
  Family family = Family::Harmonic;
  bool unit_coeffs = false;  // Harmonic only: the Fig.1 form cos(..) + sin(..)
  std::size_t dim = 1;
  HyperRect domain;
  std::map<std::string, double> params;  // a, b, k | a, b, k1..kd | a
  std::uint64_t n_samples = 10000;
  Method method = Method::Direct;
  std::optional<RefineConfig> method_config;
  std::string program_source;  // the DSL source (Family::Program; kept verbatim by from_source)

  // Exact reference DSL source of this descriptor.
  std::string source() const;
  // A reference IntegrandSpec: a built-in family when `source` is one of
  // their DSL forms (whitespace insensitive), else Family::Program.
  static IntegrandSpec from_source(std::string name, const std::string& source, std::size_t dim,
                                   HyperRect domain, std::map<std::string, double> params,
                                   std::uint64_t n_samples);
};

struct JobSpec {
  std::uint64_t seed = 0;
  std::uint32_t trials = 1;
  std::uint32_t workers = 0;  // GPUs to use when `devices` is empty (0 = all visible)
  std::vector<int> devices;   // explicit CUDA ordinals
  std::vector<IntegrandSpec> integrands;
};

// Devices for a worker count: 0..workers-1, or every visible GPU for 0.
std::vector<int> devices_for_workers(std::uint32_t workers);

struct Violation {
  std::string integrand;  // empty for job-level problems
  std::string message;
};

std::vector<Violation> validate(const JobSpec& job);

struct ValidationError : std::runtime_error {
  std::vector<Violation> violations;
  explicit ValidationError(std::vector<Violation> v);
};

// include/mcbatch/estimator.hpp:18-31
struct McEstimate {
  double value = 0.0;
  double std_error = 0.0;
  std::uint64_t n_samples = 0;
  std::uint64_t n_nonfinite = 0;
  bool nonfinite_warning = false;
  bool budget_exhausted = false;
};

struct TrialSummary {
  std::vector<McEstimate> per_trial;
  double mean = 0.0;
  double trial_stddev = 0.0;
};

struct AllSamplesNonFinite : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InsufficientTrials : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// A CUDA / device failure (there is no CPU fallback).
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// include/mcbatch/batch.hpp:53-66
struct IntegrandResult {
  std::string name;
  bool ok = false;
  std::string error;
  TrialSummary summary;
  double seconds = 0.0;  // cost-weighted share of the batch's sampling time
  bool nonfinite_warning = false;
  bool budget_exhausted = false;
};

struct BatchResult {
  std::vector<IntegrandResult> per_integrand;  // job order
  double total_seconds = 0.0;
};

// src/batch.cpp:195-333
BatchResult run_batch(const JobSpec& job);

// include/mcbatch/batch.hpp:84-91 (src/batch.cpp:41-54)
struct StratifiedPlan {
  std::uint32_t cells_per_dim = 1;
  std::uint32_t samples_per_cell = 2;
  std::uint64_t n_cells = 1;
};
StratifiedPlan stratified_plan(const IntegrandSpec& spec);

// src/batch.cpp:335-367
std::vector<TrialSummary> parameter_scan(const IntegrandSpec& tmpl, const std::string& param_name,
                                         std::span<const double> values, std::uint32_t trials,
                                         std::uint64_t seed, std::vector<int> devices = {});

// src/estimator.cpp:75-92; throws AllSamplesNonFinite like the reference.
McEstimate direct_mc(const IntegrandSpec& spec, std::uint64_t n_samples, const StreamKey& key_base,
                     int device = 0);

// include/mcbatch/estimator.hpp:59-68: one chunk's accumulator.  add / merge
// are the reference's host recurrences (src/estimator.cpp:9-34).
struct ChunkAccum {
  std::uint64_t n = 0;
  std::uint64_t n_nonfinite = 0;
  double mean = 0.0;
  double m2 = 0.0;

  void add(double x);
  void merge(const ChunkAccum& other);
};

// src/estimator.cpp:36-49: the chunk `key` (count <= kChunkSize points of the
// spec's domain) as one tile of the fused kernel on `device` (mcb_accumulate_chunk).
ChunkAccum accumulate_chunk(const IntegrandSpec& spec, const StreamKey& key, std::size_t count,
                            int device = 0);

// src/estimator.cpp:55-73: chunks merged in the given order, then the
// McEstimate; throws AllSamplesNonFinite when no finite sample survived.
McEstimate reduce_chunks(double volume, std::span<const ChunkAccum> chunks);

// include/mcbatch/estimator.hpp:33-38
struct StratumNode {
  HyperRect cell;
  McEstimate estimate;
  std::uint32_t depth = 0;
};
struct CellBudgetExceeded : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// src/estimator.cpp:161-182: cells_per_dim^d grid cells of samples_per_cell
// samples, combine_cells; throws AllSamplesNonFinite for a cell without a
// finite sample, CellBudgetExceeded past cell_cap.
std::pair<McEstimate, std::vector<StratumNode>> stratified_mc(const IntegrandSpec& spec,
                                                              std::uint32_t cells_per_dim,
                                                              std::uint32_t samples_per_cell,
                                                              const StreamKey& key_base,
                                                              std::uint64_t cell_cap = 1000000,
                                                              int device = 0);

// Host helpers of the cell methods (src/estimator.cpp:94-159).
std::uint64_t cell_grid_size(std::uint32_t cells_per_dim, std::size_t dim, std::uint64_t cap);  // throws
std::uint32_t auto_cells_per_dim(std::size_t dim, std::uint64_t cell_limit);
HyperRect grid_cell(const HyperRect& rect, std::uint32_t cells_per_dim, std::uint64_t index);
McEstimate combine_cells(std::span<const McEstimate> cells);

// src/estimator.cpp:212-318 with the config's total_budget; cells estimated on
// `device`.  Throws AllSamplesNonFinite / CellBudgetExceeded like the reference.
McEstimate tree_refine(const IntegrandSpec& spec, const RefineConfig& config, const StreamKey& key_base,
                       std::vector<StratumNode>* leaves_out = nullptr, int device = 0);

// src/estimator.cpp:320-337
TrialSummary summarize_trials(std::vector<McEstimate> per_trial);

// src/estimator.cpp:339-355
TrialSummary repeated_trials(const std::function<McEstimate(std::uint32_t)>& run,
                             std::uint32_t trials);

std::uint64_t chunk_count(std::uint64_t n_samples);

// src/job_io.cpp:336-376 (harmonic benchmark family of Fig. 1)
double harmonic_k(std::uint32_t n);
double harmonic_closed_form(double k, std::size_t dim = 4);
double analytic_harmonic(std::uint32_t n);
JobSpec make_harmonic_job(std::uint32_t n_count, std::uint64_t samples);

// Lowering to the C-ABI descriptor (integrand_index = list position).
// Family::Program needs a compiled program (see compile_program).
mcb_integrand to_descriptor(const IntegrandSpec& spec, std::uint32_t integrand_index,
                            const mcb_program* program = nullptr);

// Compiled DSL program shared by Program integrands (RAII over mcb_program).
struct CompiledSource {
  mcb_program* handle = nullptr;
  CompiledSource() = default;
  CompiledSource(const CompiledSource&) = delete;
  CompiledSource& operator=(const CompiledSource&) = delete;
  CompiledSource(CompiledSource&& o) noexcept : handle(o.handle) { o.handle = nullptr; }
  CompiledSource& operator=(CompiledSource&& o) noexcept {
    std::swap(handle, o.handle);
    return *this;
  }
  ~CompiledSource() { mcb_program_destroy(handle); }
};
// Throws std::invalid_argument with the reference's validation wording.
CompiledSource compile_program(const std::string& source, std::size_t dim,
                               const std::map<std::string, double>& params);

}  // namespace mcb
