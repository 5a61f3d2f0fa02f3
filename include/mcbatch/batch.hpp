// mcbatch/batch.hpp — source-compatible face of the reference header
// include/mcbatch/batch.hpp over libmcb: the reference's IntegrandSpec
// (free DSL `source`) and JobSpec (`workers`), run_batch, validate,
// parameter_scan.  Specs are lowered to libmcb's family descriptors when the
// source is a built-in family and to GPU-interpreted programs otherwise
// (mcb::IntegrandSpec::from_source); every estimate is computed on the GPU.
//
// `workers` keeps its meaning "how many parallel executors": here, how many
// GPUs (0 = every visible device; more than are visible = all of them).
// Results do not depend on it, as in the reference (batch.hpp:68-71).
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "mcb/mcbatch.hpp"
#include "mcbatch/estimator.hpp"
#include "mcbatch/expr.hpp"
#include "mcbatch/sampling.hpp"

namespace mcbatch {

using mcb::Method;
using mcb::method_name;
std::optional<Method> method_from_name(std::string_view name);

// The reference's integrand (batch.hpp:22-31): a free DSL source whose
// parameters bind in the map's sorted name order.
struct IntegrandSpec {
  std::string name;                       // unique within a job
  std::string source;                     // DSL text, e.g. "a*abs(x1+x2)"
  std::size_t dim{1};                     // coordinates x1..x_dim
  HyperRect domain;                       // dim-dimensional box
  std::map<std::string, double> params;   // every free parameter of `source`
  std::uint64_t n_samples{10000};         // per trial (the tree's total budget)
  Method method{Method::Direct};
  std::optional<RefineConfig> method_config;  // stratified / tree settings
};

// batch.hpp:33-38
struct JobSpec {
  std::uint64_t seed{0};
  std::uint32_t trials{1};
  std::uint32_t workers{0};               // GPUs here (0 = every visible device)
  std::vector<IntegrandSpec> integrands;  // integrand_index = position
};

using mcb::Violation;
using mcb::ValidationError;
std::vector<Violation> validate(const JobSpec& job);

using mcb::BatchResult;
using mcb::IntegrandResult;
BatchResult run_batch(const JobSpec& job);

std::vector<TrialSummary> parameter_scan(const IntegrandSpec& tmpl, const std::string& param_name,
                                         std::span<const double> values, std::uint32_t trials,
                                         std::uint64_t seed, std::uint32_t workers = 0);

using mcb::StratifiedPlan;
StratifiedPlan stratified_plan(const IntegrandSpec& spec);

// The executor count a request resolves to: `requested`, or for 0 the number
// of visible GPUs (at least 1).
std::uint32_t resolve_workers(std::uint32_t requested);

// Lowering both ways (integrand order and every field kept).
mcb::IntegrandSpec to_mcb(const IntegrandSpec& spec);
mcb::JobSpec to_mcb(const JobSpec& job);
IntegrandSpec from_mcb(const mcb::IntegrandSpec& spec);
JobSpec from_mcb(const mcb::JobSpec& job);

}  // namespace mcbatch
