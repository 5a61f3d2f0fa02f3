// ref_shim.cpp — extern "C" shim over the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file
// together with the reference's own sources, read in place from
// /root/reference/proj/src/{expr,sampling,estimator,batch,job_io}.cpp, into
// oracle/_ref/libmcbatch_ref.so (git-ignored; never shipped in the product).
// It exists so that (1) tests/golden/make_golden.py can dump golden vectors
// produced by the reference itself and (2) bench.py's cpu_baseline and
// `--impl reference` legs time the reference's own run_batch
// (src/batch.cpp:195-333) with its own thread pool.
//
// No reference source is copied here: this file only includes the public
// headers (include/mcbatch/*.hpp) and calls the public API.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <map>
#include <string>
#include <vector>

#include "mcb/mcb.h"
#include "mcbatch/batch.hpp"
#include "mcbatch/estimator.hpp"
#include "mcbatch/expr.hpp"
#include "mcbatch/job_io.hpp"
#include "mcbatch/sampling.hpp"

using namespace mcbatch;

namespace {

thread_local std::string g_err;

HyperRect rect_of(std::uint32_t dim, const double* lo, const double* hi) {
  HyperRect r;
  r.low.assign(lo, lo + dim);
  r.high.assign(hi, hi + dim);
  return r;
}

// Parameter binding for a family descriptor (names as in mcb_to_dsl).
std::map<std::string, double> params_of(const mcb_integrand& f) {
  std::map<std::string, double> p;
  switch (f.family) {
    case MCB_FAMILY_HARMONIC:
      p["k"] = f.k[0];
      if (!(f.flags & MCB_FLAG_UNIT_COEFFS)) {
        p["a"] = f.a;
        p["b"] = f.b;
      }
      break;
    case MCB_FAMILY_HARMONIC_VEC:
      p["a"] = f.a;
      p["b"] = f.b;
      for (std::uint32_t j = 0; j < f.dim; ++j) p["k" + std::to_string(j + 1)] = f.k[j];
      break;
    default:
      p["a"] = f.a;
      break;
  }
  return p;
}

void fill(const McEstimate& e, mcb_trial_stats* st) {
  st->value = e.value;
  st->std_error = e.std_error;
  st->n_samples = e.n_samples;
  st->n_nonfinite = e.n_nonfinite;
  st->status = MCB_TRIAL_OK;
  st->nonfinite_warning = e.nonfinite_warning ? 1u : 0u;
  st->budget_exhausted = e.budget_exhausted ? 1u : 0u;
}

// RefineConfig of a STRATIFIED / TREE descriptor (mcb.h field meanings).
RefineConfig refine_config_of(const mcb_integrand& f) {
  RefineConfig rc;
  rc.init_cells_per_dim = f.cells_per_dim;
  if (f.cell_cap) rc.cell_cap = f.cell_cap;
  if (f.flags & MCB_FLAG_REFINE_CONFIG) {
    rc.samples_per_cell = f.samples_per_cell;
    rc.max_depth = f.max_depth;
    rc.sigma_multiplier = f.sigma_multiplier;
  }
  rc.total_budget = f.n_samples;
  return rc;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// sample_uniform (src/sampling.cpp:102-112) with StreamKey {seed, i, t, c}.
int ref_sample_uniform(std::uint32_t dim, const double* lo, const double* hi,
                       std::uint64_t seed, std::uint32_t integrand, std::uint32_t trial,
                       std::uint64_t chunk, std::uint64_t count, double* out) {
  try {
    std::vector<double> pts =
        sample_uniform(rect_of(dim, lo, hi), StreamKey{seed, integrand, trial, chunk}, count);
    std::memcpy(out, pts.data(), pts.size() * sizeof(double));
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// CompiledProgram::evaluate (src/expr.cpp:520-553) of `source` on n points.
int ref_eval_points(const char* source, const mcb_integrand* f, const double* pts,
                    std::uint64_t n, double* out) {
  try {
    auto pm = params_of(*f);
    std::vector<std::string> names;
    std::vector<double> vals;
    for (auto& [k, v] : pm) { names.push_back(k); vals.push_back(v); }
    CompiledProgram prog = compile(parse(source), f->dim, names);
    std::vector<double> stack;
    for (std::uint64_t i = 0; i < n; ++i)
      out[i] = prog.evaluate({pts + i * f->dim, f->dim}, vals, stack);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// direct_mc (src/estimator.cpp:75-92) of the lowered family source.
int ref_direct_mc(const char* source, const mcb_integrand* f, std::uint64_t seed,
                  std::uint32_t trial, std::uint64_t chunk_base, mcb_trial_stats* out) {
  try {
    auto pm = params_of(*f);
    std::vector<std::string> names;
    std::vector<double> vals;
    for (auto& [k, v] : pm) { names.push_back(k); vals.push_back(v); }
    CompiledProgram prog = compile(parse(source), f->dim, names);
    std::memset(out, 0, sizeof *out);
    try {
      McEstimate e = direct_mc(prog, vals, rect_of(f->dim, f->low, f->high), f->n_samples,
                               StreamKey{seed, f->integrand_index, trial, chunk_base});
      fill(e, out);
    } catch (const AllSamplesNonFinite&) {
      out->status = MCB_TRIAL_ALL_NONFINITE;
      out->n_samples = f->n_samples;
      out->n_nonfinite = f->n_samples;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// run_batch (src/batch.cpp:195-333) of n integrands given as lowered sources
// + descriptors (integrand_index must equal the list position, as in the
// reference).  out_trials: n*trials McEstimates (status ALL_NONFINITE for a
// failed trial); out_mean/out_sd/out_ok per integrand; *seconds =
// BatchResult.total_seconds.
int ref_run_batch(const char* const* sources, const mcb_integrand* fns, std::size_t n,
                  std::uint64_t seed, std::uint32_t trials, std::uint32_t workers,
                  mcb_trial_stats* out_trials, double* out_mean, double* out_sd,
                  std::int32_t* out_ok, double* seconds) {
  try {
    JobSpec job;
    job.seed = seed;
    job.trials = trials;
    job.workers = workers;
    for (std::size_t i = 0; i < n; ++i) {
      IntegrandSpec s;
      s.name = "f" + std::to_string(i);
      s.source = sources[i];
      s.dim = fns[i].dim;
      s.domain = rect_of(fns[i].dim, fns[i].low, fns[i].high);
      s.params = params_of(fns[i]);
      s.n_samples = fns[i].n_samples;
      s.method = fns[i].method == MCB_METHOD_STRATIFIED
                     ? Method::Stratified
                     : (fns[i].method == MCB_METHOD_TREE ? Method::Tree : Method::Direct);
      if (s.method != Method::Direct) s.method_config = refine_config_of(fns[i]);
      job.integrands.push_back(std::move(s));
    }
    BatchResult br = run_batch(job);
    for (std::size_t i = 0; i < n; ++i) {
      const IntegrandResult& r = br.per_integrand[i];
      out_ok[i] = r.ok ? 1 : 0;
      out_mean[i] = r.ok ? r.summary.mean : NAN;
      out_sd[i] = r.ok ? r.summary.trial_stddev : NAN;
      for (std::uint32_t t = 0; t < trials; ++t) std::memset(&out_trials[i * trials + t], 0, sizeof(mcb_trial_stats));
      // per_trial holds only the successful trials, in ascending order; a
      // fully successful integrand has exactly `trials` of them.
      if (r.ok && r.summary.per_trial.size() == trials)
        for (std::uint32_t t = 0; t < trials; ++t)
          fill(r.summary.per_trial[t], &out_trials[i * trials + t]);
    }
    if (seconds) *seconds = br.total_seconds;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// make_harmonic_job (src/job_io.cpp:355-376): the reference's own k_n values.
int ref_harmonic_job(std::uint32_t n_count, std::uint64_t samples, double* k_out,
                     std::uint64_t* seed_out, std::uint32_t* trials_out) {
  try {
    JobSpec job = make_harmonic_job(n_count, samples);
    for (std::uint32_t i = 0; i < n_count; ++i) k_out[i] = job.integrands[i].params.at("k");
    *seed_out = job.seed;
    *trials_out = job.trials;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Timing leg of bench.py (reference arm and cpu_baseline): the reference's
// own make_harmonic_job(n_total, samples) (src/job_io.cpp:355-376), of which
// the integrands at positions first, first + stride, ... (count of them) form
// the job that the reference's run_batch (src/batch.cpp:195-333) runs with
// `workers` threads (0 = all hardware threads, batch.cpp:56-60).  The subset
// keeps each integrand's source, k, domain and budget; its integrand_index is
// its position in the subset (the reference's rule), so the streams differ
// from the full job's while the per-sample cost is the same.  Returns
// BatchResult.total_seconds (validate/compile excluded, batch.cpp:293-299),
// the worker count the reference resolved and the number of integrands whose
// trials all succeeded.
int ref_run_harmonic(std::uint32_t n_total, std::uint64_t samples, std::uint32_t first,
                     std::uint32_t count, std::uint32_t stride, std::uint32_t workers,
                     double* seconds, std::uint32_t* workers_used, std::uint32_t* n_ok) {
  try {
    JobSpec full = make_harmonic_job(n_total, samples);
    JobSpec job;
    job.seed = full.seed;
    job.trials = full.trials;
    job.workers = workers;
    for (std::uint32_t i = 0; i < count; ++i) {
      std::size_t pos = std::size_t(first) + std::size_t(i) * stride;
      if (pos >= full.integrands.size()) break;
      job.integrands.push_back(full.integrands[pos]);
    }
    BatchResult br = run_batch(job);
    std::uint32_t ok = 0;
    for (const IntegrandResult& r : br.per_integrand) ok += r.ok ? 1u : 0u;
    *seconds = br.total_seconds;
    *workers_used = resolve_workers(workers);
    *n_ok = ok;
    return int(job.integrands.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Expression front-end dump (parity of include/mcbatch/expr.hpp): for
// `source` compiled for `dim` coordinates and the comma-separated parameter
// names, one line "OK <stack_need> <postfix> <tree_eval hex> <to_string>" or
// "ERR <error class>".  Postfix: op:index:value-hex per instruction.
// The same format is printed by tests/cpp/test_compat.cpp for our layer.
int ref_expr_dump(const char* source, std::uint32_t dim, const char* names_csv, const double* point,
                  const double* params, char* out, std::size_t cap) {
  std::string line;
  std::vector<std::string> names;
  for (std::string cur, all = names_csv; !all.empty();) {
    std::size_t c = all.find(',');
    names.push_back(all.substr(0, c));
    all = c == std::string::npos ? "" : all.substr(c + 1);
  }
  auto hex = [](double v) {
    std::uint64_t u;
    std::memcpy(&u, &v, 8);
    char b[24];
    std::snprintf(b, sizeof b, "%016llx", (unsigned long long)u);
    return std::string(b);
  };
  try {
    Expr e = parse(source);
    CompiledProgram p = compile(e, dim, names);
    line = "OK " + std::to_string(p.stack_need()) + " ";
    for (const Instr& in : p.code())
      line += std::to_string(int(in.op)) + ":" + std::to_string(in.index) + ":" + hex(in.value) + ",";
    line += " " + hex(tree_eval(e, {point, dim}, names, {params, names.size()}));
    line += " " + std::to_string(parse(to_string(e)) == e);
  } catch (const SyntaxError&) {
    line = "ERR SyntaxError";
  } catch (const UnknownFunction&) {
    line = "ERR UnknownFunction";
  } catch (const ArityMismatch&) {
    line = "ERR ArityMismatch";
  } catch (const DimensionError&) {
    line = "ERR DimensionError";
  } catch (const UnboundParameter&) {
    line = "ERR UnboundParameter";
  } catch (const std::exception& ex) {
    line = std::string("ERR other");
  }
  std::snprintf(out, cap, "%s", line.c_str());
  return int(line.size());
}

// evaluate (src/expr.cpp:520-553) of an arbitrary source with named params.
int ref_eval_source(const char* source, std::uint32_t dim, const char* const* names,
                    const double* values, std::size_t n_params, const double* pts,
                    std::uint64_t n, double* out) {
  try {
    std::map<std::string, double> pm;
    for (std::size_t i = 0; i < n_params; ++i) pm[names[i]] = values[i];
    std::vector<std::string> nm;
    std::vector<double> vals;
    for (auto& [k, v] : pm) { nm.push_back(k); vals.push_back(v); }
    CompiledProgram prog = compile(parse(source), dim, nm);
    std::vector<double> stack;
    for (std::uint64_t i = 0; i < n; ++i) out[i] = prog.evaluate({pts + i * dim, dim}, vals, stack);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// direct_mc (src/estimator.cpp:75-92) of an arbitrary source.
int ref_direct_mc_source(const char* source, std::uint32_t dim, const char* const* names,
                         const double* values, std::size_t n_params, const double* lo,
                         const double* hi, std::uint64_t n_samples, std::uint64_t seed,
                         std::uint32_t index, std::uint32_t trial, std::uint64_t chunk_base,
                         mcb_trial_stats* out) {
  try {
    std::map<std::string, double> pm;
    for (std::size_t i = 0; i < n_params; ++i) pm[names[i]] = values[i];
    std::vector<std::string> nm;
    std::vector<double> vals;
    for (auto& [k, v] : pm) { nm.push_back(k); vals.push_back(v); }
    CompiledProgram prog = compile(parse(source), dim, nm);
    std::memset(out, 0, sizeof *out);
    try {
      fill(direct_mc(prog, vals, rect_of(dim, lo, hi), n_samples,
                     StreamKey{seed, index, trial, chunk_base}),
           out);
    } catch (const AllSamplesNonFinite&) {
      out->status = MCB_TRIAL_ALL_NONFINITE;
      out->n_samples = n_samples;
      out->n_nonfinite = n_samples;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// tree_refine (src/estimator.cpp:212-318) of an arbitrary source, config from
// the descriptor; leaves (cap entries) in the reference's order.
int ref_tree_refine_source(const char* source, const mcb_integrand* f, const char* const* names,
                           const double* values, std::size_t n_params, std::uint64_t seed,
                           std::uint32_t trial, std::uint64_t chunk_base, mcb_trial_stats* out,
                           mcb_leaf* leaves, std::size_t cap, std::size_t* n_leaves) {
  try {
    std::map<std::string, double> pm;
    for (std::size_t i = 0; i < n_params; ++i) pm[names[i]] = values[i];
    std::vector<std::string> nm;
    std::vector<double> vals;
    for (auto& [k, v] : pm) { nm.push_back(k); vals.push_back(v); }
    CompiledProgram prog = compile(parse(source), f->dim, nm);
    std::memset(out, 0, sizeof *out);
    std::vector<StratumNode> lv;
    try {
      fill(tree_refine(prog, vals, rect_of(f->dim, f->low, f->high), refine_config_of(*f),
                       StreamKey{seed, f->integrand_index, trial, chunk_base}, &lv),
           out);
    } catch (const AllSamplesNonFinite&) {
      out->status = MCB_TRIAL_ALL_NONFINITE;
    } catch (const CellBudgetExceeded&) {
      out->status = MCB_TRIAL_CELL_BUDGET;
    }
    out->n_cells = std::uint32_t(lv.size());
    if (n_leaves) *n_leaves = lv.size();
    for (std::size_t i = 0; i < lv.size() && i < cap; ++i) {
      std::memset(&leaves[i], 0, sizeof leaves[i]);
      for (std::uint32_t j = 0; j < f->dim; ++j) {
        leaves[i].low[j] = lv[i].cell.low[j];
        leaves[i].high[j] = lv[i].cell.high[j];
      }
      fill(lv[i].estimate, &leaves[i].estimate);
      leaves[i].depth = lv[i].depth;
      out->max_depth = std::max(out->max_depth, lv[i].depth);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// stratified_mc (src/estimator.cpp:161-182) of an arbitrary source; leaves
// (cap entries) in grid order.  A dead cell gives status DEAD_CELL.
int ref_stratified_mc_source(const char* source, const mcb_integrand* f, const char* const* names,
                             const double* values, std::size_t n_params, std::uint32_t cells_per_dim,
                             std::uint32_t samples_per_cell, std::uint64_t cell_cap, std::uint64_t seed,
                             std::uint32_t trial, std::uint64_t chunk_base, mcb_trial_stats* out,
                             mcb_leaf* leaves, std::size_t cap, std::size_t* n_leaves) {
  try {
    std::map<std::string, double> pm;
    for (std::size_t i = 0; i < n_params; ++i) pm[names[i]] = values[i];
    std::vector<std::string> nm;
    std::vector<double> vals;
    for (auto& [k, v] : pm) { nm.push_back(k); vals.push_back(v); }
    CompiledProgram prog = compile(parse(source), f->dim, nm);
    std::memset(out, 0, sizeof *out);
    if (n_leaves) *n_leaves = 0;
    try {
      auto [est, lv] = stratified_mc(prog, vals, rect_of(f->dim, f->low, f->high), cells_per_dim,
                                     samples_per_cell, StreamKey{seed, f->integrand_index, trial, chunk_base},
                                     cell_cap ? cell_cap : 1000000);
      fill(est, out);
      out->n_cells = std::uint32_t(lv.size());
      if (n_leaves) *n_leaves = lv.size();
      for (std::size_t i = 0; i < lv.size() && i < cap; ++i) {
        std::memset(&leaves[i], 0, sizeof leaves[i]);
        for (std::uint32_t j = 0; j < f->dim; ++j) {
          leaves[i].low[j] = lv[i].cell.low[j];
          leaves[i].high[j] = lv[i].cell.high[j];
        }
        fill(lv[i].estimate, &leaves[i].estimate);
      }
    } catch (const AllSamplesNonFinite&) {
      out->status = MCB_TRIAL_DEAD_CELL;
    } catch (const CellBudgetExceeded&) {
      out->status = MCB_TRIAL_CELL_BUDGET;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// read_job + write_job (src/job_io.cpp:114-142): re-serialise a job file.
int ref_job_roundtrip(const char* in_path, const char* out_path) {
  try {
    JobSpec job = read_job(in_path);
    write_job(job, out_path);
    return int(job.integrands.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// read_results + write_results (src/job_io.cpp:207-284): re-serialise a CSV.
int ref_results_roundtrip(const char* in_path, const char* out_path) {
  try {
    auto rows = read_results(in_path);
    write_results(rows, out_path);
    return int(rows.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// run_command (src/job_io.cpp): the reference CLI's `run` (tools/mcbatch.cpp
// needs CLI11, absent from the image; its `run` is this call).  workers < 0
// keeps the job's own worker count.
int ref_run_command(const char* job_path, const char* out_path, int workers) {
  try {
    RunOverrides ov;
    if (workers >= 0) ov.workers = std::uint32_t(workers);
    return run_command(job_path, out_path, ov);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

double ref_harmonic_closed_form(double k) { return harmonic_closed_form(k); }
double ref_analytic_harmonic(std::uint32_t n) { return analytic_harmonic(n); }

}  // extern "C"
