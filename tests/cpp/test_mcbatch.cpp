// C++ API tests (include/mcb/mcbatch.hpp) on the GPU, mirroring the
// reference's own suites case by case:
//   tests/test_batch.cpp, tests/test_estimator.cpp, tests/test_sampling.cpp,
//   tests/test_job_io.cpp (harmonic generator), tests/acceptance.cpp C2/C3.
// Built and run by tests/test_cpp_api.py (pytest -m gpu).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numbers>
#include <string>
#include <vector>

#include "mcb/mcbatch.hpp"

using namespace mcb;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                     \
  do {                                                                  \
    if (cond) {                                                         \
      ++g_pass;                                                         \
    } else {                                                            \
      ++g_fail;                                                         \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);      \
    }                                                                   \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                        \
  do {                                                                  \
    bool caught_ = false;                                               \
    try {                                                               \
      (void)(expr);                                                     \
    } catch (const T&) {                                                \
      caught_ = true;                                                   \
    } catch (...) {                                                     \
    }                                                                   \
    CHECK(caught_);                                                     \
  } while (0)

static IntegrandSpec harmonic(std::string name, double k, std::size_t dim, HyperRect dom,
                              std::uint64_t n, double a = 1.0, double b = 1.0) {
  IntegrandSpec s;
  s.name = std::move(name);
  s.family = Family::Harmonic;
  s.unit_coeffs = (a == 1.0 && b == 1.0);
  s.dim = dim;
  s.domain = std::move(dom);
  s.params = {{"k", k}};
  if (!s.unit_coeffs) {
    s.params["a"] = a;
    s.params["b"] = b;
  }
  s.n_samples = n;
  return s;
}

static IntegrandSpec absf(std::string name, Family f, std::size_t dim, HyperRect dom, std::uint64_t n,
                          double a = 1.0) {
  IntegrandSpec s;
  s.name = std::move(name);
  s.family = f;
  s.dim = dim;
  s.domain = std::move(dom);
  s.params = {{"a", a}};
  s.n_samples = n;
  return s;
}

// tests/test_batch.cpp:29-43 — constants are exact (k = 0: a*cos 0 + b*sin 0 = a)
static void constants_are_exact() {
  JobSpec job;
  job.seed = 1;
  job.trials = 3;
  job.integrands.push_back(harmonic("c7", 0.0, 1, HyperRect::unit(1), 1000, 7.0, 3.0));
  job.integrands.push_back(harmonic("c5", 0.0, 1, HyperRect::box({0}, {2}), 1000, 5.0, 1.5));
  BatchResult br = run_batch(job);
  CHECK(br.per_integrand.size() == 2);
  CHECK(br.per_integrand[0].ok);
  CHECK(br.per_integrand[0].summary.mean == 7.0);
  CHECK(br.per_integrand[0].summary.trial_stddev == 0.0);
  CHECK(br.per_integrand[1].summary.mean == 10.0);
  CHECK(br.per_integrand[1].summary.trial_stddev == 0.0);
  for (const McEstimate& e : br.per_integrand[0].summary.per_trial) CHECK(e.std_error == 0.0);
}

// tests/test_batch.cpp:45-58 and acceptance.cpp:73-103 (criterion 2)
static void mixed_dimension_batch() {
  JobSpec job;
  job.seed = 7;
  job.trials = 2;
  job.integrands.push_back(absf("g1", Family::Abs2, 2, HyperRect::unit(2), 100000));
  job.integrands.push_back(absf("g2", Family::Abs3, 3, HyperRect::unit(3), 100000));
  BatchResult br = run_batch(job);
  const double se0 = br.per_integrand[0].summary.per_trial[0].std_error;
  const double se1 = br.per_integrand[1].summary.per_trial[0].std_error;
  CHECK(std::fabs(br.per_integrand[0].summary.mean - 1.0) <= 3.0 * se0);
  CHECK(std::fabs(br.per_integrand[1].summary.mean - 7.0 / 12.0) <= 3.0 * se1);
  CHECK(job.integrands[0].source() == "abs(x1+x2)");
  CHECK(job.integrands[1].source() == "abs(x1+x2-x3)");
}

// tests/test_batch.cpp:60-89
static void validate_reports_every_violation() {
  JobSpec job;
  job.seed = 0;
  job.trials = 1;
  job.integrands.push_back(absf("a", Family::Abs3, 2, HyperRect::unit(2), 1000));
  job.integrands.push_back(harmonic("a", 1.0, 1, HyperRect::unit(1), 1000));
  IntegrandSpec unbound = harmonic("b", 1.0, 1, HyperRect::unit(1), 1000);
  unbound.params.clear();
  job.integrands.push_back(unbound);
  job.integrands.push_back(harmonic("c", 1.0, 2, HyperRect::unit(3), 1000));
  job.integrands.push_back(harmonic("d", 1.0, 1, HyperRect::unit(1), 1));
  auto v = validate(job);
  auto has = [&](const std::string& name, const std::string& frag) {
    for (const Violation& viol : v)
      if (viol.integrand == name && viol.message.find(frag) != std::string::npos) return true;
    return false;
  };
  CHECK(has("a", "x3 exceeds dim=2"));
  CHECK(has("a", "duplicate"));
  CHECK(has("b", "unbound parameter 'k'"));
  CHECK(has("c", "does not match dim=2"));
  CHECK(has("d", "samples must be >= 2"));
  CHECK_THROWS_AS(run_batch(job), ValidationError);
  JobSpec good;
  good.trials = 2;
  good.integrands.push_back(harmonic("ok", 1.0, 1, HyperRect::unit(1), 100));
  CHECK(validate(good).empty());
}

// tests/test_batch.cpp:91-121 and acceptance.cpp:106-133, for device lists
static void device_invariance() {
  JobSpec job;
  job.seed = 99;
  job.trials = 2;
  job.integrands.push_back(harmonic("osc", 9.0, 2, HyperRect::unit(2), 150000));
  job.integrands.push_back(absf("lin", Family::Abs3, 3, HyperRect::unit(3), 70000, 0.7));
  job.integrands.push_back(harmonic("h7", 2.5, 7, HyperRect::unit(7), 130001, 0.5, 2.0));
  std::vector<BatchResult> runs;
  for (std::vector<int> d : {std::vector<int>{0}, std::vector<int>{0, 0}, std::vector<int>{0, 0, 0, 0}}) {
    job.devices = d;
    runs.push_back(run_batch(job));
  }
  for (std::size_t r = 1; r < runs.size(); ++r)
    for (std::size_t i = 0; i < job.integrands.size(); ++i) {
      const TrialSummary& a = runs[0].per_integrand[i].summary;
      const TrialSummary& b = runs[r].per_integrand[i].summary;
      CHECK(std::memcmp(&a.mean, &b.mean, sizeof(double)) == 0);
      CHECK(std::memcmp(&a.trial_stddev, &b.trial_stddev, sizeof(double)) == 0);
      for (std::size_t t = 0; t < a.per_trial.size(); ++t) {
        CHECK(a.per_trial[t].value == b.per_trial[t].value);
        CHECK(a.per_trial[t].std_error == b.per_trial[t].std_error);
      }
    }
}

// tests/test_batch.cpp:123-135
static void failing_integrand_isolated() {
  JobSpec job;
  job.seed = 3;
  job.trials = 2;
  job.devices = {0, 0};
  job.integrands.push_back(harmonic("dead", 1.0, 1, HyperRect::unit(1), 1000, NAN, 1.0));
  job.integrands.push_back(absf("alive", Family::Abs2, 2, HyperRect::unit(2), 1000));
  BatchResult br = run_batch(job);
  CHECK(!br.per_integrand[0].ok);
  CHECK(!br.per_integrand[0].error.empty());
  CHECK(br.per_integrand[1].ok);
}

// tests/test_batch.cpp:137-158
static void depends_only_on_seed_index_spec() {
  IntegrandSpec a = harmonic("a", 1.0, 1, HyperRect::unit(1), 20000, 0.0, 1.0);   // sin(x1)
  IntegrandSpec b = harmonic("b", 1.0, 1, HyperRect::unit(1), 20000, 1.0, 0.0);   // cos(x1)
  JobSpec both;
  both.seed = 5;
  both.trials = 2;
  both.integrands = {a, b};
  JobSpec only_a = both;
  only_a.integrands = {a};
  BatchResult rb = run_batch(both);
  BatchResult ra = run_batch(only_a);
  CHECK(rb.per_integrand[0].summary.mean == ra.per_integrand[0].summary.mean);
  JobSpec moved = both;
  std::swap(moved.integrands[0], moved.integrands[1]);
  BatchResult rm = run_batch(moved);
  CHECK(rm.per_integrand[1].name == "a");
  CHECK(rm.per_integrand[1].summary.mean != rb.per_integrand[0].summary.mean);
}

// tests/test_batch.cpp:160-210
static void parameter_scans() {
  IntegrandSpec tmpl = harmonic("const", 0.0, 1, HyperRect::unit(1), 1000, 0.0, 1.0);
  double values[] = {1.0, 2.0, 3.0};
  auto out = parameter_scan(tmpl, "a", values, 2, 11);
  CHECK(out.size() == 3);
  CHECK(out[0].mean == 1.0);
  CHECK(out[1].mean == 2.0);
  CHECK(out[2].mean == 3.0);

  // sin(k*x1) on [0, pi]: a = 0, b = 1
  IntegrandSpec sine = harmonic("sine", 0.0, 1, HyperRect::box({0.0}, {std::numbers::pi}), 200000, 0.0, 1.0);
  double ks[] = {1.0, 2.0};
  auto so = parameter_scan(sine, "k", ks, 2, 12);
  CHECK(std::fabs(so[0].mean - 2.0) <= 3.0 * so[0].per_trial[0].std_error);
  CHECK(std::fabs(so[1].mean - 0.0) <= 3.0 * so[1].per_trial[0].std_error);

  IntegrandSpec h = harmonic("h", 0.0, 2, HyperRect::unit(2), 30000, 1.0, 0.0);  // cos(k*(x1+x2))
  double hv[] = {2.0, 4.0, 8.0};
  auto scanned = parameter_scan(h, "k", hv, 2, 77);
  JobSpec job;
  job.seed = 77;
  job.trials = 2;
  for (std::size_t i = 0; i < 3; ++i) {
    IntegrandSpec s = h;
    s.name = "x" + std::to_string(i);
    s.params["k"] = hv[i];
    job.integrands.push_back(s);
  }
  BatchResult br = run_batch(job);
  for (std::size_t i = 0; i < 3; ++i) {
    CHECK(scanned[i].mean == br.per_integrand[i].summary.mean);
    CHECK(scanned[i].trial_stddev == br.per_integrand[i].summary.trial_stddev);
  }
  double one[] = {1.0};
  CHECK_THROWS_AS(parameter_scan(h, "missing", one, 2, 0), std::invalid_argument);
  CHECK_THROWS_AS(parameter_scan(h, "a", std::span<const double>{}, 2, 0), std::invalid_argument);
}

// tests/test_estimator.cpp:44-85, 194-238
static void estimator_cases() {
  IntegrandSpec c7 = harmonic("c", 0.0, 2, HyperRect::box({0, 0}, {2, 2}), 1000, 7.0, 0.0);
  McEstimate est = direct_mc(c7, 1000, StreamKey{1, 0, 0, 0});
  CHECK(est.value == 28.0);
  CHECK(est.std_error == 0.0);
  CHECK(est.n_samples == 1000);
  CHECK(est.n_nonfinite == 0);

  const double k = 51.0 / (2.0 * std::numbers::pi);
  IntegrandSpec h = IntegrandSpec::from_source("h", "cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))", 4,
                                               HyperRect::unit(4), {{"k", k}}, 1000000);
  CHECK(h.family == Family::Harmonic && h.unit_coeffs);
  McEstimate e1 = direct_mc(h, 1000000, StreamKey{77, 0, 0, 0});
  const double truth = harmonic_closed_form(k, 4);
  CHECK(std::fabs(truth - (-0.001999358381010922)) <= 1e-12 * 0.002);
  CHECK(std::fabs(e1.value - truth) <= 3.0 * e1.std_error);
  // reference value of this exact estimate (tests/golden: reference direct_mc)
  CHECK(std::fabs(e1.value - (-0.0031516902787214725)) <= 1e-12);

  IntegrandSpec ab = absf("ab", Family::Abs2, 2, HyperRect::unit(2), 1000000);
  McEstimate e2 = direct_mc(ab, 1000000, StreamKey{3, 0, 0, 0});
  CHECK(std::fabs(e2.value - 1.0) <= 3.0 * e2.std_error);

  IntegrandSpec dead = harmonic("dead", 1.0, 1, HyperRect::unit(1), 100, NAN, 1.0);
  CHECK_THROWS_AS(direct_mc(dead, 100, StreamKey{9, 0, 0, 0}), AllSamplesNonFinite);

  // repeated_trials (tests/test_estimator.cpp:194-222)
  IntegrandSpec two = harmonic("two", 0.0, 1, HyperRect::unit(1), 100, 2.0, 0.0);
  TrialSummary s = repeated_trials(
      [&](std::uint32_t t) { return direct_mc(two, 100, StreamKey{7, 0, t, 0}); }, 10);
  CHECK(s.per_trial.size() == 10);
  CHECK(s.mean == 2.0);
  CHECK(s.trial_stddev == 0.0);
  CHECK_THROWS_AS(repeated_trials([&](std::uint32_t t) { return direct_mc(two, 100, StreamKey{7, 0, t, 0}); }, 1),
                  std::invalid_argument);
  CHECK_THROWS_AS(repeated_trials([&](std::uint32_t t) { return direct_mc(dead, 100, StreamKey{7, 0, t, 0}); }, 3),
                  InsufficientTrials);

  // seeded linearity (tests/test_estimator.cpp:224-238): same keys, a*f
  IntegrandSpec f1 = harmonic("f1", 3.0, 1, HyperRect::unit(1), 10000, 1.0, 0.5);
  IntegrandSpec f3 = harmonic("f3", 3.0, 1, HyperRect::unit(1), 10000, 3.0, 1.5);
  McEstimate ef = direct_mc(f1, 10000, StreamKey{13, 1, 0, 0});
  McEstimate ef3 = direct_mc(f3, 10000, StreamKey{13, 1, 0, 0});
  CHECK(std::fabs(ef3.value - 3.0 * ef.value) <= 1e-12 * std::fabs(ef3.value));
}

// tests/test_sampling.cpp:19-104 and tests/test_job_io.cpp:140-151
static void sampling_and_generator() {
  auto a = sample_uniform(HyperRect::unit(1), StreamKey{123, 4, 5, 6}, 3);
  auto b = sample_uniform(HyperRect::unit(1), StreamKey{123, 4, 5, 6}, 3);
  CHECK(a == b);
  auto unit = sample_uniform(HyperRect::unit(1), StreamKey{99, 0, 0, 0}, 10000);
  auto mapped = sample_uniform(HyperRect::box({-1.5}, {2.25}), StreamKey{99, 0, 0, 0}, 10000);
  bool exact = true;
  for (std::size_t i = 0; i < unit.size(); ++i) exact &= mapped[i] == -1.5 + (2.25 - -1.5) * unit[i];
  CHECK(exact);
  auto pts = sample_uniform(HyperRect::box({0, 10}, {1, 20}), StreamKey{5, 0, 0, 0}, 1000);
  bool inb = pts.size() == 2000;
  for (std::size_t i = 0; i + 1 < pts.size(); i += 2)
    inb &= pts[i] >= 0.0 && pts[i] < 1.0 && pts[i + 1] >= 10.0 && pts[i + 1] < 20.0;
  CHECK(inb);
  CHECK_THROWS_AS(HyperRect::box({1}, {1}), InvalidDomain);

  JobSpec job = make_harmonic_job(100, 1000000);
  CHECK(job.integrands.size() == 100);
  CHECK(job.trials == 10);
  CHECK(std::fabs(job.integrands[0].params.at("k") - 8.116902097686662) <= 1e-15 * 8.2);
  CHECK(std::fabs(job.integrands[99].params.at("k") - 23.873241463784303) <= 1e-15 * 24);
  CHECK(job.integrands[0].source() == "cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))");
  CHECK(validate(job).empty());
  CHECK(std::fabs(analytic_harmonic(1) - (-0.001999358381010922)) <= 1e-12 * 0.002);
  CHECK(std::fabs(analytic_harmonic(50) - 0.00032173407630372935) <= 1e-12 * 0.00033);
}

// acceptance.cpp:53-69 (criterion 1) at the full Fig. 1 budget
static void fig1_band() {
  JobSpec job = make_harmonic_job(100, 1000000);
  BatchResult br = run_batch(job);
  int passed = 0;
  for (std::uint32_t n = 1; n <= 100; ++n) {
    const TrialSummary& s = br.per_integrand[n - 1].summary;
    double mse = 0;
    for (const McEstimate& e : s.per_trial) mse += e.std_error;
    mse = mse / double(s.per_trial.size()) / std::sqrt(double(s.per_trial.size()));
    const double band = 4.0 * std::fmax(s.trial_stddev, mse);
    passed += std::fabs(s.mean - analytic_harmonic(n)) <= band;
  }
  std::printf("Fig.1: %d/100 inside the 4-sigma band, %.3f s\n", passed, br.total_seconds);
  CHECK(passed >= 95);
}

// tests/test_estimator.cpp:140-192 — tree_refine
static void tree_cases() {
  auto prog = [](std::string src, std::size_t dim) {
    return IntegrandSpec::from_source("t", src, dim, HyperRect::unit(dim), {}, 100000);
  };
  {  // constant integrand needs no refinement
    RefineConfig cfg;
    cfg.total_budget = 100000;
    std::vector<StratumNode> leaves;
    McEstimate est = tree_refine(prog("5", 2), cfg, StreamKey{1, 0, 0, 0}, &leaves);
    CHECK(std::fabs(est.value - 5.0) <= 5e-12);
    CHECK(est.std_error == 0.0);
    CHECK(!est.budget_exhausted);
    CHECK(est.n_samples <= cfg.total_budget);
    CHECK(leaves.size() == 16);
  }
  {  // gaussian peak covers the closed form; leaves tile the domain
    const double truth = 0.03141592653580133;
    RefineConfig cfg;
    cfg.total_budget = 100000;
    std::vector<StratumNode> leaves;
    McEstimate est =
        tree_refine(prog("exp(-100*((x1-0.5)^2+(x2-0.5)^2))", 2), cfg, StreamKey{21, 0, 0, 0}, &leaves);
    CHECK(std::fabs(est.value - truth) <= 3.0 * est.std_error);
    double vol = 0.0;
    for (const StratumNode& n : leaves) vol += n.cell.volume();
    CHECK(std::fabs(vol - 1.0) <= 1e-12);
    CHECK(est.n_samples <= cfg.total_budget);
  }
  {  // budget exhaustion is flagged, not an error
    RefineConfig cfg;
    cfg.init_cells_per_dim = 2;
    cfg.samples_per_cell = 256;
    cfg.total_budget = 1200;
    McEstimate est = tree_refine(prog("exp(-100*((x1-0.3)^2+(x2-0.3)^2))", 2), cfg, StreamKey{31, 0, 0, 0});
    CHECK(est.budget_exhausted);
    CHECK(std::isfinite(est.value));
  }
  {  // agrees with direct_mc on the oscillatory integrand
    const double k = 150.0 / (2.0 * std::numbers::pi);
    IntegrandSpec f = harmonic("osc", k, 4, HyperRect::unit(4), 200000);
    RefineConfig cfg;
    cfg.total_budget = 200000;
    McEstimate tree = tree_refine(f, cfg, StreamKey{5, 0, 0, 0});
    McEstimate direct = direct_mc(f, 200000, StreamKey{5, 0, 1, 0});
    const double band = 3.0 * std::sqrt(tree.std_error * tree.std_error + direct.std_error * direct.std_error);
    CHECK(std::fabs(tree.value - direct.value) <= band);
  }
  {  // failures throw like the reference
    RefineConfig cfg;
    cfg.cell_cap = 3;
    CHECK_THROWS_AS(tree_refine(prog("exp(x1)", 2), cfg, StreamKey{16, 0, 0, 0}), CellBudgetExceeded);
    RefineConfig c2;
    c2.samples_per_cell = 100;
    c2.total_budget = 10000;
    CHECK_THROWS_AS(tree_refine(prog("sqrt(-1-x1)", 1), c2, StreamKey{9, 0, 0, 0}), AllSamplesNonFinite);
  }
  {  // run_batch Tree branch: budget = n_samples, budget_exhausted reported, devices invariant
    JobSpec job;
    job.seed = 3;
    job.trials = 3;
    IntegrandSpec t = prog("exp(-100*((x1-0.3)^2+(x2-0.3)^2))", 2);
    t.name = "peak";
    t.method = Method::Tree;
    RefineConfig rc;
    rc.init_cells_per_dim = 2;
    rc.samples_per_cell = 256;
    t.method_config = rc;
    t.n_samples = 1200;
    job.integrands.push_back(t);
    IntegrandSpec h = harmonic("h", 3.0, 2, HyperRect::unit(2), 50000);
    h.method = Method::Tree;
    job.integrands.push_back(h);
    CHECK(validate(job).empty());
    BatchResult a = run_batch(job);
    CHECK(a.per_integrand[0].ok && a.per_integrand[0].budget_exhausted);
    CHECK(a.per_integrand[1].ok);
    job.devices = {0, 0};
    BatchResult b = run_batch(job);
    for (int i = 0; i < 2; ++i)
      for (int r = 0; r < 3; ++r) {
        const McEstimate &x = a.per_integrand[i].summary.per_trial[r], &y = b.per_integrand[i].summary.per_trial[r];
        CHECK(std::memcmp(&x.value, &y.value, 8) == 0 && std::memcmp(&x.std_error, &y.std_error, 8) == 0 &&
              x.n_samples == y.n_samples && x.budget_exhausted == y.budget_exhausted);
      }
  }
}

// tests/test_estimator.cpp:87-138 — stratified_mc and the cell helpers
static void stratified_cases() {
  IntegrandSpec f = IntegrandSpec::from_source("s", "sin(x1)*x2", 2, HyperRect::box({0.25, -1.0}, {0.75, 3.0}),
                                               {}, 5000);
  auto [one, leaves1] = stratified_mc(f, 1, 5000, StreamKey{11, 2, 0, 0});
  McEstimate d = direct_mc(f, 5000, StreamKey{11, 2, 0, 0});
  CHECK(leaves1.size() == 1);
  CHECK(std::fabs(one.value - d.value) <= 1e-13 * std::fabs(d.value));  // 1x1 cells = direct_mc
  auto [est, leaves] = stratified_mc(f, 4, 200, StreamKey{3, 0, 0, 0});
  CHECK(leaves.size() == 16);
  double vol = 0.0;
  for (const StratumNode& n : leaves) vol += n.cell.volume();
  CHECK(std::fabs(vol - 2.0) <= 1e-12);
  CHECK(est.n_samples == 16 * 200);
  CHECK(cell_grid_size(4, 2, 1000000) == 16);
  CHECK_THROWS_AS(cell_grid_size(10, 7, 1000000), CellBudgetExceeded);
  CHECK(auto_cells_per_dim(4, 4096) == 8);
  const HyperRect c = grid_cell(HyperRect::box({0.25, -1.0}, {0.75, 3.0}), 4, 5);
  CHECK(c.low == leaves[5].cell.low && c.high == leaves[5].cell.high);
  std::vector<McEstimate> cells;
  for (const StratumNode& n : leaves) cells.push_back(n.estimate);
  const McEstimate comb = combine_cells(cells);
  CHECK(comb.value == est.value && comb.std_error == est.std_error);
  IntegrandSpec lg = IntegrandSpec::from_source("l", "log(x1)", 1, HyperRect::box({-1.0}, {1.0}), {}, 4000);
  CHECK_THROWS_AS(stratified_mc(lg, 4, 1000, StreamKey{9, 0, 0, 0}), AllSamplesNonFinite);
  CHECK_THROWS_AS(stratified_mc(f, 10, 10, StreamKey{3, 0, 0, 0}, 50), CellBudgetExceeded);
}

// src/batch.cpp:302-331: trials that fail are dropped; the integrand is ok
// ("partial: trial t: ...") with at least two successful trials when trials
// >= 2, else failed.  One stratified cell of 2 samples of sqrt(x1 - 0.5) on
// [0,1]: a trial whose two points (cell 0 = chunk key 0, StreamKey {seed, 0,
// t, 0}, points 0 and 1 — checked independently with sample_uniform) both lie
// below 0.5 has a dead cell and fails.
static void partial_trials() {
  for (std::uint32_t trials : {12u, 3u}) {
    IntegrandSpec s = IntegrandSpec::from_source("half", "sqrt(x1 - 0.5)", 1, HyperRect::unit(1), {}, 2);
    s.method = Method::Stratified;
    RefineConfig rc;
    rc.init_cells_per_dim = 1;
    s.method_config = rc;
    for (std::uint64_t seed = 1; seed < 40; ++seed) {
      JobSpec job;
      job.seed = seed;
      job.trials = trials;
      job.integrands = {s};
      std::vector<std::uint32_t> dead;
      for (std::uint32_t t = 0; t < trials; ++t) {
        const std::vector<double> x = sample_uniform(HyperRect::unit(1), StreamKey{seed, 0, t, 0}, 2);
        if (x[0] < 0.5 && x[1] < 0.5) dead.push_back(t);
      }
      if (dead.empty()) continue;
      const BatchResult br = run_batch(job);
      const IntegrandResult& r = br.per_integrand[0];
      const std::size_t n_ok = trials - dead.size();
      const std::string first = "trial " + std::to_string(dead[0]) + ": ";
      if (n_ok >= 2) {
        CHECK(r.ok);
        CHECK(r.summary.per_trial.size() == n_ok);
        CHECK(r.error.rfind("partial: " + first, 0) == 0);
      } else {
        CHECK(!r.ok);
        CHECK(r.error.rfind(first, 0) == 0);
      }
    }
  }
}

#define RUN(f)                                         \
  do {                                                 \
    if (std::getenv("MCB_TEST_TRACE")) {               \
      std::fprintf(stderr, "[test] %s\n", #f);        \
      std::fflush(stderr);                             \
    }                                                  \
    f();                                               \
  } while (0)

int main() {
  RUN(constants_are_exact);
  RUN(tree_cases);
  RUN(stratified_cases);
  RUN(mixed_dimension_batch);
  RUN(validate_reports_every_violation);
  RUN(device_invariance);
  RUN(failing_integrand_isolated);
  RUN(depends_only_on_seed_index_spec);
  RUN(parameter_scans);
  RUN(estimator_cases);
  RUN(sampling_and_generator);
  RUN(fig1_band);
  RUN(partial_trials);
  std::printf("%d checks passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
