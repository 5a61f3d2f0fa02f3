// Job files, results tables and the Fig. 1 checker (include/mcb/job_io.hpp),
// mirroring the reference's tests/test_job_io.cpp case by case.  Runs without
// a GPU except the `run` cases (argv[1] == "gpu").  Writes its files under
// argv[2] (a scratch directory) so tests/test_job_io.py can hand them to the
// reference for the cross-reads.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <limits>
#include <numbers>
#include <string>

#include "mcb/job_io.hpp"

using namespace mcb;
namespace fs = std::filesystem;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                \
  do {                                                             \
    if (cond) {                                                    \
      ++g_pass;                                                    \
    } else {                                                       \
      ++g_fail;                                                    \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond); \
    }                                                              \
  } while (0)
#define CHECK_THROWS_AS(expr, T)   \
  do {                             \
    bool caught_ = false;          \
    try {                          \
      (void)(expr);                \
    } catch (const T&) {           \
      caught_ = true;              \
    } catch (...) {                \
    }                              \
    CHECK(caught_);                \
  } while (0)

static fs::path dir;

static IntegrandSpec spec(std::string name, std::string src, std::size_t dim, HyperRect dom,
                          std::uint64_t n, std::map<std::string, double> params = {}) {
  return IntegrandSpec::from_source(std::move(name), src, dim, std::move(dom), std::move(params), n);
}

// test_job_io.cpp:52-81 — JSON round trip
static void json_round_trip() {
  JobSpec job;
  job.seed = 123456789012345ull;
  job.trials = 7;
  job.workers = 3;
  job.integrands.push_back(spec("h1", "cos(k*(x1+x2)) + sin(k*(x1+x2))", 2, HyperRect::box({0, -1}, {1, 2.5}),
                                1000, {{"k", 0.1}}));
  IntegrandSpec s2 = spec("p", "exp(-a*x1^2) * log(1+x2)", 2, HyperRect::unit(2), 99, {{"a", 3.25}});
  s2.method = Method::Stratified;
  RefineConfig rc;
  rc.init_cells_per_dim = 3;
  rc.sigma_multiplier = 1.5;
  s2.method_config = rc;
  job.integrands.push_back(s2);
  job.integrands.push_back(spec("abs", "abs(x1+x2-x3)", 3, HyperRect::unit(3), 5000));
  const fs::path p = dir / "roundtrip_job.json";
  write_job(job, p);
  JobSpec back = read_job(p);
  CHECK(back.seed == job.seed && back.trials == job.trials && back.workers == job.workers);
  CHECK(back.integrands.size() == 3);
  for (std::size_t i = 0; i < 3; ++i) {
    const IntegrandSpec &a = job.integrands[i], &b = back.integrands[i];
    CHECK(a.name == b.name);
    CHECK(a.source() == b.source());
    CHECK(a.dim == b.dim);
    CHECK(a.domain.low == b.domain.low && a.domain.high == b.domain.high);
    CHECK(a.params == b.params);
    CHECK(a.n_samples == b.n_samples);
    CHECK(a.method == b.method);
    CHECK(a.family == b.family);
  }
  CHECK(back.integrands[0].family == Family::Harmonic && back.integrands[0].unit_coeffs);
  CHECK(back.integrands[1].family == Family::Program);
  CHECK(back.integrands[1].method_config && back.integrands[1].method_config->init_cells_per_dim == 3);
  CHECK(back.integrands[1].method_config->sigma_multiplier == 1.5);
  CHECK(back.integrands[2].family == Family::Abs3);
}

// test_job_io.cpp:83-96 — strict fields
static void strict_fields() {
  CHECK_THROWS_AS(job_from_json_text(R"({"seed":1,"trials":1,"integrands":[],"extra":2})"), JobFileError);
  CHECK_THROWS_AS(job_from_json_text(R"({"seed":1,"integrands":[]})"), JobFileError);
  CHECK_THROWS_AS(job_from_json_text(R"({"seed":1,"trials":1,"integrands":[{"name":"a","expr":"x1",
      "dim":1,"low":[0],"high":[1],"samples":10,"colour":"red"}]})"),
                  JobFileError);
  CHECK_THROWS_AS(job_from_json_text("{not json"), JobFileError);
  CHECK_THROWS_AS(job_from_json_text("[1,2]"), JobFileError);
  CHECK_THROWS_AS(job_from_json_text(R"({"seed":1,"trials":1,"integrands":[{"name":"a","expr":"x1",
      "dim":1,"low":[0],"high":[1],"samples":10,"method":"quantum"}]})"),
                  JobFileError);
  try {
    job_from_json_text(R"({"seed":1,"trials":1,"integrands":[],"bogus":1})");
  } catch (const JobFileError& e) {
    CHECK(std::string(e.what()) == "unknown field 'bogus' in job");
  }
  JobSpec ok = job_from_json_text(R"({"seed": 5, "trials": 2, "integrands": [
      {"name": "t", "expr": "x1 * a", "dim": 1, "low": [0], "high": [1e0], "samples": 10,
       "params": {"a": -2.5E-1}, "method": "direct"}]})");
  CHECK(ok.integrands.size() == 1 && ok.integrands[0].source() == "x1 * a");
  CHECK(ok.integrands[0].params.at("a") == -0.25);
}

// test_job_io.cpp:98-138 — 17-digit CSV round trip, bit-exact
static void csv_round_trip() {
  std::vector<ResultsRow> rows;
  for (int i = 0; i < 6; ++i) {
    ResultsRow r;
    r.name = "r" + std::to_string(i);
    r.index = uint32_t(i + 1);
    r.dim = 4;
    r.method = "direct";
    r.samples = 1000000;
    r.trials = 10;
    r.ok = i != 3;
    r.mean = std::sin(double(i) * 1.2345) / 3.0;
    r.trial_stddev = 1.0 / (double(i) + 3.0);
    r.mean_std_error = std::nextafter(1e-3, 1.0) * double(i + 1);
    if (i % 2) r.analytic = std::cos(double(i)) * 1e-7;
    if (i % 3 == 0) r.abs_error = 1e-300 * double(i + 1);
    r.warnings = i == 3 ? "FAILED;trial 0: boom" : (i == 4 ? "nonfinite" : "");
    if (i == 3) r.mean = r.trial_stddev = r.mean_std_error = std::numeric_limits<double>::quiet_NaN();
    rows.push_back(r);
  }
  const fs::path p = dir / "roundtrip_results.csv";
  write_results(rows, p);
  auto back = read_results(p);
  CHECK(back.size() == rows.size());
  for (std::size_t i = 0; i < rows.size(); ++i) {
    if (i != 3) {
      CHECK(back[i].mean == rows[i].mean);
      CHECK(back[i].trial_stddev == rows[i].trial_stddev);
      CHECK(back[i].mean_std_error == rows[i].mean_std_error);
    } else {
      CHECK(std::isnan(back[i].mean) && !back[i].ok);
    }
    CHECK(back[i].analytic == rows[i].analytic);
    CHECK(back[i].abs_error == rows[i].abs_error);
    CHECK(back[i].warnings == rows[i].warnings);
  }
  std::ofstream(dir / "empty.csv").close();
  CHECK_THROWS_AS(read_results(dir / "empty.csv"), MalformedResults);
}

// test_job_io.cpp:140-151 and :194-224 — generator and checker
static void fig1_generator_and_checker() {
  gen_fig1(100, 1000000, dir / "fig1_job.json");
  JobSpec job = read_job(dir / "fig1_job.json");
  CHECK(job.integrands.size() == 100 && job.trials == 10 && job.seed == 20200814);
  CHECK(std::fabs(job.integrands[0].params.at("k") - 8.116902097686662) <= 1e-15 * 8.2);
  CHECK(job.integrands[0].family == Family::Harmonic && job.integrands[0].unit_coeffs);
  CHECK(job.integrands[0].source() == "cos(k*(x1+x2+x3+x4)) + sin(k*(x1+x2+x3+x4))");
  CHECK(validate(job).empty());
  std::vector<ResultsRow> rows;
  for (std::uint32_t n = 1; n <= 20; ++n) {
    ResultsRow r;
    char name[16];
    std::snprintf(name, sizeof name, "f%02u", n);
    r.name = name;
    r.index = n;
    r.ok = true;
    r.mean = analytic_harmonic(n) + 1e-5;
    r.trial_stddev = 1e-4;
    r.mean_std_error = 1e-4;
    rows.push_back(r);
  }
  Fig1Check c = check_fig1(rows);
  CHECK(c.passed == 20);
  for (auto& r : rows) r.mean = 0.0;  // sabotage
  Fig1Check bad = check_fig1(rows);
  CHECK(bad.passed < 20);
  CHECK_THROWS_AS(check_fig1({}), MalformedResults);
}

// test_job_io.cpp:233-284 — run_command exit codes (GPU)
static void run_command_exit_codes() {
  const fs::path good = dir / "good_job.json", out = dir / "good_out.csv";
  {
    JobSpec job;
    job.seed = 5;
    job.trials = 2;
    job.workers = 1;
    job.integrands.push_back(spec("c7", "7", 1, HyperRect::unit(1), 100));
    job.integrands.push_back(spec("c5", "5", 1, HyperRect::box({0}, {2}), 100));
    write_job(job, good);
  }
  CHECK(run_command(good, out, {}) == 0);
  auto rows = read_results(out);
  CHECK(rows.size() == 2);
  CHECK(rows[0].mean == 7.0);
  CHECK(rows[1].mean == 10.0);
  CHECK(rows[0].trial_stddev == 0.0);
  CHECK(run_command(good, out, {std::nullopt, 3, std::nullopt}) == 0);
  CHECK(read_results(out)[0].trials == 3);
  const fs::path bad = dir / "bad_job.json";
  std::ofstream(bad) << R"({"seed":1,"trials":1,"integrands":[{"name":"a","expr":"x3",
       "dim":2,"low":[0,0],"high":[1,1],"samples":100}]})";
  CHECK(run_command(bad, out, {}) == 2);
  CHECK(run_command(dir / "missing_job.json", out, {}) == 2);
  const fs::path dead = dir / "dead_job.json";
  std::ofstream(dead) << R"j({"seed":1,"trials":2,"integrands":[{"name":"d","expr":"sqrt(-1-x1)",
       "dim":1,"low":[0],"high":[1],"samples":100}]})j";
  CHECK(run_command(dead, out, {}) == 3);
  // a tree job (ref tests/test_job_io.cpp:26-50 method round trip), run on the GPU
  const fs::path tree = dir / "tree_job.json";
  std::ofstream(tree) << R"j({"seed":31,"trials":2,"integrands":[{"name":"peak",
       "expr":"exp(-100*((x1-0.3)^2+(x2-0.3)^2))","dim":2,"low":[0,0],"high":[1,1],"samples":1200,
       "method":"tree","method_config":{"cells_per_dim":2,"samples_per_cell":256}}]})j";
  CHECK(run_command(tree, out, {}) == 0);
  auto trows = read_results(out);
  CHECK(trows.size() == 1 && trows[0].method == "tree" && trows[0].ok);
  CHECK(trows[0].warnings == "budget_exhausted");
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::string(argv[1]) == "gpu";
  dir = argc > 2 ? fs::path(argv[2]) : fs::temp_directory_path() / "mcb_job_io_test";
  fs::create_directories(dir);
  json_round_trip();
  strict_fields();
  csv_round_trip();
  fig1_generator_and_checker();
  if (gpu) run_command_exit_codes();
  std::printf("%d checks passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
