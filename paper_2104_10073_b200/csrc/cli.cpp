// cli.cpp — `mcb`, the command-line front end on the GPU backend, with the
// reference CLI's subcommands, options and exit codes (ref tools/mcbatch.cpp):
//
//   mcb run <job.json> [--out results.csv] [--seed S] [--trials R] [--workers W]
//   mcb gen-fig1 [--n 100] [--samples 1000000] --out job.json
//   mcb check-fig1 <results.csv> [--plot-out plot.csv]
//   mcb validate <job.json>
//
// --workers (env MCBATCH_WORKERS) is the number of GPUs (0 = all visible).
#include <cstdint>
#include <cstdlib>
#include <iostream>
#include <optional>
#include <string>
#include <vector>

#include "mcb/job_io.hpp"
#include "mcb/mcbatch.hpp"

namespace {

int usage() {
  std::cerr << "mcb - batched Monte Carlo integration of many integrands (B200 backend)\n"
               "usage:\n"
               "  mcb run <job> [--out F] [--seed S] [--trials R] [--workers W]\n"
               "  mcb gen-fig1 [--n N] [--samples S] --out F\n"
               "  mcb check-fig1 <results> [--plot-out F]\n"
               "  mcb validate <job>\n";
  return 2;
}

template <class T>
bool parse_uint(const std::string& s, T& out) {
  if (s.empty()) return false;
  char* end = nullptr;
  const unsigned long long v = std::strtoull(s.c_str(), &end, 10);
  if (*end != '\0') return false;
  out = T(v);
  return true;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) return usage();
  const std::string cmd = argv[1];
  std::vector<std::string> pos;
  std::vector<std::pair<std::string, std::string>> opts;
  for (int i = 2; i < argc; ++i) {
    const std::string a = argv[i];
    if (a.rfind("--", 0) == 0) {
      if (i + 1 >= argc) {
        std::cerr << "error: " << a << " needs a value\n";
        return 2;
      }
      opts.emplace_back(a, argv[++i]);
    } else {
      pos.push_back(a);
    }
  }
  auto opt = [&](const char* name) -> std::optional<std::string> {
    for (const auto& [k, v] : opts)
      if (k == name) return v;
    return std::nullopt;
  };
  auto known = [&](std::initializer_list<const char*> names) {
    for (const auto& [k, v] : opts) {
      bool ok = false;
      for (const char* n : names) ok = ok || k == n;
      if (!ok) {
        std::cerr << "error: unknown option " << k << "\n";
        return false;
      }
    }
    return true;
  };

  if (cmd == "run") {
    if (pos.size() != 1 || !known({"--out", "--seed", "--trials", "--workers"})) return usage();
    mcb::RunOverrides ov;
    uint64_t u64;
    uint32_t u32;
    if (auto s = opt("--seed")) {
      if (!parse_uint(*s, u64)) return usage();
      ov.seed = u64;
    }
    if (auto s = opt("--trials")) {
      if (!parse_uint(*s, u32)) return usage();
      ov.trials = u32;
    }
    std::optional<std::string> w = opt("--workers");
    if (!w) {
      if (const char* env = std::getenv("MCBATCH_WORKERS")) w = std::string(env);
    }
    if (w) {
      if (!parse_uint(*w, u32)) return usage();
      ov.workers = u32;
    }
    return mcb::run_command(pos[0], opt("--out").value_or("results.csv"), ov);
  }
  if (cmd == "gen-fig1") {
    if (!pos.empty() || !known({"--n", "--samples", "--out"}) || !opt("--out")) return usage();
    uint32_t n = 100;
    uint64_t samples = 1000000;
    if (auto s = opt("--n"); s && !parse_uint(*s, n)) return usage();
    if (auto s = opt("--samples"); s && !parse_uint(*s, samples)) return usage();
    try {
      return mcb::gen_fig1(n, samples, *opt("--out"));
    } catch (const std::exception& e) {
      std::cerr << "error: " << e.what() << "\n";
      return 3;
    }
  }
  if (cmd == "check-fig1") {
    if (pos.size() != 1 || !known({"--plot-out"})) return usage();
    std::optional<std::filesystem::path> plot;
    if (auto s = opt("--plot-out")) plot = *s;
    return mcb::check_fig1_command(pos[0], plot);
  }
  if (cmd == "validate") {
    if (pos.size() != 1 || !opts.empty()) return usage();
    try {
      const mcb::JobSpec job = mcb::read_job(pos[0]);
      const auto violations = mcb::validate(job);
      if (violations.empty()) {
        std::cout << "ok: " << job.integrands.size() << " integrand(s)\n";
        return 0;
      }
      for (const auto& v : violations)
        std::cerr << (v.integrand.empty() ? std::string("job") : v.integrand) << ": " << v.message << "\n";
      return 2;
    } catch (const std::exception& e) {
      std::cerr << "error: " << e.what() << "\n";
      return 2;
    }
  }
  return usage();
}
