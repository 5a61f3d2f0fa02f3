// The per-chunk layer of the reference's estimator API (include/mcbatch/
// estimator.hpp:59-78, sampling.hpp:46-65) through this repo's source-
// compatible headers, written as a reference user would.  Prints hex values
// that tests/test_chunks.py compares with the oracle.
#include <cmath>
#include <cstdio>
#include <string>
#include <vector>

#include "mcbatch/estimator.hpp"
#include "mcbatch/expr.hpp"
#include "mcbatch/sampling.hpp"

using namespace mcbatch;

int main() {
  // draws of one key, and the host Welford over them
  UniformStream s(StreamKey{123456789, 7, 3, 11});
  ChunkAccum w;
  std::printf("draws");
  for (int i = 0; i < 10000; ++i) {
    const double x = s.next();
    std::printf(" %a", x);
    w.add(x);
  }
  std::printf("\nwelford %llu %llu %a %a\n", (unsigned long long)w.n, (unsigned long long)w.n_nonfinite, w.mean,
              w.m2);

  // one chunk of a program on the GPU
  const std::vector<std::string> none;
  const CompiledProgram p = compile(parse("abs(x1+x2-x3)"), 3, none);
  const HyperRect unit = HyperRect::unit(3);
  const ChunkAccum c = accumulate_chunk(p, {}, unit, StreamKey{5, 2, 1, 4}, 30000);
  std::printf("chunk %llu %llu %a %a\n", (unsigned long long)c.n, (unsigned long long)c.n_nonfinite, c.mean, c.m2);

  // direct_mc decomposed into its chunks (src/estimator.cpp:75-92) and reduced
  const std::vector<std::string> names{"k"};
  const CompiledProgram h = compile(parse("cos(k*(x1+x2)) + sin(k*(x1+x2))"), 2, names);
  const std::vector<double> k{4.0};
  const HyperRect box = HyperRect::box({0.0, -1.0}, {1.0, 0.5});
  const std::uint64_t n = 150000;
  const StreamKey base{42, 9, 2, 100};
  std::vector<ChunkAccum> parts;
  for (std::uint64_t i = 0; i < chunk_count(n); ++i) {
    const std::size_t cnt = std::size_t(std::min<std::uint64_t>(kChunkSize, n - i * kChunkSize));
    parts.push_back(accumulate_chunk(h, k, box, base.with_chunk(base.chunk_index + i), cnt));
  }
  const McEstimate r = reduce_chunks(box.volume(), parts);
  const McEstimate d = direct_mc(h, k, box, n, base);
  const bool ok = r.n_samples == d.n_samples && std::fabs(r.value - d.value) <= 1e-12 * std::fabs(d.value) + 1e-15 &&
                  std::fabs(r.std_error - d.std_error) <= 1e-9 * d.std_error;
  std::printf("reduce %s %a %a %a %a\n", ok ? "ok" : "MISMATCH", r.value, d.value, r.std_error, d.std_error);

  // the reference's error behaviour
  bool threw = false;
  try {
    UniformStream bad(StreamKey{1, 0, 0, 0x100000000ull});
  } catch (const std::out_of_range&) {
    threw = true;
  }
  std::vector<ChunkAccum> dead(2);
  dead[0].add(NAN);
  try {
    (void)reduce_chunks(1.0, dead);
    threw = false;
  } catch (const AllSamplesNonFinite&) {
  }
  return ok && threw ? 0 : 1;
}
