// Host build of the device arithmetic (paper_2104_10073_b200/csrc/mcb_device.cuh,
// compiled with g++ -ffp-contract=off) checked against the C oracle
// (oracle/mcb_oracle.c, itself pinned to the reference).  Runs without a GPU.
//
//  1. philox_block(make_prefix(...)) == philox_block of the reference
//     (src/sampling.cpp:51-70) for random keys / counters, incl. chunk, trial > 0
//  2. u_scaled(hi, lo) * 2^-64 == to_unit_double(hi, lo) bit-exactly
//     (src/sampling.cpp:72-75)
//  3. the 2^-64 folding used by the FAST variants is bit-exact
//  4. the table-form sin/cos (the kernel's reduction): absolute error < 3 * 2^-53
//  5. a*cos t + b*sin t in table form: error < 2.5 * max(|a|,|b|) * 2^-52
//  6. trig_table.inc holds correctly rounded cos/sin of m*pi/256
//  7. the folded-shift form g = a*cos t + b*sin t - c (kFoldShift):
//     error < 3.5 * max(|a|,|b|,|c|) * 2^-52 per sample (a rounded f minus c:
//     ~2.4); the per-entry part, A_m - c, is correctly rounded, so the only
//     systematic error a Monte Carlo mean can pick up is <= 0.5 ulp
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>

#include "mcb_device.cuh"

extern "C" {
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double orc_to_unit_double(uint32_t hi, uint32_t lo);
}

using namespace mcb::dev;

static int g_fail = 0;
#define CHECK(cond, ...)                      \
  do {                                        \
    if (!(cond)) {                            \
      if (g_fail < 20) {                      \
        std::printf("FAIL %s:%d ", __FILE__, __LINE__); \
        std::printf(__VA_ARGS__);             \
        std::printf("\n");                    \
      }                                       \
      ++g_fail;                               \
    }                                         \
  } while (0)

static uint64_t bits(double x) {
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return b;
}

int main() {
  std::mt19937_64 rng(20200814);
  // 1. Philox with the CTA prefix
  for (int i = 0; i < 200000; ++i) {
    const uint32_t k0 = uint32_t(rng()), k1 = uint32_t(rng());
    const uint32_t chunk = (i & 3) ? uint32_t(rng()) : 0u, trial = (i & 1) ? uint32_t(rng()) : 0u;
    const uint32_t b = uint32_t(rng() % 300000);
    PhiloxPrefix P = make_prefix(k0, k1, chunk, trial);
    uint32_t got[4], want[4];
    philox_block(P, b, got);
    const uint32_t ctr[4] = {b, 0u, chunk, trial}, key[2] = {k0, k1};
    orc_philox4x32_10(ctr, key, want);
    CHECK(std::memcmp(got, want, 16) == 0, "philox k=%08x,%08x b=%u", k0, k1, b);
  }
  // 2. exact 53-bit conversion
  const uint32_t edge[] = {0u, 1u, 0x7FFu, 0x800u, 0x7FFFFFFFu, 0x80000000u, 0xFFFFF7FFu, 0xFFFFFFFFu};
  for (uint32_t hi : edge)
    for (uint32_t lo : edge)
      CHECK(bits(u_scaled(hi, lo) * kTwoM64) == bits(orc_to_unit_double(hi, lo)), "u53 %08x %08x", hi, lo);
  for (int i = 0; i < 1000000; ++i) {
    const uint32_t hi = uint32_t(rng()), lo = uint32_t(rng());
    CHECK(bits(u_scaled(hi, lo) * kTwoM64) == bits(orc_to_unit_double(hi, lo)), "u53 %08x %08x", hi, lo);
  }
  // 3. folding: RN(k' * ((v1+v2)+v3)) == RN(k * ((u1+u2)+u3)) with k' = k*2^-64,
  //    and low + w'*v == low + w*u
  for (int i = 0; i < 1000000; ++i) {
    double v[3], u[3];
    for (int j = 0; j < 3; ++j) {
      v[j] = u_scaled(uint32_t(rng()), uint32_t(rng()));
      u[j] = v[j] * kTwoM64;
    }
    const double k = std::ldexp(double(rng() >> 11) * 0x1p-53 + 0.5, int(rng() % 200) - 100);
    const double sv = (v[0] + v[1]) + v[2], su = (u[0] + u[1]) + u[2];
    CHECK(bits((k * kTwoM64) * sv) == bits(k * su), "fold k=%a", k);
    const double w = std::ldexp(1.0 + double(rng() >> 12) * 0x1p-52, int(rng() % 60) - 30);
    const double lo = double(int64_t(rng() % 2001) - 1000) * 0.37;
    CHECK(bits(lo + (w * kTwoM64) * v[0]) == bits(lo + w * u[0]), "fold w=%a", w);
  }
  // 4. table-form sin/cos accuracy (same reduction as the kernel)
  const TrigConsts K = MCB_TRIG_CONSTS;
  double max_s = 0, max_c = 0;
  for (int e = -3; e <= 19; ++e) {
    std::uniform_real_distribution<double> U(-std::ldexp(1.0, e), std::ldexp(1.0, e));
    for (int i = 0; i < 200000; ++i) {
      const double t = U(rng);
      double s, c;
      sincos_table(K, g_trig_host, t, s, c);
      max_s = std::fmax(max_s, double(std::fabs((long double)s - sinl((long double)t))) / 0x1p-53);
      max_c = std::fmax(max_c, double(std::fabs((long double)c - cosl((long double)t))) / 0x1p-53);
    }
  }
  // absolute error in units of 2^-53 (half an ulp of 1): what a Monte Carlo
  // mean sees; glibc's correctly rounded sin/cos are within 1 of these units
  std::printf("table sin/cos max abs error: sin %.3f, cos %.3f x 2^-53\n", max_s, max_c);
  CHECK(max_s < 3.0 && max_c < 3.0, "sincos accuracy sin %.3f cos %.3f", max_s, max_c);
  // 5. harmonic value a*cos t + b*sin t in table form vs correctly rounded,
  //    in units of the coefficient scale max(|a|,|b|) * 2^-52
  double max_h = 0, max_u = 0;
  for (int i = 0; i < 2000000; ++i) {
    const double t = std::uniform_real_distribution<double>(-700, 700)(rng);
    const double a = std::uniform_real_distribution<double>(-3, 3)(rng);
    const double b = std::uniform_real_distribution<double>(-3, 3)(rng);
    double r, s, c;
    uint32_t m;
    trig_reduce(K, t, r, m);
    trig_sc(K, r, s, c);
    const double h = trig_combine(trig_ab<false>(g_trig_host[m], a, b), s, c);
    const long double ex = (long double)a * cosl((long double)t) + (long double)b * sinl((long double)t);
    max_h = std::fmax(max_h, double(std::fabs((long double)h - ex)) / (std::fmax(std::fabs(a), std::fabs(b)) * 0x1p-52));
    const double u = trig_combine(trig_ab<true>(g_trig_host[m], 1.0, 1.0), s, c);
    const long double exu = cosl((long double)t) + sinl((long double)t);
    max_u = std::fmax(max_u, double(std::fabs((long double)u - exu)) / 0x1p-52);
  }
  std::printf("a cos t + b sin t: max error %.3f x max(|a|,|b|) 2^-52; unit form %.3f x 2^-52\n", max_h, max_u);
  CHECK(max_h < 2.5 && max_u < 2.0, "harmonic value accuracy %.3f %.3f", max_h, max_u);
  // 7. folded shift: g = A_m cm1(r) + (B_m sin r + (A_m - c)) against the exact
  //    a cos t + b sin t - c, c anywhere in the integrand's range
  double max_g = 0, max_gu = 0, max_sub = 0;
  for (int i = 0; i < 2000000; ++i) {
    const double t = std::uniform_real_distribution<double>(-700, 700)(rng);
    const double a = std::uniform_real_distribution<double>(-3, 3)(rng);
    const double b = std::uniform_real_distribution<double>(-3, 3)(rng);
    const double c = std::uniform_real_distribution<double>(-1, 1)(rng) * (std::fabs(a) + std::fabs(b));
    const double cu = std::uniform_real_distribution<double>(-1.5, 1.5)(rng);
    double r, s, cm1;
    uint32_t m;
    trig_reduce(K, t, r, m);
    trig_sc_m1(K, r, s, cm1);
    const TrigAB e = trig_ab<false>(g_trig_host[m], a, b);
    const double g = trig_combine_shifted(trig_abs_entry(g_trig_host[m], a, b, c, false), s, cm1);
    const long double ex =
        (long double)a * cosl((long double)t) + (long double)b * sinl((long double)t) - (long double)c;
    const double scale = std::fmax(std::fmax(std::fabs(a), std::fabs(b)), std::fabs(c));
    max_g = std::fmax(max_g, double(std::fabs((long double)g - ex)) / (scale * 0x1p-52));
    {  // the unfolded alternative: rounded f, then a rounded subtraction
      double s0, c0;
      trig_sc(K, r, s0, c0);
      const double sub = trig_combine(e, s0, c0) - c;
      max_sub = std::fmax(max_sub, double(std::fabs((long double)sub - ex)) / (scale * 0x1p-52));
    }
    const double gu = trig_combine_shifted(trig_abs_entry(g_trig_host[m], 1.0, 1.0, cu, true), s, cm1);
    const long double exu = cosl((long double)t) + sinl((long double)t) - (long double)cu;
    max_gu = std::fmax(max_gu, double(std::fabs((long double)gu - exu)) / (std::fmax(1.0, std::fabs(cu)) * 0x1p-52));
  }
  std::printf("folded shift a cos t + b sin t - c: max error %.3f x max(|a|,|b|,|c|) 2^-52 "
              "(unfolded f - c: %.3f); unit form %.3f\n", max_g, max_sub, max_gu);
  CHECK(max_g < 3.5 && max_gu < 3.5, "folded-shift accuracy %.3f %.3f (unfolded %.3f)",
        max_g, max_gu, max_sub);
  // constant integrand (t = 0 on the whole domain, c = f(0)): g is exactly 0
  {
    double r, s, cm1;
    uint32_t m;
    trig_reduce(K, 0.0, r, m);
    trig_sc_m1(K, r, s, cm1);
    const double c = 0.75 * g_trig_host[0].c + -1.25 * g_trig_host[0].s;  // a*cos 0 + b*sin 0
    CHECK(trig_combine_shifted(trig_abs_entry(g_trig_host[0], 0.75, -1.25, c, false), s, cm1) == 0.0,
          "folded constant");
    CHECK(trig_combine_shifted(trig_abs_entry(g_trig_host[0], 1.0, 1.0, 1.0, true), s, cm1) == 0.0,
          "folded constant, unit form");
  }
  // 6. the table itself: entries equal the correctly rounded cos/sin
  for (int mm = 0; mm < 512; ++mm) {
    const long double ang = (long double)mm * 3.14159265358979323846264338327950288L / 256.0L;
    CHECK(std::fabs((long double)g_trig_host[mm].c - cosl(ang)) <= 0x1p-53, "table c %d", mm);
    CHECK(std::fabs((long double)g_trig_host[mm].s - sinl(ang)) <= 0x1p-53, "table s %d", mm);
  }
  std::printf("%s (%d failures)\n", g_fail ? "FAILED" : "OK", g_fail);
  return g_fail ? 1 : 0;
}
