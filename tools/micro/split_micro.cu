// Can Philox's 32x32->64 multiplies leave the FP64 pipe?  IMAD.WIDE runs on
// the FP64 pipe on B200; IMAD.HI + IMAD (lo) may not.  Compare Philox-only and
// Philox+sincos throughput with (a) IMAD.WIDE, (b) IMAD.HI + IMAD, (c) a mix.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "mcb_device.cuh"
using namespace mcb::dev;

__device__ __forceinline__ void mul_split(uint32_t a, uint32_t b, uint32_t zero, uint32_t& hi, uint32_t& lo) {
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(a), "r"(b));
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(lo) : "r"(a), "r"(b), "r"(zero));
}

// MODE bit i (0..15): multiply #i of the 16 in rounds 3..10 is split.
template <uint32_t MASK>
__device__ __forceinline__ void philox_p(const PhiloxPrefix& P, uint64_t p0, uint32_t zero, uint32_t out[4]) {
  uint32_t hi0 = uint32_t(p0 >> 32), lo0 = uint32_t(p0), hi1, lo1;
  uint32_t c0 = P.r1_c0, c1 = P.r1_c1, c2 = hi0 ^ P.r1_x2, c3 = lo0;
  if (MASK & 0x10000u) mul_split(kM1, c2, zero, hi1, lo1); else mulhilo(kM1, c2, hi1, lo1);
  c0 = hi1 ^ P.r2_x0; c1 = lo1; c2 = c3 ^ P.r2_x2; c3 = P.r2_c3;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    if (MASK & (1u << (2 * r))) mul_split(kM0, c0, zero, hi0, lo0); else mulhilo(kM0, c0, hi0, lo0);
    if (MASK & (1u << (2 * r + 1))) mul_split(kM1, c2, zero, hi1, lo1); else mulhilo(kM1, c2, hi1, lo1);
    c0 = hi1 ^ c1 ^ P.k0[r]; c1 = lo1; c2 = hi0 ^ c3 ^ P.k1[r]; c3 = lo0;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

__constant__ TrigConsts KC = MCB_TRIG_CONSTS;

template <uint32_t MASK, bool TRIG>
__global__ void __launch_bounds__(256) k(const uint32_t* key, uint32_t* out, int iters) {
  const uint32_t zero = key[2];
  const PhiloxPrefix P = make_prefix(key[0], key[1], blockIdx.x & 15, blockIdx.x >> 4);
  uint64_t pb = uint64_t(kM0) * (threadIdx.x * 4u);
  uint32_t acc = 0;
  double dacc = 0.0;
  double t = 0.01 * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t o[4];
      philox_p<MASK>(P, pb + uint64_t(i) * kM0, zero, o);
      acc ^= o[0] ^ o[1] ^ o[2] ^ o[3];
      if (TRIG && (i & 1)) {  // one 14-op harmonic evaluation per 2 blocks (a 4-D sample)
        double r, s, c;
        uint32_t m;
        trig_reduce(KC, t + double(o[0] & 0xFFFF) * 1e-3, r, m);
        trig_sc(KC, r, s, c);
        dacc = fma(dacc, 0.5, fma(s, 0.3, c));
      }
    }
    pb += uint64_t(kM0) * 1024u;
  }
  if (acc == 0x1234567u || dacc == 1.2345) out[blockIdx.x] = acc;
}

template <class K>
float timeit(K kern) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  kern();
  cudaEventRecord(a); kern(); cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 1 << 20);
  uint32_t key[3] = {0x37ba30ca, 0xccc782d2, 0};
  cudaMemcpy(d, key, 12, cudaMemcpyHostToDevice);
  const int ctas = 148 * 8, iters = 1500;
  const double blocks = double(ctas) * 256 * iters * 4;
#define RUN(M, T, name) { float t = timeit([&] { k<M, T><<<ctas, 256>>>(d, d + 16, iters); }); \
  printf("%-34s %.3f ms  %.3f blocks/clk/SM\n", name, t, blocks / (t * 1e-3) / (148 * 1.965e9)); }
  RUN(0x00000u, false, "philox  WIDE x17");
  RUN(0x1FFFFu, false, "philox  HI+LO x17");
  RUN(0x05555u, false, "philox  8 split (M0 side)");
  RUN(0x0AAAAu, false, "philox  8 split (M1 side)");
  RUN(0x1AAAAu, false, "philox  9 split (M1 side + r2)");
  RUN(0x00000u, true, "ph+trig WIDE x17");
  RUN(0x1FFFFu, true, "ph+trig HI+LO x17");
  RUN(0x05555u, true, "ph+trig 8 split (M0 side)");
  RUN(0x0AAAAu, true, "ph+trig 8 split (M1 side)");
  RUN(0x1AAAAu, true, "ph+trig 9 split");
  RUN(0x03333u, true, "ph+trig 8 split (pairs)");
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
