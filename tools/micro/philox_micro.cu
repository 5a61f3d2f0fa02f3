// Microbenchmark: Philox4x32-10 throughput with round keys in uniform
// registers (kernel parameter) vs vector registers (global load), and the
// FP64 sincos_core throughput.  Run: nvcc -gencode arch=compute_100a,code=sm_100a -O3 ...
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "mcb_device.cuh"
using namespace mcb::dev;

template <bool UKEY>
__global__ void __launch_bounds__(256) k_philox(const uint32_t* gkey, uint32_t pkey0, uint32_t pkey1,
                                                uint32_t* out, int iters) {
  uint32_t k0 = UKEY ? pkey0 : gkey[0], k1 = UKEY ? pkey1 : gkey[1];
  const PhiloxPrefix P = make_prefix(k0, k1, blockIdx.x & 15, blockIdx.x >> 4);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t b = (it * 256 + threadIdx.x) * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t o[4];
      philox_block(P, b + i, o);
      acc ^= o[0] ^ o[1] ^ o[2] ^ o[3];
    }
  }
  if (acc == 0x1234567u) out[blockIdx.x] = acc;
}

__constant__ SinCosConsts KC = MCB_SINCOS_CONSTS;
__global__ void __launch_bounds__(256) k_sincos(double* out, int iters, double k) {
  double acc = 0.0;
  double t = k * (threadIdx.x + 1);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double s, c;
      uint32_t q;
      sincos_core(KC, t + i * 0.37, s, c, q);
      acc += s + c + double(q & 3);
    }
    t += 0.001;
  }
  if (acc == 1.2345) out[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(256) k_mixed(uint32_t* out, int iters, double k, uint32_t k0, uint32_t k1) {
  const PhiloxPrefix P = make_prefix(k0, k1, blockIdx.x & 15, blockIdx.x >> 4);
  uint32_t acc = 0;
  double dacc = 0.0;
  double t = k * (threadIdx.x + 1);
  for (int it = 0; it < iters; ++it) {
    const uint32_t b = (it * 256 + threadIdx.x) * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      uint32_t o[4];
      philox_block(P, b + i, o);
      acc ^= o[0] ^ o[1] ^ o[2] ^ o[3];
      double s, c;
      uint32_t q;
      sincos_core(KC, t + i * 0.37, s, c, q);
      dacc += s + c + double(q & 3);
    }
    t += 0.001;
  }
  if (acc == 0x1234567u || dacc == 1.2345) out[blockIdx.x] = acc;
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 1 << 20);
  cudaMemset(d, 0x5a, 1 << 20);
  double* dd;
  cudaMalloc(&dd, 1 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int ctas = 148 * 8, iters = 2000;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a);
    k_philox<true><<<ctas, 256>>>(d, 0x37ba30ca, 0xccc782d2, d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double blocks = double(ctas) * 256 * iters * 4;
    printf("philox UR keys : %.3f ms  %.3e blocks/s  %.2f blocks/clk/SM @1965\n", ms, blocks / ms * 1e3,
           blocks / (ms * 1e-3) / (148 * 1.965e9));
    cudaEventRecord(a);
    k_philox<false><<<ctas, 256>>>(d, 0, 0, d, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("philox VR keys : %.3f ms  %.3e blocks/s  %.2f blocks/clk/SM @1965\n", ms, blocks / ms * 1e3,
           blocks / (ms * 1e-3) / (148 * 1.965e9));
    cudaEventRecord(a);
    k_sincos<<<ctas, 256>>>(dd, iters, 0.01);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double sc = double(ctas) * 256 * iters * 4;
    printf("sincos_core    : %.3f ms  %.3e /s  %.3f per clk/SM @1965\n", ms, sc / ms * 1e3,
           sc / (ms * 1e-3) / (148 * 1.965e9));
  }
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(a);
    k_mixed<<<ctas, 256>>>(d, iters, 0.01, 0x37ba30ca, 0xccc782d2);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("mixed 4 philox + 4 sincos: %.3f ms\n", ms);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
