// Pipe model of the fused direct-MC kernel's instruction mix on B200 (sm_100a).
//
// Each kernel runs 8 independent dependency chains per thread (256 threads,
// 148*8 CTAs) of one instruction class, or an interleaving of two classes, so
// the time is set by the pipe that executes them, not by latency or issue.
// Reported: warp-instructions per SMSP per clock -> cycles per warp
// instruction (the roofline denominators), at the SM clock given on the
// command line (read it from nvidia-smi while the box is loaded).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_micro pipe_micro.cu
//   ./pipe_micro [sm_mhz]
// Run under `ncu --metrics sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,
//   sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed,
//   sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,...` to see which
// pipe each class occupies.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

constexpr uint32_t kM0 = 0xD2511F53u;

// MODE: 0 WIDE (x = lo ^ hi of M*x: IMAD.WIDE.U32 + LOP3)
//       1 DFMA
//       2 WIDE:DFMA 1:1 (4 chains each)
//       3 WIDE:DFMA 2:1 (per step: 2 WIDE chains advanced twice, 2 DFMA once... see code)
//       4 I2F.F64.U64 (independent conversions, results folded with LOP3)
//       5 I2F.F64.S32
//       6 DADD
//       7 WIDE + I2F.F64.U64 1:1
//       8 DFMA + I2F.F64.U64 1:1
//       9 IMAD (lo) + DFMA 1:1
//      10 LOP3 only (x = x ^ (x >> 7) ^ it pattern)
template <int MODE>
__global__ void __launch_bounds__(256) k(uint64_t* out, int iters, double c) {
  uint32_t x[8];
  double y[8];
  uint64_t acc = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = threadIdx.x * 2654435761u + i * 977u + blockIdx.x;
    y[i] = double(x[i]) * 1e-9;
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const bool lo_half = i < 4;
      if (MODE == 0 || ((MODE == 2 || MODE == 7) && lo_half) || (MODE == 3 && i < 6)) {
        const uint64_t p = uint64_t(x[i]) * kM0;
        x[i] = uint32_t(p) ^ uint32_t(p >> 32);
      }
      if (MODE == 1 || ((MODE == 2 || MODE == 8 || MODE == 9) && !lo_half) || (MODE == 3 && i >= 6))
        y[i] = fma(y[i], c, 0.25);
      if (MODE == 4 || ((MODE == 7 || MODE == 8) && (MODE == 7 ? !lo_half : lo_half))) {
        double d;
        asm volatile("cvt.rn.f64.u64 %0, %1;" : "=d"(d) : "l"((uint64_t(x[i]) << 32) ^ uint64_t(it)));
        acc ^= uint64_t(__double_as_longlong(d));
        x[i] += 0x9E3779B9u;
      }
      if (MODE == 5) {
        double d;
        asm volatile("cvt.rn.f64.s32 %0, %1;" : "=d"(d) : "r"(int32_t(x[i] ^ uint32_t(it))));
        acc ^= uint64_t(__double_as_longlong(d));
        x[i] += 0x9E3779B9u;
      }
      if (MODE == 6) y[i] = y[i] + c;
      if (MODE == 9 && lo_half) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(kM0), "r"(it));
      if (MODE == 10) x[i] = x[i] ^ (x[i] >> 7) ^ uint32_t(it);
    }
  }
  double d = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    acc ^= x[i];
    d += y[i];
  }
  if (acc == 0x1234567ull || d == 1.5) out[blockIdx.x] = acc;
}

template <class K>
float timeit(K kern) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern();
  cudaEventRecord(a);
  kern();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main(int argc, char** argv) {
  const double mhz = argc > 1 ? atof(argv[1]) : 1965.0;
  uint64_t* d;
  cudaMalloc(&d, 1 << 20);
  const int ctas = 148 * 8, iters = 4000;
  // warp-instructions of the chain ops per SMSP
  const double warp_ops = double(ctas) * (256 / 32) * iters * 8 / (148.0 * 4);
  float t;
#define RUN(M, name)                                                                              \
  t = timeit([&] { k<M><<<ctas, 256>>>(d, iters, 0.999); });                                      \
  printf("%-34s %8.3f ms  %6.3f clk per chain warp-op per SMSP\n", name, t,                         \
         t * 1e-3 * mhz * 1e6 / warp_ops);
  RUN(0, "IMAD.WIDE (+LOP3)");
  RUN(1, "DFMA");
  RUN(6, "DADD");
  RUN(2, "IMAD.WIDE : DFMA 1:1");
  RUN(3, "IMAD.WIDE : DFMA 3:1");
  RUN(4, "I2F.F64.U64 (+LOP3/IADD)");
  RUN(5, "I2F.F64.S32 (+LOP3/IADD)");
  RUN(7, "IMAD.WIDE : I2F.F64.U64 1:1");
  RUN(8, "DFMA : I2F.F64.U64 1:1");
  RUN(9, "IMAD(lo) : DFMA 1:1");
  RUN(10, "LOP3/SHF only");
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
