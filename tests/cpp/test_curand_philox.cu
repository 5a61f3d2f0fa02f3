// The device Philox4x32-10 of the fused kernels (mcb_device.cuh: CTA prefix
// + philox_block_p with the round-1 product advanced by adds) against an
// independent implementation on the GPU: cuRAND's curand_Philox4x32_10
// (curand_philox4x32_x.h), SURVEY.md §8(c)(3).  Counter {b, 0, chunk, trial},
// random keys / chunks / trials, blocks from 0 and near 2^32.
#include <cuda_runtime.h>
#include <curand_philox4x32_x.h>

#include <cstdio>
#include <cstdint>
#include <random>
#include <vector>

#include "mcb_device.cuh"

struct Case {
  uint32_t key0, key1, chunk, trial, block;
};

__global__ void k_compare(const Case* cases, int n, uint32_t* bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Case c = cases[i];
  const mcb::dev::PhiloxPrefix P = mcb::dev::make_prefix(c.key0, c.key1, c.chunk, c.trial);
  uint32_t ours[4];
  mcb::dev::philox_block(P, c.block, ours);
  // consecutive-block form used by the kernels: p0 advanced by M0 per block
  uint32_t adv[4];
  mcb::dev::philox_block_p(P, uint64_t(mcb::dev::kM0) * uint64_t(c.block), adv);
  const uint4 r = curand_Philox4x32_10(make_uint4(c.block, 0u, c.chunk, c.trial), make_uint2(c.key0, c.key1));
  const bool ok = ours[0] == r.x && ours[1] == r.y && ours[2] == r.z && ours[3] == r.w && adv[0] == r.x &&
                  adv[1] == r.y && adv[2] == r.z && adv[3] == r.w;
  if (!ok) atomicAdd(bad, 1u);
}

int main() {
  std::mt19937_64 rng(2104);
  std::vector<Case> cases;
  for (int i = 0; i < 1 << 20; ++i) {
    Case c;
    c.key0 = uint32_t(rng());
    c.key1 = uint32_t(rng());
    c.chunk = (i & 3) ? uint32_t(rng() % 200) : uint32_t(rng());
    c.trial = (i & 7) ? uint32_t(rng() % 16) : uint32_t(rng());
    c.block = (i & 1) ? uint32_t(rng() % 300000) : uint32_t(0xFFFFFFFFu - rng() % 1000);
    cases.push_back(c);
  }
  Case* d_cases;
  uint32_t* d_bad;
  cudaMalloc(&d_cases, sizeof(Case) * cases.size());
  cudaMalloc(&d_bad, sizeof(uint32_t));
  cudaMemset(d_bad, 0, sizeof(uint32_t));
  cudaMemcpy(d_cases, cases.data(), sizeof(Case) * cases.size(), cudaMemcpyHostToDevice);
  k_compare<<<(int(cases.size()) + 255) / 256, 256>>>(d_cases, int(cases.size()), d_bad);
  uint32_t bad = 0;
  cudaError_t e = cudaMemcpy(&bad, d_bad, sizeof bad, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) {
    std::printf("CUDA error: %s\n", cudaGetErrorString(e));
    return 2;
  }
  std::printf("%zu Philox blocks vs curand_Philox4x32_10: %u mismatches\n", cases.size(), bad);
  return bad ? 1 : 0;
}
