// mcbatch/sampling.hpp — source-compatible face of the reference header
// include/mcbatch/sampling.hpp (namespace mcbatch), over libmcb.
//
// Same names and meanings: kChunkSize, HyperRect, InvalidDomain, StreamKey,
// UniformStream, sample_uniform.  Draws and points are generated on the GPU
// (bit-exact with src/sampling.cpp:78-112): UniformStream fetches its draws
// from the device in batches (the fused kernels generate the same stream in
// registers).
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <vector>

#include "mcb/mcbatch.hpp"

namespace mcbatch {

inline constexpr std::size_t kChunkSize = mcb::kChunkSize;  // sampling.hpp:11

using mcb::HyperRect;      // sampling.hpp:14-24
using mcb::InvalidDomain;  // sampling.hpp:26-28
using mcb::StreamKey;      // sampling.hpp:33-44

// sampling.hpp:46-65: the Philox4x32-10 stream of unit doubles of one key,
// draw i = to_unit_double of block i/2 (words 0-1, then 2-3).  The
// constructor throws std::out_of_range for a chunk_index past 32 bits
// (src/sampling.cpp:79-81); draws come from the GPU (device 0), kBatch at a
// time, the same values in the same order as the reference's refill/next.
class UniformStream {
 public:
  explicit UniformStream(const StreamKey& key);

  double next() {
    if (pos_ == kBatch) refill();
    return buf_[pos_++];
  }

 private:
  static constexpr std::size_t kBatch = 4096;
  void refill();

  StreamKey key_;
  std::uint64_t drawn_ = 0;  // draws fetched so far
  std::size_t pos_ = kBatch;
  std::array<double, kBatch> buf_{};
};

// sampling.hpp:75-78: `count` points of rect's dimension, row-major.  The
// returning form is mcb's own (its trailing `device` defaults to 0), so that
// argument-dependent lookup on the shared HyperRect / StreamKey types finds
// one function, not two.
using mcb::sample_uniform;
inline void sample_uniform(const HyperRect& rect, const StreamKey& key, std::size_t count,
                           std::vector<double>& out) {
  out = mcb::sample_uniform(rect, key, count);
}

}  // namespace mcbatch
