// mcbatch/sampling.hpp — source-compatible face of the reference header
// include/mcbatch/sampling.hpp (namespace mcbatch), over libmcb.
//
// Same names and meanings: kChunkSize, HyperRect, InvalidDomain, StreamKey,
// sample_uniform.  Points are generated on the GPU (sample_uniform of
// src/sampling.cpp:102-112, bit-exact).  Not provided: the host-side
// UniformStream class — the fused kernels generate the stream in registers;
// mcb_debug_points / sample_uniform expose it.
#pragma once

#include <cstddef>
#include <vector>

#include "mcb/mcbatch.hpp"

namespace mcbatch {

inline constexpr std::size_t kChunkSize = mcb::kChunkSize;  // sampling.hpp:11

using mcb::HyperRect;      // sampling.hpp:14-24
using mcb::InvalidDomain;  // sampling.hpp:26-28
using mcb::StreamKey;      // sampling.hpp:33-44

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
