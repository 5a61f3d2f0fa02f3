// jit.hpp — runtime specialisation of DSL programs (MCB_FAMILY_PROGRAM).
//
// A compiled program (program.hpp) is emitted as straight-line CUDA
// (prog::emit_cuda), compiled by NVRTC for sm_100a together with the
// jit_kernels.cuh templates (their text and the headers they need are
// embedded in libmcb.so at build time), loaded into the current device's
// primary context and launched instead of the bytecode interpreter.  Results
// are bit-identical to the interpreter's (same operations, same sample order
// and reduction shape).  Modules are cached per (device, program source).
// When NVRTC cannot be loaded or a compile fails, the interpreter kernels
// run instead — both are the sm_100a GPU path; there is no CPU path.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace mcb {
namespace prog {
struct Program;
}
namespace dev {
struct FnDesc;
struct TilePartial;
}
namespace jit {

// Process-wide mode: 0 off (bytecode interpreter), 1 automatic (default:
// specialised kernels for programs whose cubin is cached — in memory or on
// disk — or that a plan will reuse, or whose launch is large enough to repay
// its ~0.3 s compile; the interpreter otherwise), 2 always (compile before the
// first launch).  MCB_PROGRAM_JIT=0 / =always select 0 / 2; set_mode()
// overrides.  enabled() / mode() report 0 when NVRTC is unavailable.  No
// background threads: every compile completes inside the call that needs it.
bool enabled();
int mode();
void set_mode(int m);
void set_enabled(bool on);
// Why the last compile or the NVRTC load failed ("" if none).
std::string last_error();

// Launch the specialised kernel of `p` in kernel mode `mode` (0 direct, 1
// direct on the unit cube, 2 cells CTA-per-tile, 3 small cells
// warp-per-tile, 4 small cells of a large grid thread-per-cell) over `ctas`
// CTAs of 128 threads starting at tile `tile0`;
// `samples` (the launch's work) decides whether the automatic mode compiles
// an uncached program.  Returns false (nothing launched) when the caller
// should run the interpreter.
bool launch(const prog::Program& p, int mode, uint32_t ctas, uint64_t samples, const dev::FnDesc* fns,
            const uint32_t* tile_fn, uint64_t tile0, dev::TilePartial* part, cudaStream_t s, cudaError_t* err);

// Ahead of launches, for (program, kernel mode) pairs: look the kernels up in
// the disk cache and, with
// `compile` (a plan that will be relaunched) or in mode 2, compile the
// missing ones in parallel.
void prepare(const std::vector<std::pair<const prog::Program*, int>>& kernels, bool compile);

// NVRTC-compile `p`'s five kernel modes (or find them in the disk cache)
// without a device: warms the on-disk cache ahead of time and checks the
// generated code.
bool compile_only(const prog::Program& p, std::string* err);

// Number of NVRTC compilations performed so far (tests / tracing).
uint64_t compile_count();

}  // namespace jit
}  // namespace mcb
