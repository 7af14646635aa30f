// trb_common.cuh — shared definitions for the sm_100a kernels and the host
// engine of the B200-native front end.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "../../include/trb.h"

namespace trb {

// Error carrying a trb_status; the C ABI converts it to a return code and
// trb_last_error() text.  Messages reuse the reference's wording.
struct Error : std::runtime_error {
  trb_status code;
  Error(trb_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorMemoryAllocation) throw Error(TRB_OUT_OF_MEMORY, std::string(what) + ": " + cudaGetErrorString(e));
    throw Error(TRB_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define TRB_CUDA(x) ::trb::cuda_check((x), #x)
#define TRB_LAUNCH_CHECK(name) ::trb::cuda_check(cudaGetLastError(), name)

// Programmatic dependent launch: a kernel launched with launch_pdl may start
// while the previous kernel on the stream drains; it must call pdl_wait()
// before touching memory that kernel reads or writes (the wait returns once
// the previous grid has completed and its writes are visible).  Saves the
// launch gap between the short kernels of a frame (CCL chain, tracker chain).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, kern, args...), "cudaLaunchKernelEx (programmatic dependent launch)");
}

// Tile geometry of the connected-component kernels: a CTA owns a 32x32
// pixel tile; a tile holds at most 512 components (4-connected
// checkerboard), which bounds the per-stream slot table at px/2.
constexpr int kTileW = 32;
constexpr int kTileH = 32;
constexpr int kTilePx = kTileW * kTileH;
constexpr int kMaxTileComps = kTilePx / 2;

inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
inline int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Exact unsigned division n / d for n < 2^28, d < 2^12 by one 64-bit
// multiply: q = (n * M) >> 40 with M = ceil(2^40 / d).  Used for the Mean
// background (2*sum + W) / (2W) (motion.hpp:185).
struct FastDiv {
  uint64_t m;
  static FastDiv make(uint32_t d) { return FastDiv{((1ull << 40) + d - 1) / d}; }
  __host__ __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return static_cast<uint32_t>((static_cast<uint64_t>(n) * m) >> 40);
  }
};

}  // namespace trb
