// sf_common.cuh -- shared definitions for the sm_100a Online-FISTA engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include "sarfista_b200.h"

namespace sf {

// Edge of one stored square tile of Re(A).  Tiles are 128x128 fp32 so one
// tile is exactly one tcgen05 M=128,N=128 accumulator (128 TMEM lanes x 128
// columns) and 64 KiB of HBM.
constexpr int kTile = 128;
constexpr int kTileElems = kTile * kTile;

// Gram K-dimension granule: the packed operator rows [Re G | Im G] are padded
// to a multiple of this many values (one pipeline stage of the f16x3 Gram
// kernel: 32 fp16 = 4 UMMA core matrices along K).
constexpr int kKChunk = 32;

constexpr double kSpeedOfLight = 299792458.0;  // geometry.py:11

// Thread-local error channel of the C ABI.
void set_error(const std::string &msg);
sf_status fail(sf_status st, const std::string &msg);

extern std::atomic<int64_t> g_launches;
inline void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

#define SF_CUDA_TRY(expr)                                                     \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      return ::sf::fail(_e == cudaErrorMemoryAllocation ? SF_ENOMEM           \
                                                        : SF_ECUDA,           \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));  \
    }                                                                         \
  } while (0)

#define SF_LAUNCH_CHECK()                                                     \
  do {                                                                        \
    ::sf::count_launch();                                                     \
    cudaError_t _e = cudaGetLastError();                                      \
    if (_e != cudaSuccess)                                                    \
      return ::sf::fail(SF_ECUDA, std::string("kernel launch: ") +            \
                                      cudaGetErrorString(_e));                \
  } while (0)

// Element (r, c) of one tile inside its 16384-float block.
// Layout [c/4][r][c%4]: a float4 "slab" holds 4 adjacent columns of one row,
// and the 128 rows of a slab are contiguous (2 KiB).  A warp reading 32
// consecutive rows of one slab issues a fully coalesced 512-byte request, and
// the tcgen05 epilogue (thread = TMEM lane = row) writes the same pattern.
__host__ __device__ inline int64_t tile_offset(int r, int c) {
  return (int64_t)(c >> 2) * (kTile * 4) + (int64_t)r * 4 + (c & 3);
}

// Programmatic dependent launch (PDL): kernels of the FISTA chain let the next
// kernel start launching at once (griddepcontrol.launch_dependents) and wait for
// their producer's completion and memory (griddepcontrol.wait) before reading
// it, hiding the ~4 us launch gap between dependent kernels.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace sf
