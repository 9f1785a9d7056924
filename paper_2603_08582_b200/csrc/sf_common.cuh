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

// cudaFuncSetAttribute applies to the context of the current device only, so
// every call site that opts a kernel into more shared memory keeps one flag
// bit per device ordinal.
inline bool attr_pending(const std::atomic<uint64_t> &done) {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) return true;
  return !(done.load(std::memory_order_acquire) & (1ull << (d & 63)));
}
inline void attr_done(std::atomic<uint64_t> &done) {
  int d = 0;
  if (cudaGetDevice(&d) == cudaSuccess) done.fetch_or(1ull << (d & 63), std::memory_order_release);
}

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

// SF_DEBUG_SYNC=1: synchronise after every launch and name the failing site
// (never while this thread captures a CUDA graph)
bool debug_sync();
void set_capturing(bool on);
#define SF_LAUNCH_CHECK()                                                     \
  do {                                                                        \
    ::sf::count_launch();                                                     \
    cudaError_t _e = cudaGetLastError();                                      \
    if (_e == cudaSuccess && ::sf::debug_sync()) _e = cudaDeviceSynchronize(); \
    if (_e != cudaSuccess)                                                    \
      return ::sf::fail(SF_ECUDA, std::string("kernel launch (") + __FILE__ + \
                                      ":" + std::to_string(__LINE__) + "): " + \
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


// mbarrier + bulk-copy (TMA, non-tensor) helpers for the streaming kernels.
namespace bulk {
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// global -> shared bulk copy completing `bytes` of transaction on `bar`;
// evict_first: the streamed data is not re-read within the launch
__device__ __forceinline__ void g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar,
                                    uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
}  // namespace bulk

}  // namespace sf
