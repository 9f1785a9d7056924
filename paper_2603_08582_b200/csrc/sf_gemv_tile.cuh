// sf_gemv_tile.cuh -- row/column partials of one 128x128 tile of the packed
// symmetric store; shared by the streaming matvec kernels (sf_fista.cu) and the
// on-chip FISTA kernel (sf_fista_chip.cu) so both sum in the same order.
#pragma once

#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {

// kBar = 0: __syncthreads(); kBar > 0: named barrier kBar over the 256 threads
// of the calling group (warps 8(kBar-1) .. 8(kBar-1)+7, or the TMA consumers)
template <int kBar>
__device__ __forceinline__ void gemv_bar() {
  if (kBar > 0) asm volatile("bar.sync %0, 256;\n" ::"n"(kBar) : "memory");
  else __syncthreads();
}

// Row and column partials of one tile whose 128x128 elements are already in
// registers (a[s4][i] = tile float4 (warp + 8 s4) * 128 + lane + 32 i).
template <int kBar>
__device__ __forceinline__ void gemv_tile_compute(const float4 (&a)[4][4], int I, int J,
                                                  const float *__restrict__ z32,
                                                  float *__restrict__ P, int nt, int sym,
                                                  float (*s_row)[kTile], float *s_col) {
  const int gt = threadIdx.x & 255;  // thread within the 256-thread group
  const int lane = gt & 31, warp = gt >> 5;
  {
    float zr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) zr[i] = __ldcg(z32 + (int64_t)I * kTile + lane + 32 * i);
    float4 zc[4];
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4)
      zc[s4] = __ldcg(reinterpret_cast<const float4 *>(z32 + (int64_t)J * kTile) + warp + 8 * s4);

    float rp[4];
    float cp[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) rp[i] = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) cp[k] = 0.f;
    const bool diag_sym = sym && (I == J);
    if (diag_sym) {
      // keep c >= r for the row partial, c > r for the column partial
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = lane + 32 * i, c0 = 4 * (warp + 8 * s4);
          float4 v = a[s4][i];
          v.x = (c0 + 0 >= row) ? v.x : 0.f;
          v.y = (c0 + 1 >= row) ? v.y : 0.f;
          v.z = (c0 + 2 >= row) ? v.z : 0.f;
          v.w = (c0 + 3 >= row) ? v.w : 0.f;
          rp[i] += v.x * zc[s4].x + v.y * zc[s4].y + v.z * zc[s4].z + v.w * zc[s4].w;
          cp[4 * s4 + 0] += (c0 + 0 > row) ? v.x * zr[i] : 0.f;
          cp[4 * s4 + 1] += (c0 + 1 > row) ? v.y * zr[i] : 0.f;
          cp[4 * s4 + 2] += (c0 + 2 > row) ? v.z * zr[i] : 0.f;
          cp[4 * s4 + 3] += (c0 + 3 > row) ? v.w * zr[i] : 0.f;
        }
      }
    } else {
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 v = a[s4][i];
          rp[i] += v.x * zc[s4].x + v.y * zc[s4].y + v.z * zc[s4].z + v.w * zc[s4].w;
          cp[4 * s4 + 0] += v.x * zr[i];
          cp[4 * s4 + 1] += v.y * zr[i];
          cp[4 * s4 + 2] += v.z * zr[i];
          cp[4 * s4 + 3] += v.w * zr[i];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) s_row[warp][lane + 32 * i] = rp[i];

    const bool do_col = sym;
    if (do_col) {
      // butterfly reduce-scatter of 16 column partials over the 32 lanes
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const bool hi = lane & 16;
        const float send = hi ? cp[k] : cp[k + 8];
        const float keep = hi ? cp[k + 8] : cp[k];
        cp[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool hi = lane & 8;
        const float send = hi ? cp[k] : cp[k + 4];
        const float keep = hi ? cp[k + 4] : cp[k];
        cp[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const bool hi = lane & 4;
        const float send = hi ? cp[k] : cp[k + 2];
        const float keep = hi ? cp[k + 2] : cp[k];
        cp[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
      }
      {
        const bool hi = lane & 2;
        const float send = hi ? cp[0] : cp[1];
        const float keep = hi ? cp[1] : cp[0];
        cp[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
      }
      cp[0] += __shfl_xor_sync(0xffffffffu, cp[0], 1);
      if ((lane & 1) == 0) {
        const int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 +
                        ((lane >> 1) & 1);
        const int col = 4 * (warp + 8 * (idx >> 2)) + (idx & 3);
        if (diag_sym) s_col[col] = cp[0];
        else P[((int64_t)J * nt + I) * kTile + col] = cp[0];
      }
    }
    gemv_bar<kBar>();
    if (gt < kTile) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += s_row[w][gt];
      if (diag_sym) s += s_col[gt];
      P[((int64_t)I * nt + J) * kTile + gt] = s;
    }
    gemv_bar<kBar>();
  }
}

}  // namespace sf
