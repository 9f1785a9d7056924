// sf_fista.cu -- the warm-started FISTA inner loop on the packed symmetric Re(A).
//
// Reference: solver.py:209-226 (online_fista_pulse) and kernels.py:78-103
// (_fista_inner_jit).  Per step:
//   g = Re(A) z - Re(b);  u = z - tau g;  c = sign(u) max(|u| - thresh, 0)
//   t' = (1 + sqrt(1 + 4 t^2)) / 2;  z = c + ((t - 1)/t') (c - c_prev)
//
// Re(A) is read from HBM once per step.  With the upper-triangle tile store
// each tile (I,J), I < J, contributes to two blocks of y = Re(A) z:
//   y_I += A_IJ z_J  (row partial)   and   y_J += A_IJ^T z_I  (column partial),
// so the step streams M^2/2 floats instead of M^2.  Partials go to a slot array
// P[block][contributor][128]; k_fista_step sums each block's nt slots in a
// fixed order (bitwise run-to-run reproducible, no float atomics), then applies
// the shrink + momentum update in fp64.
#include <cooperative_groups.h>
#include <float.h>
#include <stdlib.h>

#include <string>

#include "sf_common.cuh"
#include "sf_kernels.cuh"
#include "sf_gemv_tile.cuh"

namespace sf {

// max_j |b_j| (numpy abs of complex = hypot) as ordered fp64 bits; the
// per-pulse value is produced by k_compose, this kernel recomputes it after a
// state restore.
__global__ void __launch_bounds__(1024)
k_bmax(const double2 *__restrict__ b, int64_t m_atoms, unsigned long long *__restrict__ bmax) {
  __shared__ double red[32];
  double mx = 0.0;
  for (int64_t i = threadIdx.x; i < m_atoms; i += blockDim.x) {
    const double2 v = b[i];
    mx = fmax(mx, hypot(v.x, v.y));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (threadIdx.x == 0) *bmax = (unsigned long long)__double_as_longlong(mx);
  }
}

// tau = 1/L (solver.py:220); lambda = lam or lam_rel * max_j |b_j| (device
// side lambda rule); thresh = lambda * tau (solver.py:225).
// With wv != nullptr also the momentum weights of `steps` steps from t0
// (kernels.py:87-88), rounded exactly like the host's sf_fista loop so the
// returned t and the device weights agree: w_k = (t_k - 1) / t_{k+1},
// t_{k+1} = 0.5 (1 + sqrt(1 + (4 t_k) t_k)), no contraction.
__global__ void k_fista_setup(const double *__restrict__ L,
                              const unsigned long long *__restrict__ bmax, double lam,
                              double lam_rel, double *__restrict__ scal, double t0, int steps,
                              double *__restrict__ wv) {
  L += blockIdx.x;  // batched scenes: one block each; block 0 writes the weights
  bmax += blockIdx.x;
  scal += blockIdx.x * 4;
  if (blockIdx.x > 0) wv = nullptr;
  if (threadIdx.x == 0) {
    const double mx = __longlong_as_double((long long)*bmax);
    const double tau = 1.0 / L[0];
    const double lmb = (lam > 0.0) ? lam : lam_rel * mx;
    scal[0] = tau;
    scal[1] = lmb * tau;
    scal[2] = lmb;
    if (wv != nullptr) {
      double t = t0;
      for (int k = 0; k < steps; ++k) {
        const double tn =
            __dmul_rn(0.5, __dadd_rn(1.0, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(__dmul_rn(4.0, t), t)))));
        wv[k] = __ddiv_rn(__dsub_rn(t, 1.0), tn);
        t = tn;
      }
    }
  }
}

const void *fista_setup_kernel() { return (const void *)k_fista_setup; }

__global__ void k_fista_init(const double *__restrict__ c0, int64_t m_atoms, int64_t m_pad,
                             double *__restrict__ zd, double *__restrict__ cprev,
                             float *__restrict__ z32, int64_t zstride) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m_pad) return;
  c0 += blockIdx.y * m_atoms;  // batched scenes: grid y
  zd += blockIdx.y * m_pad;
  cprev += blockIdx.y * m_pad;
  z32 += blockIdx.y * zstride;
  const double v = (i < m_atoms) ? c0[i] : 0.0;
  zd[i] = v;
  cprev[i] = v;
  z32[i] = (float)v;
}

// y partials for one step.  256 threads per CTA, persistent over the tile list.
// Warp w covers column slabs {w, w+8, w+16, w+24} (16 columns); lane l covers
// rows {l, l+32, l+64, l+96}: 16 independent 16-byte loads per thread per tile.
// In the symmetric store a diagonal tile contributes through its upper
// triangle only (element (r,c), c > r, acts as both (r,c) and (c,r)), so the
// operator is exactly symmetric whatever rounding the Gram update left in the
// tile's lower half; this replaces the reference's A <- (A + A^H)/2
// (solver.py:193).
__device__ __forceinline__ void gemv_tile(const float *__restrict__ A,
                                          const int2 *__restrict__ tiles, int64_t t,
                                          const float *__restrict__ z32, float *__restrict__ P,
                                          int nt, int sym, float (*s_row)[kTile], float *s_col) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int2 ij = tiles[t];
  const int64_t store = sym ? tri_index(ij.x, ij.y, nt) : (int64_t)ij.x * nt + ij.y;
  const float4 *T = reinterpret_cast<const float4 *>(A + store * (int64_t)kTileElems);
  float4 a[4][4];
#pragma unroll
  for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
    for (int i = 0; i < 4; ++i) a[s4][i] = __ldg(T + (int64_t)(warp + 8 * s4) * kTile + lane + 32 * i);
  gemv_tile_compute<0>(a, ij.x, ij.y, z32, P, nt, sym, s_row, s_col);
}

// The tile store is read-only for the whole FISTA call (the state stream's
// Gram update that wrote it completed before the call's first kernel), so a
// CTA issues its first tile's loads BEFORE griddepcontrol.wait: under
// programmatic dependent launch they overlap the tail of the producer of x
// (k_hz) instead of following it.  Only x and the slot array P depend on the
// producer; both are touched after the wait.
__global__ void __launch_bounds__(256, 2)
k_gemv_sym(const float *__restrict__ A, const int2 *__restrict__ tiles, int64_t n_tiles,
           const float *__restrict__ z32, float *__restrict__ P, int nt, int sym, int batch,
           int64_t xstride, int reverse) {
  __shared__ float s_row[8][kTile];
  __shared__ float s_col[kTile];
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  // batched scenes share the tile list: work item t covers scene t / n_tiles
  const int64_t a_stride = (int64_t)nt * (sym ? nt + 1 : 2 * nt) / 2 * kTileElems;
  const int64_t p_stride = (int64_t)nt * nt * kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t total = n_tiles * batch;
  float4 a[4][4];
  auto load = [&](int64_t t, int2 &ij) {
    if (reverse) t = total - 1 - t;
    const int64_t sc = t / n_tiles;
    ij = tiles[t - sc * n_tiles];
    const int64_t store = sym ? tri_index(ij.x, ij.y, nt) : (int64_t)ij.x * nt + ij.y;
    const float4 *T = reinterpret_cast<const float4 *>(A + sc * a_stride + store * (int64_t)kTileElems);
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
      for (int i = 0; i < 4; ++i) a[s4][i] = __ldg(T + (int64_t)(warp + 8 * s4) * kTile + lane + 32 * i);
  };
  int64_t t = blockIdx.x;
  int2 ij = make_int2(0, 0);
  if (t < total) load(t, ij);
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  for (; t < total; t += gridDim.x) {
    if (t != blockIdx.x) load(t, ij);
    const int64_t sc = (reverse ? total - 1 - t : t) / n_tiles;
    gemv_tile_compute<0>(a, ij.x, ij.y, z32 + sc * xstride, P + sc * p_stride, nt, sym, s_row,
                         s_col);
  }
}


// k_gemv_sym with a one-tile prefetch (opt-in, see gemv_prefetch): while a CTA computes the tile held in
// registers, the bulk-copy engine (TMA, non-tensor) brings its next tile into a
// 64 KiB shared-memory buffer; both loads are issued before
// griddepcontrol.wait.  With two CTAs per SM the first two tiles of every CTA
// are in flight at once, so a store of <= 4 tiles per SM (cfg1: 528 tiles on
// 148 SMs) is read in one latency instead of two back-to-back ones.  Same
// thread mapping and summation order as k_gemv_sym (bitwise-equal slots).
__global__ void __launch_bounds__(256, 2)
k_gemv_sym_pf(const float *__restrict__ A, const int2 *__restrict__ tiles, int64_t n_tiles,
              const float *__restrict__ z32, float *__restrict__ P, int nt, int sym, int batch,
              int64_t xstride) {
  extern __shared__ __align__(128) unsigned char pf_buf[];
  __shared__ float s_row[8][kTile];
  __shared__ float s_col[kTile];
  __shared__ uint64_t bar;
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int64_t a_stride = (int64_t)nt * (sym ? nt + 1 : 2 * nt) / 2 * kTileElems;
  const int64_t p_stride = (int64_t)nt * nt * kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t total = n_tiles * batch;
  const int64_t G = gridDim.x;
  auto tile_ptr = [&](int64_t t, int2 &ij) {
    const int64_t sc = t / n_tiles;
    ij = tiles[t - sc * n_tiles];
    const int64_t store = sym ? tri_index(ij.x, ij.y, nt) : (int64_t)ij.x * nt + ij.y;
    return reinterpret_cast<const float4 *>(A + sc * a_stride + store * (int64_t)kTileElems);
  };
  int64_t t = blockIdx.x;
  int2 ij = make_int2(0, 0), ijn = make_int2(0, 0);
  if (threadIdx.x == 0) {
    bulk::mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    if (t + G < total) {
      bulk::arrive_expect_tx(&bar, kTileElems * 4);
      bulk::g2s(pf_buf, tile_ptr(t + G, ijn), kTileElems * 4, &bar, bulk::policy_evict_normal());
    }
  }
  float4 a[4][4];
  if (t < total) {
    const float4 *T = tile_ptr(t, ij);
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
      for (int i = 0; i < 4; ++i) a[s4][i] = __ldg(T + (int64_t)(warp + 8 * s4) * kTile + lane + 32 * i);
  }
  __syncthreads();  // barrier initialised
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  uint32_t phase = 0;
  const float4 *S = reinterpret_cast<const float4 *>(pf_buf);
  for (; t < total; t += G) {
    const int64_t sc = t / n_tiles;
    gemv_tile_compute<0>(a, ij.x, ij.y, z32 + sc * xstride, P + sc * p_stride, nt, sym, s_row,
                         s_col);
    const int64_t tn = t + G;
    if (tn >= total) break;
    tile_ptr(tn, ij);
    bulk::mbar_wait(&bar, phase);
    phase ^= 1u;
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
      for (int i = 0; i < 4; ++i) a[s4][i] = S[(warp + 8 * s4) * kTile + lane + 32 * i];
    __syncthreads();  // every thread has its copy of the buffer
    if (threadIdx.x == 0 && tn + G < total) {
      bulk::arrive_expect_tx(&bar, kTileElems * 4);
      bulk::g2s(pf_buf, tile_ptr(tn + G, ijn), kTileElems * 4, &bar, bulk::policy_evict_normal());
    }
  }
}

// Opt-in (SF_GEMV_PF=1): measured slower on B200 (cfg1 FISTA 14.74 vs 14.25
// us/step, cfg3 98.8 vs 98.75): the warm 34.6 MB store streams from L2 at the
// same ~5.6 TB/s as a plain read kernel (tools/gemv_bench.cu: 6.16 us), so the
// second tile's latency was not the limit.  Read per launch (graphs capture it
// once per engine), so tests can compare both.
bool gemv_prefetch() {
  const char *v = getenv("SF_GEMV_PF");
  return v && v[0] == '1';
}



// y_pix = Re(B) x with the slot reduction fused in (unsharded pixel mode): after
// writing a tile's partials the CTA counts one contribution for each block it
// touched; the CTA that completes a block (nt contributions) sums that block's
// slots in fixed order and resets the counter.  Deterministic: the sum order
// does not depend on which CTA performs it.
__global__ void __launch_bounds__(256, 2)
k_gemv_sym_reduce(const float *__restrict__ A, const int2 *__restrict__ tiles, int64_t n_tiles,
                  const float *__restrict__ x, float *__restrict__ P, int nt,
                  int *__restrict__ cnt, double *__restrict__ ypix) {
  __shared__ float s_row[8][kTile];
  __shared__ float s_col[kTile];
  __shared__ int s_last[2];
  __shared__ double s_red[kTile];
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
    gemv_tile(A, tiles, t, x, P, nt, 1, s_row, s_col);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int2 ij = tiles[t];
      s_last[0] = (atomicAdd(cnt + ij.x, 1) == nt - 1) ? ij.x : -1;
      s_last[1] = (ij.y != ij.x && atomicAdd(cnt + ij.y, 1) == nt - 1) ? ij.y : -1;
    }
    __syncthreads();
#pragma unroll 1
    for (int q = 0; q < 2; ++q) {
      const int blk = s_last[q];
      if (blk < 0) continue;
      __threadfence();
      const int r = threadIdx.x & (kTile - 1), half = threadIdx.x >> 7;
      const float *src = P + (int64_t)blk * nt * kTile + r;
      const int k0 = half * ((nt + 1) / 2), k1 = half ? nt : (nt + 1) / 2;
      double s0 = 0.0, s1 = 0.0;
      int kk = k0;
      for (; kk + 2 <= k1; kk += 2) {
        s0 += (double)__ldcg(src + (int64_t)kk * kTile);
        s1 += (double)__ldcg(src + (int64_t)(kk + 1) * kTile);
      }
      if (kk < k1) s0 += (double)__ldcg(src + (int64_t)kk * kTile);
      if (half) s_red[r] = s0 + s1;
      __syncthreads();
      if (!half) ypix[(int64_t)blk * kTile + r] = (s0 + s1) + s_red[r];
      if (threadIdx.x == 0) cnt[blk] = 0;
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// Streaming matvec over the tile store, TMA-staged (the default).  One CTA per
// SM: warp 8 is the producer -- one lane streams the CTA's tiles with 64 KiB
// bulk copies into a kGemvStages-deep shared-memory ring (mbarrier full/empty
// pairs) -- and warps 0-7 consume a tile from shared memory into the same
// register layout gemv_tile uses.  The tile store is constant during the FISTA
// loop (written by the Gram update before the loop's first ordinary launch),
// so the producer starts streaming BEFORE the programmatic-dependency wait and
// the first tiles load while the previous kernel (H z) drains; only the
// consumers wait for z.  With ypix != nullptr the fixed-order slot reduction of
// k_gemv_sym_reduce is fused in (unsharded pixel mode).
constexpr int kGemvStages = 3;
constexpr uint32_t kTileBytes = kTileElems * sizeof(float);
constexpr size_t kGemvSmem = (size_t)kGemvStages * kTileBytes;

__global__ void __launch_bounds__(288, 1)
k_gemv_tma(const float *__restrict__ A, const int2 *__restrict__ tiles, int64_t n_tiles,
           const float *__restrict__ z32, float *__restrict__ P, int nt, int sym,
           int *__restrict__ cnt, double *__restrict__ ypix, int stream_policy) {
  extern __shared__ __align__(128) unsigned char g_smem[];
  const float4 *stage = reinterpret_cast<const float4 *>(g_smem);
  __shared__ __align__(8) uint64_t full[kGemvStages], empty[kGemvStages];
  __shared__ float s_row[8][kTile];
  __shared__ float s_col[kTile];
  __shared__ int s_last[2];
  __shared__ double s_red[kTile];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int q = 0; q < kGemvStages; ++q) {
      bulk::mbar_init(&full[q], 1);
      bulk::mbar_init(&empty[q], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (warp == 8) {  // producer
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    if (lane == 0) {
      const uint64_t pol = stream_policy ? bulk::policy_evict_first() : bulk::policy_evict_last();
      int k = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
        const int q = k % kGemvStages;
        if (k >= kGemvStages) bulk::mbar_wait(&empty[q], ((k / kGemvStages) - 1) & 1);
        const int2 ij = tiles[t];
        const int64_t store = sym ? tri_index(ij.x, ij.y, nt) : (int64_t)ij.x * nt + ij.y;
        bulk::arrive_expect_tx(&full[q], kTileBytes);
        bulk::g2s((void *)(stage + (size_t)q * (kTileElems / 4)), A + store * (int64_t)kTileElems,
                  kTileBytes, &full[q], pol);
      }
    }
    return;
  }
  pdl_enter();
  int k = 0;
  for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x, ++k) {
    const int q = k % kGemvStages;
    bulk::mbar_wait(&full[q], (k / kGemvStages) & 1);
    const float4 *T = stage + (size_t)q * (kTileElems / 4);
    float4 a[4][4];
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
      for (int i = 0; i < 4; ++i) a[s4][i] = T[(warp + 8 * s4) * kTile + lane + 32 * i];
    __syncwarp();
    if (lane == 0) bulk::arrive(&empty[q]);
    const int2 ij = tiles[t];
    gemv_tile_compute<1>(a, ij.x, ij.y, z32, P, nt, sym, s_row, s_col);
    if (ypix == nullptr) continue;
    // fused slot reduction (see k_gemv_sym_reduce); gemv_tile_compute ended
    // with a consumer barrier, so all of this tile's slots are written
    if (threadIdx.x == 0) {
      __threadfence();
      s_last[0] = (atomicAdd(cnt + ij.x, 1) == nt - 1) ? ij.x : -1;
      s_last[1] = (ij.y != ij.x && atomicAdd(cnt + ij.y, 1) == nt - 1) ? ij.y : -1;
    }
    gemv_bar<1>();
#pragma unroll 1
    for (int qq = 0; qq < 2; ++qq) {
      const int blk = s_last[qq];
      if (blk < 0) continue;
      __threadfence();
      const int r = threadIdx.x & (kTile - 1), half = threadIdx.x >> 7;
      const float *src = P + (int64_t)blk * nt * kTile + r;
      const int k0 = half * ((nt + 1) / 2), k1 = half ? nt : (nt + 1) / 2;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      int kk = k0;
      for (; kk + 4 <= k1; kk += 4) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = __ldcg(src + (int64_t)(kk + u) * kTile);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc[u] += (double)v[u];
      }
      for (; kk < k1; ++kk) acc[0] += (double)__ldcg(src + (int64_t)kk * kTile);
      const double part = (acc[0] + acc[1]) + (acc[2] + acc[3]);
      if (half) s_red[r] = part;
      gemv_bar<1>();
      if (!half) ypix[(int64_t)blk * kTile + r] = part + s_red[r];
      if (threadIdx.x == 0) cnt[blk] = 0;
      gemv_bar<1>();
    }
  }
}

static sf_status launch_gemv_tma(const float *A, const int2 *tiles, int64_t n_tiles,
                                 const float *z32, float *P, int nt, int sym, int *cnt,
                                 double *ypix, int grid, cudaStream_t st) {
  static std::atomic<uint64_t> attr_set{0};
  if (attr_pending(attr_set)) {
    cudaError_t ce = cudaFuncSetAttribute(k_gemv_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)kGemvSmem);
    if (ce != cudaSuccess)
      return fail(SF_ECUDA, std::string("k_gemv_tma smem attribute: ") + cudaGetErrorString(ce));
    attr_done(attr_set);
  }
  // stores beyond ~half of L2 are streamed (evict_first) so the vectors stay
  // resident; smaller stores are kept (evict_last) and re-read from L2 each step
  const int policy = (n_tiles * (int64_t)kTileBytes > ((int64_t)64 << 20)) ? 1 : 0;
  const int64_t g = n_tiles < grid ? n_tiles : grid;
  cudaError_t ce = launch_pdl(k_gemv_tma, dim3((unsigned)g), dim3(288), kGemvSmem, st, A, tiles,
                              n_tiles, z32, P, nt, sym, cnt, ypix, policy);
  if (ce != cudaSuccess) return fail(SF_ECUDA, std::string("k_gemv_tma: ") + cudaGetErrorString(ce));
  SF_LAUNCH_CHECK();
  return SF_OK;
}

// Register-streaming kernels are the default: measured in the pipelined bench
// (operator kernels running beside the FISTA chain) they beat the TMA ring --
// cfg1 4143 vs 3613 pulses/s, cfg3 466 vs 449 -- and are equal alone (cfg3
// 84 vs 88 us per matvec).  SF_GEMV_TMA=1 selects k_gemv_tma.
static bool gemv_ldg() {
  static const bool v = getenv("SF_GEMV_TMA") == nullptr;
  return v;
}

sf_status launch_gemv_reduce(const float *A, const int2 *tiles, int64_t n_tiles, const float *x,
                             float *P, int nt, int *cnt, double *ypix, int grid, cudaStream_t st) {
  if (n_tiles == 0) return SF_OK;
  if (!gemv_ldg()) return launch_gemv_tma(A, tiles, n_tiles, x, P, nt, 1, cnt, ypix, grid / 2, st);
  const int64_t g = n_tiles < grid ? n_tiles : grid;
  k_gemv_sym_reduce<<<(unsigned)g, 256, 0, st>>>(A, tiles, n_tiles, x, P, nt, cnt, ypix);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

// ---------------------------------------------------------------------------
// Persistent FISTA loop for pixel-space statistics: one cooperative launch runs
// `steps` iterations of
//   x = H z  ->  y_pix = Re(B) x  ->  g = H^T y_pix - Re(b), shrink, momentum
// with grid-wide barriers between the phases (kernels.py:85-102).  The slot
// reduction of y_pix is fused into the GEMV phase: each 128-pixel block counts
// its nt contributions and the CTA that delivers the last one sums the block's
// slots in fixed order.  Data produced by other CTAs in the same launch is read
// with ld.global.cg (L2), never through L1.
namespace cg = cooperative_groups;

__device__ __forceinline__ void hz_phase(const PixFistaArgs &a) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); p < a.n_pad;
       p += warps) {
    double s = 0.0;
    if (p < a.n)
      for (int64_t k = a.csr_ptr[p] + lane; k < a.csr_ptr[p + 1]; k += 32)
        s += a.csr_w[k] * __ldcg(a.zd + a.csr_atom[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) a.x[p] = (float)s;
  }
}

__device__ __forceinline__ void trace_mark(const PixFistaArgs &a, int &n) {
  if (a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[n] = t;
  }
  ++n;
}

__global__ void __launch_bounds__(256, 2) k_fista_pix(PixFistaArgs a) {
  cg::grid_group grid = cg::this_grid();
  int tn = 0;
  trace_mark(a, tn);
  __shared__ float s_row[8][kTile];
  __shared__ float s_col[kTile];
  const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t gthreads = (int64_t)gridDim.x * blockDim.x;
  if (a.init) {
    for (int64_t j = gtid; j < a.m; j += gthreads) {
      const double v = a.c0[j];
      a.zd[j] = v;
      a.cprev[j] = v;
    }
    grid.sync();
    hz_phase(a);
    grid.sync();
  }
  const double tau = a.scal[0], thresh = a.scal[1];
  for (int k = 0; k < a.steps; ++k) {
    // ---- partial slots of y_pix = Re(B) x over the tile triangle
    for (int64_t t = blockIdx.x; t < a.n_tiles; t += gridDim.x)
      gemv_tile(a.B, a.tiles, t, a.x, a.P, a.nt, 1, s_row, s_col);
    trace_mark(a, tn);
    grid.sync();
    trace_mark(a, tn);
    // ---- y_pix: each pixel's nt slots summed by an 8-lane group (lane g takes
    // slots g, g+8, ...), then a fixed 3-level shuffle tree
    for (int64_t e8 = gtid; e8 < a.n_pad * 8; e8 += gthreads) {
      const int64_t i = e8 >> 3;
      const int g = (int)(e8 & 7);
      const int64_t blk = i / kTile;
      const int r = (int)(i - blk * kTile);
      const float *src = a.P + blk * (int64_t)a.nt * kTile + r;
      double y = 0.0;
      for (int q = g; q < a.nt; q += 8) y += (double)__ldcg(src + (int64_t)q * kTile);
      y += __shfl_xor_sync(0xffffffffu, y, 1);
      y += __shfl_xor_sync(0xffffffffu, y, 2);
      y += __shfl_xor_sync(0xffffffffu, y, 4);
      if (g == 0) a.ypix[i] = y;
    }
    trace_mark(a, tn);
    grid.sync();
    trace_mark(a, tn);
    // ---- atom step: g = H^T y_pix - Re(b); kernels.py:90-97
    const double w = a.w[k];
    const bool last = a.last_chunk && (k == a.steps - 1);
    for (int64_t j = gtid; j < a.m; j += gthreads) {
      int32_t pi[8];
      double wi[8];
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        pi[l] = (l < a.width) ? a.ell_idx[j * a.width + l] : -1;
        wi[l] = (l < a.width) ? a.ell_w[j * a.width + l] : 0.0;
      }
      double y = 0.0;
#pragma unroll
      for (int l = 0; l < 8; ++l)
        if (pi[l] >= 0) y += wi[l] * __ldcg(a.ypix + pi[l]);
      const double z = a.zd[j];
      const double u = z - tau * (y - a.b[j].x);
      double ci;
      if (u > thresh) ci = u - thresh;
      else if (u < -thresh) ci = u + thresh;
      else ci = 0.0;
      const double zn = ci + w * (ci - a.cprev[j]);
      a.cprev[j] = ci;
      a.zd[j] = zn;
      if (last) a.c_out[j] = ci;
    }
    trace_mark(a, tn);
    if (last) break;
    grid.sync();
    trace_mark(a, tn);
    hz_phase(a);
    trace_mark(a, tn);
    grid.sync();
    trace_mark(a, tn);
  }
}

sf_status launch_fista_pix(PixFistaArgs &a, int grid, cudaStream_t st) {
  void *args[] = {&a};
  cudaError_t e = cudaLaunchCooperativeKernel((const void *)k_fista_pix, dim3(grid), dim3(256),
                                              args, 0, st);
  count_launch();
  if (e != cudaSuccess) return fail(SF_ECUDA, std::string("cooperative FISTA launch: ") +
                                                  cudaGetErrorString(e));
  return SF_OK;
}

int fista_pix_max_grid(int device) {
  int per_sm = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fista_pix, 256, 0);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return per_sm * sms;
}

// Reduce the nt partial slots of each element and apply the step (fp64).
__global__ void __launch_bounds__(256)
k_fista_step(const float *__restrict__ P, int nt, const double2 *__restrict__ b,
             const double *__restrict__ corr, int64_t m_atoms, int64_t m_pad,
             double *__restrict__ zd, double *__restrict__ cprev, float *__restrict__ z32,
             const double *__restrict__ scal, double w, double *__restrict__ c_out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= m_pad) return;
  const int64_t blk = i / kTile;
  const int r = (int)(i - blk * kTile);
  const float *src = P + blk * (int64_t)nt * kTile + r;
  double y0 = 0.0, y1 = 0.0, y2 = 0.0, y3 = 0.0;
  int k = 0;
  for (; k + 4 <= nt; k += 4) {
    y0 += (double)src[(int64_t)(k + 0) * kTile];
    y1 += (double)src[(int64_t)(k + 1) * kTile];
    y2 += (double)src[(int64_t)(k + 2) * kTile];
    y3 += (double)src[(int64_t)(k + 3) * kTile];
  }
  for (; k < nt; ++k) y0 += (double)src[(int64_t)k * kTile];
  const double y = (y0 + y1) + (y2 + y3);
  if (i >= m_atoms) return;
  const double tau = scal[0], thresh = scal[1];
  const double bre = (corr != nullptr) ? corr[i] : b[i].x;
  // kernels.py:90-97
  const double z = zd[i];
  const double u = z - tau * (y - bre);
  double ci;
  if (u > thresh) ci = u - thresh;
  else if (u < -thresh) ci = u + thresh;
  else ci = 0.0;
  const double zn = ci + w * (ci - cprev[i]);
  cprev[i] = ci;
  zd[i] = zn;
  z32[i] = (float)zn;
  if (c_out != nullptr) c_out[i] = ci;
}

// dense fp64 [m][m] (row-major) -> tile store (fp32); zero outside [0,m)
__global__ void k_pack_tiles(const double *__restrict__ dense, int64_t m,
                             const int2 *__restrict__ tiles, float *__restrict__ A) {
  const int64_t t = blockIdx.x;
  const int2 ij = tiles[t];
  for (int e = threadIdx.x; e < kTileElems; e += blockDim.x) {
    const int r = e / kTile, c = e % kTile;
    const int64_t gi = (int64_t)ij.x * kTile + r, gj = (int64_t)ij.y * kTile + c;
    const double v = (gi < m && gj < m) ? dense[gi * m + gj] : 0.0;
    A[t * kTileElems + tile_offset(r, c)] = (float)v;
  }
}

// tile store -> dense fp64 [m][m]; sym=1 mirrors the upper triangle
__global__ void k_unpack_tiles(const float *__restrict__ A, const int2 *__restrict__ tiles,
                               int64_t m, int sym, double *__restrict__ dense) {
  const int64_t t = blockIdx.x;
  const int2 ij = tiles[t];
  for (int e = threadIdx.x; e < kTileElems; e += blockDim.x) {
    const int r = e / kTile, c = e % kTile;
    const int64_t gi = (int64_t)ij.x * kTile + r, gj = (int64_t)ij.y * kTile + c;
    if (gi >= m || gj >= m) continue;
    if (sym && ij.x == ij.y && c < r) continue;  // lower half of a diagonal tile is unused
    const double v = (double)A[t * kTileElems + tile_offset(r, c)];
    dense[gi * m + gj] = v;
    if (sym) dense[gj * m + gi] = v;
  }
}

sf_status launch_bmax(const double2 *b, int64_t m_atoms, unsigned long long *bmax,
                      cudaStream_t st) {
  k_bmax<<<1, 1024, 0, st>>>(b, m_atoms, bmax);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_fista_setup(const double *L, const unsigned long long *bmax, double lam,
                             double lam_rel, double *scal, cudaStream_t st, double t0, int steps,
                             double *wv, int batch) {
  k_fista_setup<<<batch, 32, 0, st>>>(L, bmax, lam, lam_rel, scal, t0, steps, wv);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_fista_init(const double *c0, int64_t m_atoms, int64_t m_pad, double *zd,
                            double *cprev, float *z32, cudaStream_t st, int batch,
                            int64_t zstride) {
  const int bs = 256;
  k_fista_init<<<dim3((unsigned)((m_pad + bs - 1) / bs), batch), bs, 0, st>>>(
      c0, m_atoms, m_pad, zd, cprev, z32, zstride);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_gemv(const float *A, const int2 *tiles, int64_t n_tiles, const float *z32,
                      float *P, int nt, int sym, int grid, cudaStream_t st, int batch,
                      int64_t xstride, int reverse) {
  if (n_tiles == 0) return SF_OK;
  if (!gemv_ldg() && batch == 1)
    return launch_gemv_tma(A, tiles, n_tiles, z32, P, nt, sym, nullptr, nullptr, grid / 2, st);
  const int64_t tot = n_tiles * batch;
  const int64_t g = tot < grid ? tot : grid;
  cudaError_t ce;
  if (gemv_prefetch()) {
    static std::atomic<uint64_t> set{0};
    if (attr_pending(set)) {
      SF_CUDA_TRY(cudaFuncSetAttribute(k_gemv_sym_pf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kTileElems * 4));
      attr_done(set);
    }
    ce = launch_pdl(k_gemv_sym_pf, dim3((unsigned)g), dim3(256), (size_t)kTileElems * 4, st, A,
                    tiles, n_tiles, z32, P, nt, sym, batch, xstride);
  } else {
    ce = launch_pdl(k_gemv_sym, dim3((unsigned)g), dim3(256), 0, st, A, tiles, n_tiles, z32, P,
                    nt, sym, batch, xstride, reverse);
  }
  if (ce != cudaSuccess) return fail(SF_ECUDA, std::string("k_gemv_sym: ") + cudaGetErrorString(ce));
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_fista_step(const float *P, int nt, const double2 *b, const double *corr,
                            int64_t m_atoms, int64_t m_pad, double *zd, double *cprev,
                            float *z32, const double *scal, double w, double *c_out,
                            cudaStream_t st) {
  const int bs = 256;
  k_fista_step<<<(unsigned)((m_pad + bs - 1) / bs), bs, 0, st>>>(
      P, nt, b, corr, m_atoms, m_pad, zd, cprev, z32, scal, w, c_out);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_pack_tiles(const double *dense, int64_t m, const int2 *tiles, int64_t n_tiles,
                            float *A, cudaStream_t st) {
  if (n_tiles == 0) return SF_OK;
  k_pack_tiles<<<(unsigned)n_tiles, 256, 0, st>>>(dense, m, tiles, A);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_unpack_tiles(const float *A, const int2 *tiles, int64_t n_tiles, int64_t m,
                              int sym, double *dense, cudaStream_t st) {
  if (n_tiles == 0) return SF_OK;
  k_unpack_tiles<<<(unsigned)n_tiles, 256, 0, st>>>(A, tiles, m, sym, dense);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

}  // namespace sf
