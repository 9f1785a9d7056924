// sf_dirichlet.cu -- closed-form pixel-space Gram update for a uniform
// frequency grid (precision SF_PREC_DIRICHLET, pixel mode).
//
// The reference forms dA = G^H G / sigma^2 with G = F H (solver.py:178-183,
// geometry.py:97-107); in pixel space the state update is
//   Re(B) += Re(F^H F) / sigma^2,   Re(F^H F)[i][j] = sum_m cos(w_m (tau_i - tau_j)).
// geometry.angular_frequencies (geometry.py:78-90) is 2 pi linspace(...), so
// w_m = w_0 + m delta and the sum over the N_r frequencies is a Dirichlet
// kernel (exact identity, no approximation):
//   sum_m cos(w_m D) = cos(w_c D) * sin(N_r pi x) / sin(pi x),
//   w_c = (w_0 + w_{N_r-1}) / 2,   x = delta D / (2 pi),   D = tau_i - tau_j.
// Each stored entry therefore costs O(1) instead of the 2 N_r multiply-adds of
// the tensor-core contraction (k_gram_f16x3): the update becomes a pure
// read-modify-write of the packed triangle, bounded by HBM (cfg3/cfg4) instead
// of the tensor pipe.
//
// Precision (vs the float64 oracle): per pixel the table holds
//   u_i = tau_i delta / (2 pi)  (fp64),  C_i, S_i = cos, sin(w_c tau_i)  (fp32 of fp64 sincos)
// so cos(w_c D) = C_i C_j + S_i S_j to ~1e-7 absolute.  x = u_i - u_j is
// reduced modulo 1 in fp64 (r = x - k, |r| <= 1/2, exact), so the only fp32
// rounding is that of r itself -- relative, which keeps the steep main and
// grating lobes of the kernel accurate (an absolute error in r would be
// amplified by the lobe slope ~N_r^2).  Then
//   sin(N pi x) / sin(pi x) = (-1)^(k (N-1)) sinpi(N r) / sinpi(r)   (= N at r = 0).
// Measured entry error <= ~2e-7 relative to N_r (tests/test_gpu_parity.py::
// test_dirichlet_gram_matches_oracle), against ~5e-6 for the f16x3 path.
//
// Frequencies that are not uniformly spaced (beyond 1e-12 relative) cannot use
// this path: host inputs are rejected at the call, device inputs raise the
// engine's device error flag (bit 1), reported by the next sf_get_scalars.
#include <math.h>

#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {

// Per-pulse pixel table.  Padded pixels (p >= N) get C = S = 0, which makes
// their contribution exactly zero.
__global__ void __launch_bounds__(256)
k_dirichlet_prep(const double *__restrict__ tau, int64_t n_pix, int64_t dpad,
                 const double *__restrict__ in, int64_t in_stride, int n_r,
                 DirPix *__restrict__ tab, int *__restrict__ flag) {
  const int sc = blockIdx.y;
  tau += sc * n_pix;
  tab += sc * dpad;
  const double *w = in + sc * in_stride;  // omega at offset 0 of each scene block
  const double w0 = w[0], w1 = w[n_r - 1];
  const double delta = n_r > 1 ? (w1 - w0) / (double)(n_r - 1) : 0.0;
  const double wc = 0.5 * (w0 + w1);
  if (blockIdx.x == 0) {  // uniform grid check, one block per scene
    const double tol = 1e-12 * fmax(fabs(w0), fabs(w1));
    bool bad = false;
    for (int m = threadIdx.x; m < n_r; m += blockDim.x)
      bad |= !(fabs(w[m] - fma((double)m, delta, w0)) <= tol);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 2);
  }
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= dpad) return;
  DirPix v;
  if (p < n_pix) {
    const double t = tau[p];
    v.u = t * (delta * (0.5 / 3.14159265358979323846));
    double s, c;
    sincos(wc * t, &s, &c);
    v.c = (float)c;
    v.s = (float)s;
  } else {
    v.u = 0.0;
    v.c = 0.f;
    v.s = 0.f;
  }
  tab[p] = v;
}

// sin(pi r) for |r| <= 1/2: odd minimax polynomial, max relative error 1.8e-7
// in fp32 (no range reduction, no conversions).
__device__ __forceinline__ float sinpi_half(float r) {
  const float s = r * r;
  float p = fmaf(s, 0.07756056636571884f, -0.5982431769371033f);
  p = fmaf(s, p, 2.55007004737854f);
  p = fmaf(s, p, -5.167709827423096f);
  p = fmaf(s, p, 3.1415927410125732f);
  return r * p;
}

// sin(N pi x) / sin(pi x) with x = ur - uc (see the file comment).  Integer
// rounding by the 1.5 * 2^52 (fp64) and 1.5 * 2^23 (fp32) magic constants, so
// the parities come from mantissa bits and the only conversion-pipe
// instructions are one F2F and one MUFU.RCP per entry.
__device__ __forceinline__ float dirichlet_ratio(double ur, double uc, float nr, uint32_t neven) {
  const double x = ur - uc;
  const double t = x + 6755399441055744.0;
  const double k = t - 6755399441055744.0;   // nearest integer to x
  // x - k is exact in fp64, |f| <= 1/2.  The 1e-20 offset keeps f = 0 (the
  // diagonal, equal ranges) off 0/0: the ratio is N (1 - O(N^2 f^2)) there, and
  // every other |f| is >= ulp(u) ~ 1e-14, where the offset is far below rounding.
  const float f = (float)(x - k) + 1e-20f;
  const uint32_t kodd = (uint32_t)__double2loint(t) & 1u;
  const float y = nr * f;
  const float ty = y + 12582912.f;
  const float j = ty - 12582912.f;           // nearest integer to y
  const uint32_t jodd = __float_as_uint(ty) & 1u;
  // sin(N pi x) = (-1)^(N k) sin(pi y) = (-1)^(N k + j) sin(pi (y - j)),  sin(pi x) = (-1)^k sin(pi f)
  float rc;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(sinpi_half(f)));
  const float q = sinpi_half(y - j) * rc;
  const uint32_t flip = ((kodd & neven) ^ jodd) << 31;
  return __uint_as_float(__float_as_uint(q) ^ flip);
}

// Re(B)_out = Re(B)_in + Re(F^H F) / sigma^2 on the listed tiles (all scenes).
// Persistent, one CTA of 512 threads per SM, tiles claimed from a counter, tiles streamed through shared
// memory by the bulk-copy engine (TMA, non-tensor): a 3-stage ring of 64 KiB
// tiles, thread 0 keeps two tile loads in flight while every thread updates the
// current tile in place in shared memory (thread = rows r and r + 64, slabs
// 4h..4h+3 = 16 columns; the column table is read as warp-uniform broadcasts),
// then thread 0 writes the tile back with one bulk shared -> global copy.  The
// ~40 instructions per entry then overlap the HBM read-modify-write instead of
// alternating with it.
namespace dir {
constexpr int kThreads = 512;
constexpr int kStages = 3;
constexpr uint32_t kTileBytes = kTileElems * 4;
}  // namespace dir

__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(bulk::smem_u32(src)), "r"(bytes)
               : "memory");
}

__global__ void __launch_bounds__(dir::kThreads, 1)
k_gram_dirichlet(const DirPix *__restrict__ tab, int64_t dpad, const int2 *__restrict__ tiles,
                 int64_t n_tiles, int nt, const double *__restrict__ in, int64_t in_stride,
                 int64_t off_s, int n_r, const float *Ain, float *A, int batch, int64_t a_stride,
                 unsigned long long *__restrict__ next) {
  using namespace dir;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t full[kStages];
  __shared__ int64_t s_it[kStages];  // work item held by each stage (>= total: none)
  const int r = threadIdx.x & 63;  // rows r and r + 64
  const int h = threadIdx.x >> 6;  // slabs 4h .. 4h+3 (16 columns)
  const float nr = (float)n_r;
  const uint32_t neven = (n_r & 1) ? 0u : 1u;
  const int64_t total = n_tiles * batch;
  auto tile_off = [&](int64_t it) {
    const int sc = (int)(it / n_tiles);
    const int2 ij = tiles[it - (int64_t)sc * n_tiles];
    return ((int64_t)ij.x * nt - (int64_t)ij.x * (ij.x - 1) / 2 + (ij.y - ij.x)) * kTileElems +
           sc * a_stride;
  };
  const uint64_t pol = bulk::policy_evict_normal();
  // work items are claimed from a global counter (thread 0, one ahead of the
  // two in flight): a CTA that becomes resident late -- its SM busy with the
  // FISTA chain when the kernel starts -- simply claims fewer tiles, instead of
  // finishing a fixed share after everyone else.  Every tile's update is
  // independent, so the result does not depend on who claims it.
  auto claim = [&](int st) {
    const int64_t it = (int64_t)atomicAdd(next, 1ull);
    s_it[st] = it;
    if (it < total) {
      bulk::arrive_expect_tx(&full[st], kTileBytes);
      bulk::g2s(smem + st * kTileBytes, Ain + tile_off(it), kTileBytes, &full[st], pol);
    } else {
      bulk::arrive(&full[st]);
    }
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) bulk::mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    claim(0);
    claim(1);
  }
  __syncthreads();
  for (int64_t k = 0;; ++k) {
    const int st = (int)(k % kStages);
    bulk::mbar_wait(&full[st], (uint32_t)(k / kStages) & 1u);
    const int64_t it = s_it[st];
    if (it >= total) break;  // claims are increasing: nothing later either
    const int sc = (int)(it / n_tiles);
    const int2 ij = tiles[it - (int64_t)sc * n_tiles];
    const DirPix *ts = tab + sc * dpad;
    const double is = in[sc * in_stride + off_s];  // 1 / sigma
    const float inv = (float)(is * is);
    const DirPix pa = ts[(int64_t)ij.x * kTile + r];
    const DirPix pb = ts[(int64_t)ij.x * kTile + r + 64];
    const float ca = pa.c * inv, sa = pa.s * inv, cb = pb.c * inv, sb = pb.s * inv;
    const DirPix *pc = ts + (int64_t)ij.y * kTile + 16 * h;
    float4 *T = reinterpret_cast<float4 *>(smem + st * kTileBytes);
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      float va[4], vb[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const DirPix c = pc[4 * s + q];
        va[q] = fmaf(ca, c.c, sa * c.s) * dirichlet_ratio(pa.u, c.u, nr, neven);
        vb[q] = fmaf(cb, c.c, sb * c.s) * dirichlet_ratio(pb.u, c.u, nr, neven);
      }
      float4 &oa = T[(4 * h + s) * kTile + r];
      float4 &ob = T[(4 * h + s) * kTile + r + 64];
      float4 x = oa, y = ob;
      x.x += va[0];
      x.y += va[1];
      x.z += va[2];
      x.w += va[3];
      y.x += vb[0];
      y.y += vb[1];
      y.z += vb[2];
      y.w += vb[3];
      oa = x;
      ob = y;
    }
    // every writer makes its generic-proxy stores visible to the async proxy
    // before the barrier; thread 0 then issues the bulk store of the tile
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();  // the whole tile is updated in shared memory
    if (threadIdx.x == 0) {
      bulk_s2g(A + tile_off(it), T, kTileBytes);
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      // stage (k+2)%3 last held tile k-1: its store must have read it
      asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
      claim((int)((k + 2) % kStages));
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

sf_status launch_dirichlet_prep(const double *tau, int64_t n_pix, int64_t dpad, const double *in,
                                int64_t in_stride, int n_r, DirPix *tab, int *flag,
                                cudaStream_t st, int batch) {
  const int bs = 256;
  k_dirichlet_prep<<<dim3((unsigned)((dpad + bs - 1) / bs), batch), bs, 0, st>>>(
      tau, n_pix, dpad, in, in_stride, n_r, tab, flag);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_gram_dirichlet(const DirPix *tab, int64_t dpad, const int2 *tiles,
                                int64_t n_tiles, int nt, const double *in, int64_t in_stride,
                                int64_t off_s, int n_r, const float *Ain, float *A, int grid,
                                cudaStream_t st, int batch, int64_t a_stride,
                                unsigned long long *next) {
  const int64_t total = n_tiles * batch;
  if (total == 0) return SF_OK;
  const size_t smem = (size_t)dir::kStages * dir::kTileBytes;
  static std::atomic<uint64_t> set{0};
  if (attr_pending(set)) {
    SF_CUDA_TRY(cudaFuncSetAttribute(k_gram_dirichlet, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    attr_done(set);
  }
  SF_CUDA_TRY(cudaMemsetAsync(next, 0, sizeof(unsigned long long), st));
  const int64_t g = total < grid ? total : grid;
  k_gram_dirichlet<<<(unsigned)g, dir::kThreads, smem, st>>>(tab, dpad, tiles, n_tiles, nt, in,
                                                             in_stride, off_s, n_r, Ain, A, batch,
                                                             a_stride, next);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

bool omega_uniform(const double *w, int n_r) {
  if (n_r < 3) return true;
  const double w0 = w[0], w1 = w[n_r - 1];
  const double delta = (w1 - w0) / (double)(n_r - 1);
  const double tol = 1e-12 * fmax(fabs(w0), fabs(w1));
  for (int m = 0; m < n_r; ++m)
    if (!(fabs(w[m] - fma((double)m, delta, w0)) <= tol)) return false;
  return true;
}

}  // namespace sf
