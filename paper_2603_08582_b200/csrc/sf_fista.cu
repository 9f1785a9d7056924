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
#include <float.h>
#include <stdlib.h>

#include <string>

#include "sf_common.cuh"
#include "sf_kernels.cuh"

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
