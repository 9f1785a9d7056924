// sf_exact.cu -- the complex atom-space statistics kept exactly (keep_complex).
//
// The reference's SufficientStatistics holds the full complex A (solver.py:88-109)
// and updates it in float64: dA = G^H R^-1 G, A <- (A + dA + (A + dA)^H) / 2
// (solver.py:178-193).  The engine's FISTA reads fp32 Re(A) tiles; with
// keep_complex an atom-mode engine also keeps A in fp64 (small M: the
// reference-API drop-in path, tests with random dense operators) and derives
// the tiles from it after every pulse, so `stats.A`, its text checkpoint and
// a resumed stream are exact.
//   k_herk_c64       A += G^H G / sigma^2 (upper triangle computed, lower
//                    mirrored as the conjugate: exactly Hermitian)
//   k_kgram_c64      per-split partials of K~ = G G^H / sigma^2 in fp64 (the
//                    N_r-space power-iteration operator)
//   k_pack_re        fp32 tiles <- Re(A)
//   k_dense_residual / k_dense_grad   batch_objective / batch_gradient terms
//                    of one whitened pulse (solver.py:243-264)
//   k_gemv64 / k_seam_step   the float64 kernels.fista_inner seam (kernels.py:32-53)
#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {

// One 32 x 32 block of A per CTA (upper triangle of blocks only); the sum over
// the n_r samples runs in order in fp64.
__global__ void __launch_bounds__(256)
k_herk_c64(const double2 *__restrict__ G, int n_r, int64_t m, double inv_s2,
           double2 *__restrict__ A) {
  const int64_t nb = (m + 31) / 32;
  int64_t bi = 0, rem = blockIdx.x;
  while (rem >= nb - bi) {  // row block bi holds blocks (bi, bi..nb-1)
    rem -= nb - bi;
    ++bi;
  }
  const int64_t bj = bi + rem;
  __shared__ double2 si[32][33], sj[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double2 acc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < n_r; k0 += 32) {
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
      const int kk = e >> 5, c = e & 31;
      const int k = k0 + kk;
      const int64_t ci = bi * 32 + c, cj = bj * 32 + c;
      si[kk][c] = (k < n_r && ci < m) ? G[(int64_t)k * m + ci] : make_double2(0.0, 0.0);
      sj[kk][c] = (k < n_r && cj < m) ? G[(int64_t)k * m + cj] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const int kn = min(32, n_r - k0);
    for (int kk = 0; kk < kn; ++kk) {
      const double2 gj = sj[kk][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 gi = si[kk][ty + 8 * q];
        // conj(gi) * gj
        acc[q].x += gi.x * gj.x + gi.y * gj.y;
        acc[q].y += gi.x * gj.y - gi.y * gj.x;
      }
    }
    __syncthreads();
  }
  const int64_t j = bj * 32 + tx;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t i = bi * 32 + ty + 8 * q;
    if (i >= m || j >= m || j < i) continue;
    double2 a = A[i * m + j];
    a.x += acc[q].x * inv_s2;
    a.y += acc[q].y * inv_s2;
    if (i == j) a.y = 0.0;  // Hermitian: real diagonal
    A[i * m + j] = a;
    if (i != j) A[j * m + i] = make_double2(a.x, -a.y);
  }
}

// Kpart[split][a][c] = inv_s2 * sum_{j in split} G[a][j] conj(G[c][j]), fp64.
__global__ void __launch_bounds__(256)
k_kgram_c64(const double2 *__restrict__ G, int64_t m, int n_r, double inv_s2,
            int64_t per_split, double2 *__restrict__ Kpart) {
  __shared__ double2 s1[32][33], s2[32][33];
  const int nb = (n_r + 31) / 32;
  const int ab = blockIdx.x / nb, cb = blockIdx.x % nb;
  const int split = blockIdx.y;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t j0 = (int64_t)split * per_split;
  const int64_t j1 = min(m, j0 + per_split);
  double2 acc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = make_double2(0.0, 0.0);
  for (int64_t jc = j0; jc < j1; jc += 32) {
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
      const int jj = e >> 5, r = e & 31;
      const int64_t j = jc + jj;
      const int a = ab * 32 + r, c = cb * 32 + r;
      s1[jj][r] = (j < j1 && a < n_r) ? G[(int64_t)a * m + j] : make_double2(0.0, 0.0);
      s2[jj][r] = (j < j1 && c < n_r) ? G[(int64_t)c * m + j] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    for (int jj = 0; jj < 32; ++jj) {
      const double2 g2 = s2[jj][tx];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double2 g1 = s1[jj][ty + 8 * q];
        acc[q].x += g1.x * g2.x + g1.y * g2.y;  // g1 * conj(g2)
        acc[q].y += g1.y * g2.x - g1.x * g2.y;
      }
    }
    __syncthreads();
  }
  const int c = cb * 32 + tx;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int a = ab * 32 + ty + 8 * q;
    if (a < n_r && c < n_r)
      Kpart[((int64_t)split * n_r + a) * n_r + c] =
          make_double2(acc[q].x * inv_s2, acc[q].y * inv_s2);
  }
}

__global__ void k_pack_re(const double2 *__restrict__ A, int64_t m, const int2 *__restrict__ tiles,
                          float *__restrict__ T) {
  const int64_t t = blockIdx.x;
  const int2 ij = tiles[t];
  for (int e = threadIdx.x; e < kTileElems; e += blockDim.x) {
    const int r = e / kTile, c = e % kTile;
    const int64_t gi = (int64_t)ij.x * kTile + r, gj = (int64_t)ij.y * kTile + c;
    const double v = (gi < m && gj < m) ? A[gi * m + gj].x : 0.0;
    T[t * kTileElems + tile_offset(r, c)] = (float)v;
  }
}

// r = G c - d (one thread per sample, in-order sum over atoms); quad = |r|^2 / s2
__global__ void k_dense_residual(const double2 *__restrict__ G, const double2 *__restrict__ d,
                                 int n_r, int64_t m, const double *__restrict__ c,
                                 double2 *__restrict__ r) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n_r) return;
  double re = 0.0, im = 0.0;
  for (int64_t j = 0; j < m; ++j) {
    const double2 g = G[(int64_t)k * m + j];
    re += g.x * c[j];
    im += g.y * c[j];
  }
  r[k] = make_double2(re - d[k].x, im - d[k].y);
}

// grad[j] += Re(sum_k conj(G[k][j]) r[k]) / s2; quad = sum_k |r_k|^2 / s2 (block 0)
__global__ void k_dense_grad(const double2 *__restrict__ G, const double2 *__restrict__ r,
                             int n_r, int64_t m, double inv_s2, double *__restrict__ grad,
                             double *__restrict__ quad) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < m) {
    double s = 0.0;
    for (int k = 0; k < n_r; ++k) {
      const double2 g = G[(int64_t)k * m + j];
      s += g.x * r[k].x + g.y * r[k].y;
    }
    grad[j] += s * inv_s2;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double q = 0.0;
    for (int k = 0; k < n_r; ++k) q += r[k].x * r[k].x + r[k].y * r[k].y;
    *quad = q * inv_s2;
  }
}

// y = gram z, one warp per row, fp64 (the seam's matrix is a host float64 array)
__global__ void __launch_bounds__(256)
k_gemv64(const double *__restrict__ gram, int64_t m, const double *__restrict__ z,
         double *__restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= m) return;
  const double *g = gram + row * m;
  double s = 0.0;
  for (int64_t j = lane; j < m; j += 32) s = fma(g[j], z[j], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] = s;
}

// kernels.py:46-52: g = y - corr; u = z - tau g; c = sign(u) max(|u| - thresh, 0);
// z = c + w (c - c_prev); c_prev = c
__global__ void k_seam_step(const double *__restrict__ y, const double *__restrict__ corr,
                            int64_t m, double tau, double thresh, double w,
                            double *__restrict__ z, double *__restrict__ cprev) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const double u = z[j] - tau * (y[j] - corr[j]);
  const double au = fabs(u) - thresh;
  const double c = au > 0.0 ? copysign(au, u) : 0.0;
  z[j] = c + w * (c - cprev[j]);
  cprev[j] = c;
}

sf_status launch_seam_fista64(const double *gram, const double *corr, int64_t m, double tau,
                              double thresh, const double *w, int steps, double *z, double *cprev,
                              double *y, cudaStream_t st) {
  for (int k = 0; k < steps; ++k) {
    k_gemv64<<<(unsigned)((m * 32 + 255) / 256), 256, 0, st>>>(gram, m, z, y);
    SF_LAUNCH_CHECK();
    k_seam_step<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(y, corr, m, tau, thresh, w[k], z,
                                                            cprev);
    SF_LAUNCH_CHECK();
  }
  return SF_OK;
}

sf_status launch_herk_c64(const double2 *G, int n_r, int64_t m, double inv_s2, double2 *A,
                          cudaStream_t st) {
  const int64_t nb = (m + 31) / 32;
  k_herk_c64<<<(unsigned)(nb * (nb + 1) / 2), 256, 0, st>>>(G, n_r, m, inv_s2, A);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_kgram_c64(const double2 *G, int64_t m, int n_r, double inv_s2, int nsplit,
                           double2 *Kpart, cudaStream_t st) {
  const int nb = (n_r + 31) / 32;
  const int64_t per = ((m + nsplit - 1) / nsplit + 31) / 32 * 32;
  k_kgram_c64<<<dim3(nb * nb, nsplit), 256, 0, st>>>(G, m, n_r, inv_s2, per, Kpart);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_pack_re(const double2 *A, int64_t m, const int2 *tiles, int64_t n_tiles,
                         float *T, cudaStream_t st) {
  if (n_tiles == 0) return SF_OK;
  k_pack_re<<<(unsigned)n_tiles, 256, 0, st>>>(A, m, tiles, T);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_dense_residual(const double2 *G, const double2 *d, int n_r, int64_t m,
                                const double *c, double inv_s2, double2 *r, double *grad,
                                double *quad, cudaStream_t st) {
  k_dense_residual<<<(n_r + 127) / 128, 128, 0, st>>>(G, d, n_r, m, c, r);
  SF_LAUNCH_CHECK();
  k_dense_grad<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(G, r, n_r, m, inv_s2, grad, quad);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

}  // namespace sf
