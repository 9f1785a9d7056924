// sf_misc.cu -- image synthesis, proximal map, dense helpers for the seam API.
//
//   k_reconstruct     image = H c via the pixel-major (CSR) transpose of the
//                     ELL dictionary; fixed summation order, no atomics.
//                     solver.py:294-299, dictionary.py:160-166
//   k_soft_threshold  solver.py:229-240
//   k_zgemv           dense complex matvec for hermitian_top_eigenvalue on a
//                     caller-supplied matrix (solver.py:139-175)
//   k_compose_dense   compose(F, H) with H as ELL (dictionary.py:151-157)
//   k_metrics_*       per-pulse reconstruction metrics (metrics.py:31-56,
//                     harness.py:288-318): image = H c, mean magnitudes of the
//                     image and the BP image on / off the truth mask, the
//                     squared residual to the truth, count(|c| > threshold)
#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {

__global__ void k_reconstruct(const int64_t *__restrict__ ptr, const int32_t *__restrict__ atom,
                              const double *__restrict__ w, int64_t n,
                              const double *__restrict__ c, double *__restrict__ img) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  double s = 0.0;
  for (int64_t k = ptr[p]; k < ptr[p + 1]; ++k) s += w[k] * c[atom[k]];
  img[p] = s;
}

// sign/phase-preserving shrinkage: 0 if |u| <= alpha else u (1 - alpha/|u|)
__global__ void k_soft_threshold(const double *__restrict__ u, int64_t n, int is_complex,
                                 double alpha, double *__restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (is_complex) {
    const double re = u[2 * i], im = u[2 * i + 1];
    const double mag = hypot(re, im);
    const double keep = fmax(mag - alpha, 0.0);
    const double scale = mag > 0.0 ? keep / mag : 0.0;
    out[2 * i] = re * scale;
    out[2 * i + 1] = im * scale;
  } else {
    const double x = u[i];
    const double mag = fabs(x);
    const double keep = fmax(mag - alpha, 0.0);
    const double scale = mag > 0.0 ? keep / mag : 0.0;
    out[i] = x * scale;
  }
}

// w = X v, X [n][n] complex row-major; one warp per row, fixed shuffle tree.
__global__ void k_zgemv(const double2 *__restrict__ X, int64_t n, const double2 *__restrict__ v,
                        double2 *__restrict__ w) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (row >= n) return;
  double re = 0.0, im = 0.0;
  for (int64_t c = lane; c < n; c += 32) {
    const double2 x = X[row * n + c], y = v[c];
    re += x.x * y.x - x.y * y.y;
    im += x.x * y.y + x.y * y.x;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    re += __shfl_xor_sync(0xffffffffu, re, o);
    im += __shfl_xor_sync(0xffffffffu, im, o);
  }
  if (lane == 0) w[row] = make_double2(re, im);
}

// G[m][j] = sum_l w_jl F[m][idx_jl]
__global__ void k_compose_dense(const double2 *__restrict__ F, int n_r, int64_t n,
                                const int32_t *__restrict__ idx, const double *__restrict__ wt,
                                int64_t m, int width, double2 *__restrict__ G) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m * n_r) return;
  const int row = (int)(e / m);
  const int64_t j = e - (int64_t)row * m;
  double re = 0.0, im = 0.0;
  for (int l = 0; l < width; ++l) {
    const int32_t p = idx[j * width + l];
    if (p < 0) break;
    const double2 f = F[(int64_t)row * n + p];
    re += wt[j * width + l] * f.x;
    im += wt[j * width + l] * f.y;
  }
  G[e] = make_double2(re, im);
}

sf_status launch_reconstruct(const int64_t *csr_ptr, const int32_t *csr_atom, const double *csr_w,
                             int64_t n_pixels, const double *c, double *img, cudaStream_t st) {
  const int bs = 256;
  k_reconstruct<<<(unsigned)((n_pixels + bs - 1) / bs), bs, 0, st>>>(csr_ptr, csr_atom, csr_w,
                                                                    n_pixels, c, img);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_soft_threshold(const double *u, int64_t n, int is_complex, double alpha,
                                double *out, cudaStream_t st) {
  if (n == 0) return SF_OK;
  const int bs = 256;
  k_soft_threshold<<<(unsigned)((n + bs - 1) / bs), bs, 0, st>>>(u, n, is_complex, alpha, out);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_zgemv(const double2 *X, int64_t n, const double2 *v, double2 *w, cudaStream_t st) {
  const int64_t threads = n * 32;
  const int bs = 256;
  k_zgemv<<<(unsigned)((threads + bs - 1) / bs), bs, 0, st>>>(X, n, v, w);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_compose_ell_dense(const double2 *F, int n_r, int64_t n, const int32_t *ell_idx,
                                   const double *ell_w, int64_t m, int ell_width, double2 *G,
                                   cudaStream_t st) {
  const int64_t tot = m * n_r;
  if (tot == 0) return SF_OK;
  const int bs = 256;
  k_compose_dense<<<(unsigned)((tot + bs - 1) / bs), bs, 0, st>>>(F, n_r, n, ell_idx, ell_w, m,
                                                                  ell_width, G);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

// ---- per-pulse metrics -----------------------------------------------------------
// Eight sums per block in a fixed order (grid-stride, warp shuffle tree, then
// the 8 warps in order), then one block adds the block partials in order:
// {n_large, |img| on, |img| off, |bp| on, |bp| off, |img - truth|^2, n_on, n_off}.
constexpr int kMetricBlocks = 256;
__global__ void __launch_bounds__(256)
k_metrics_partial(const int64_t *__restrict__ ptr, const int32_t *__restrict__ atom,
                  const double *__restrict__ w, int64_t n, const double *__restrict__ c,
                  int64_t m, const uint8_t *__restrict__ mask, const double2 *__restrict__ truth,
                  const double2 *__restrict__ bp, double inv_count, double threshold,
                  double *__restrict__ part) {
  double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < m; j += stride)
    acc[0] += fabs(c[j]) > threshold ? 1.0 : 0.0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += stride) {
    double img = 0.0;
    for (int64_t k = ptr[p]; k < ptr[p + 1]; ++k) img += w[k] * c[atom[k]];
    const bool on = mask[p] != 0;
    const double a = fabs(img);
    const double b = bp ? hypot(bp[p].x, bp[p].y) * inv_count : 0.0;
    acc[on ? 1 : 2] += a;
    acc[on ? 3 : 4] += b;
    if (truth) {
      const double dr = img - truth[p].x, di = truth[p].y;
      acc[5] += dr * dr + di * di;
    } else {
      acc[5] += img * img;
    }
    acc[on ? 6 : 7] += 1.0;
  }
  __shared__ double red[8][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    double v = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < 8) {
    double v = 0.0;
    for (int k = 0; k < 8; ++k) v += red[k][threadIdx.x];
    part[blockIdx.x * 8 + threadIdx.x] = v;
  }
}
__global__ void k_metrics_final(const double *__restrict__ part, int nblk, double *__restrict__ out) {
  if (threadIdx.x < 8) {
    double v = 0.0;
    for (int b = 0; b < nblk; ++b) v += part[b * 8 + threadIdx.x];
    out[threadIdx.x] = v;
  }
}

sf_status launch_pulse_metrics(const int64_t *csr_ptr, const int32_t *csr_atom,
                               const double *csr_w, int64_t n, const double *c, int64_t m,
                               const uint8_t *mask, const double2 *truth, const double2 *bp,
                               double inv_count, double threshold, double *scratch, double *out,
                               cudaStream_t st) {
  k_metrics_partial<<<kMetricBlocks, 256, 0, st>>>(csr_ptr, csr_atom, csr_w, n, c, m, mask, truth,
                                                   bp, inv_count, threshold, scratch);
  SF_LAUNCH_CHECK();
  k_metrics_final<<<1, 32, 0, st>>>(scratch, kMetricBlocks, out);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

}  // namespace sf
