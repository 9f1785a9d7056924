// sf_batch.cu -- the step-size bound of the batch oracle on the device.
//
// Reference: solver.batch_fista (solver.py:267-291) sums every retained
// pulse's increments into one Hermitian A = sum_k G_k^H G_k / sigma_k^2 and
// takes L = hermitian_top_eigenvalue(A) (solver.py:139-175, power iteration
// from counter_unit_complex_vector(M)).  The engine keeps only Re(B) in pixel
// space, so the power iteration runs matrix-free in M space with the exact
// operator of the reference:
//
//   A v = H^T ( sum_k F_k^H F_k (H v) / sigma_k^2 )          (H real)
//
// per iteration: x = H v (CSR), y_k = F_k x (one CTA per (frequency, pulse),
// the simulator kernel), z = sum_k F_k^H y_k / sigma_k^2 (one thread per
// pixel, phases recomputed exactly as k_pixel_delays / k_delay_phase form
// them), w = H^T z (ELL), then lambda = Re(v^H w), |w|, v <- w / |w| with the
// reference's stopping rule, tail bias and non-convergence result.
#include <math.h>

#include <string>
#include <vector>

#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {

__global__ void __launch_bounds__(256)
k_adjoint_all(const double *__restrict__ omega, int n_r, const double *__restrict__ gammas,
              const double *__restrict__ inv_s2, int n_pulses, const double *__restrict__ xyz,
              int64_t n, const double2 *__restrict__ y, double2 *__restrict__ z) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  const double px = xyz[3 * p], py = xyz[3 * p + 1], pz = xyz[3 * p + 2];
  double re = 0.0, im = 0.0;
  for (int k = 0; k < n_pulses; ++k) {
    const double dx = __dsub_rn(px, gammas[3 * k]);
    const double dy = __dsub_rn(py, gammas[3 * k + 1]);
    const double dz = __dsub_rn(pz, gammas[3 * k + 2]);
    const double tau = __dmul_rn(
        2.0 / kSpeedOfLight,
        __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz))));
    double sr = 0.0, si = 0.0;
    for (int m = 0; m < n_r; ++m) {
      double s, c;
      sincos(__dmul_rn(omega[m], tau), &s, &c);
      const double2 v = y[(int64_t)k * n_r + m];
      // conj(F) y = (c + j s)(v.x + j v.y)
      sr += c * v.x - s * v.y;
      si += c * v.y + s * v.x;
    }
    re += inv_s2[k] * sr;
    im += inv_s2[k] * si;
  }
  z[p] = make_double2(re, im);
}

// out = {Re(v^H w), |w|^2} in a fixed order (one block)
__global__ void __launch_bounds__(1024)
k_dot_norm(const double2 *__restrict__ v, const double2 *__restrict__ w, int64_t m,
           double *__restrict__ out) {
  __shared__ double r1[32], r2[32];
  double a = 0.0, b = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
    const double2 x = v[i], y = w[i];
    a += x.x * y.x + x.y * y.y;
    b += y.x * y.x + y.y * y.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    r1[warp] = a;
    r2[warp] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      sa += r1[i];
      sb += r2[i];
    }
    out[0] = sa;
    out[1] = sb;
  }
}

__global__ void k_scale_div(const double2 *__restrict__ w, int64_t m, double norm,
                            double2 *__restrict__ v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < m) v[i] = make_double2(__ddiv_rn(w[i].x, norm), __ddiv_rn(w[i].y, norm));
}

sf_status batch_lipschitz(const BatchLipArgs &a, double rel_tol, int max_iter, double *lam_out,
                          int *converged, cudaStream_t st) {
  const int64_t m = a.m, n = a.n;
  double2 *v = a.work, *w = v + m, *x = w + m, *z = x + n;
  double2 *y = z + n;  // [P][n_r]
  double *red = reinterpret_cast<double *>(y + (int64_t)a.n_pulses * a.n_r);
  SF_CUDA_TRY(cudaMemcpyAsync(v, a.v0, m * sizeof(double2), cudaMemcpyDeviceToDevice, st));
  double lam_prev = 0.0, delta_prev = 0.0;
  bool have_prev = false, have_dprev = false;
  sf_status s;
  const int bs = 256;
  for (int it = 0; it < max_iter; ++it) {
    if ((s = launch_hv0(a.csr_ptr, a.csr_atom, a.csr_w, n, v, x, st))) return s;
    if ((s = launch_simulate_echo(a.omega, a.n_r, a.gammas, a.n_pulses, a.xyz, x, n, y, st)))
      return s;
    k_adjoint_all<<<(unsigned)((n + bs - 1) / bs), bs, 0, st>>>(a.omega, a.n_r, a.gammas, a.inv_s2,
                                                               a.n_pulses, a.xyz, n, y, z);
    SF_LAUNCH_CHECK();
    if ((s = launch_bupdate(a.ell_idx, a.ell_w, a.ell_width, m, z, w, a.bmax_scratch, st))) return s;
    k_dot_norm<<<1, 1024, 0, st>>>(v, w, m, red);
    SF_LAUNCH_CHECK();
    double h[2];
    SF_CUDA_TRY(cudaMemcpyAsync(h, red, sizeof(h), cudaMemcpyDeviceToHost, st));
    SF_CUDA_TRY(cudaStreamSynchronize(st));
    const double lam = h[0], norm_w = sqrt(h[1]);
    if (norm_w == 0.0) {  // solver.py:162-163
      *lam_out = 0.0;
      *converged = 1;
      return SF_OK;
    }
    k_scale_div<<<(unsigned)((m + bs - 1) / bs), bs, 0, st>>>(w, m, norm_w, v);
    SF_LAUNCH_CHECK();
    if (have_prev) {  // solver.py:165-173
      const double delta = lam - lam_prev;
      if (fabs(delta) <= rel_tol * fmax(fabs(lam), 1e-300)) {
        double tail = 0.0;
        if (have_dprev && fabs(delta_prev) > fabs(delta) && fabs(delta) > 0.0) {
          const double q = delta / delta_prev;
          if (q > 0.0 && q < 1.0) tail = delta * q / (1.0 - q);
        }
        *lam_out = lam + tail + fabs(delta);
        *converged = 1;
        return SF_OK;
      }
      delta_prev = delta;
      have_dprev = true;
    }
    lam_prev = lam;
    have_prev = true;
  }
  *lam_out = have_prev ? lam_prev : 0.0;  // solver.py:175
  *converged = 0;
  return SF_OK;
}

}  // namespace sf
