// sf_geom.cu -- per-pulse operator synthesis, b update and the Lipschitz
// increment, all on the device.
//
//   k_pixel_delays   tau_p = (2/c)|gamma - x_p|          geometry.py:97-104
//   k_forward_t      F[m,p] = exp(-j w_m tau_p)          kernels.py:27-29,66-76
//   k_compose        G~ = F H / sigma (ELL gather), b += G~^H d~, u0 += G~ v0
//                                                          dictionary.py:151-157,
//                                                          solver.py:178-183,191-193
//   k_kgram          K~ = G~ G~^H (N_r x N_r)
//   k_power_cl /     power iteration of solver.py:139-175 re-expressed on K~,
//   k_power_cluster
//                    L += max(inc, 0), Frobenius fallback   solver.py:194-199
//
// G~ is stored "packed": row j (atom) holds [Re G~[:,j] | Im G~[:,j]] as fp32,
// K_pad = round_up(2 N_r, kKChunk) columns, zero padded.  This is the K-major
// operand of the Gram update Re(A) += P^T P (sf_gram.cu).
#include <cooperative_groups.h>
#include <math.h>
#include <stdlib.h>

#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {

// ---------------------------------------------------------------------------
// Round-trip delays.  Mirrors geometry.py:100-104 operation by operation in
// IEEE fp64 without FMA contraction so the delays are bit-identical to numpy:
//   diff = pos - gamma; d = sqrt((dx*dx + dy*dy) + dz*dz); tau = (2/c) * d.
__global__ void k_pixel_delays(const double *__restrict__ xyz, int64_t n,
                               const double *__restrict__ gamma,
                               double *__restrict__ tau,
                               int *__restrict__ zero_flag, int64_t in_stride) {
  int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  gamma += blockIdx.y * in_stride;  // batched scenes: one grid row per scene
  tau += blockIdx.y * n;
  const double gx = gamma[0], gy = gamma[1], gz = gamma[2];
  double dx = __dsub_rn(xyz[3 * p + 0], gx);
  double dy = __dsub_rn(xyz[3 * p + 1], gy);
  double dz = __dsub_rn(xyz[3 * p + 2], gz);
  double s = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                       __dmul_rn(dz, dz));
  double d = __dsqrt_rn(s);
  if (d == 0.0 && zero_flag != nullptr) atomicOr(zero_flag, 1);
  tau[p] = __dmul_rn(2.0 / kSpeedOfLight, d);
}

// F transposed: Ft[p][m] = exp(-j w_m tau_p) = (cos(w tau), -sin(w tau)).
// The argument w*tau (up to ~4e6 rad at 10 km / 10 GHz) is the
// same IEEE product numpy forms; sincos() does a full-precision reduction.
__global__ void k_forward_t(const double *__restrict__ omega, int n_r,
                            const double *__restrict__ tau, int64_t n,
                            double2 *__restrict__ Ft) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n * n_r) return;
  int64_t p = idx / n_r;
  int m = (int)(idx - p * n_r);
  double ph = __dmul_rn(omega[m], tau[p]);
  double s, c;
  sincos(ph, &s, &c);
  Ft[idx] = make_double2(c, -s);
}

// Same phase fill for the engine-less seam (row-major [m][i] like numpy).
__global__ void k_delay_phase(const double *__restrict__ omega, int n_r,
                              const double *__restrict__ tau, int64_t n,
                              double2 *__restrict__ F) {
  int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n * n_r) return;
  int m = (int)(idx / n);
  int64_t p = idx - (int64_t)m * n;
  double ph = __dmul_rn(omega[m], tau[p]);
  double s, c;
  sincos(ph, &s, &c);
  F[idx] = make_double2(c, -s);
}

// ---------------------------------------------------------------------------
// compose + b update + u0 partials.  One warp per atom j (grid-stride over
// atoms with a fixed grid, so every reduction order is fixed), lanes over the
// N_r frequency samples.
//   g_mj = inv_sigma * sum_l w_jl F[m, idx_jl]            (G = F H, / sigma)
//   b_j += sum_m conj(g_mj) * d~_m        d~ = d / sigma  (b += G^H R^-1 d)
//   (dt holds the raw d; it is scaled by inv_sigma on load)
//   u0_m += g_mj * v0_j                  (power-iteration start)
// Dense mode (ell == nullptr): g_mj = inv_sigma * Gd[m][j].
template <int MAXQ>
__global__ void __launch_bounds__(256)
k_compose(const double2 *__restrict__ Ft, const int32_t *__restrict__ ell_idx,
          const double *__restrict__ ell_w, int ell_width,
          const double2 *__restrict__ Gd, int64_t m_atoms, int64_t m_pad,
          int n_r, int k_pad, double inv_sigma,
          const double2 *__restrict__ dt, const double2 *__restrict__ v0,
          float *__restrict__ Gp, double2 *__restrict__ b,
          double2 *__restrict__ u0part, unsigned *__restrict__ maxbits,
          unsigned long long *__restrict__ bmax) {
  __shared__ double2 s_d[512];
  __shared__ double2 s_u0[512];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  for (int m = threadIdx.x; m < n_r; m += blockDim.x) {
    s_d[m] = make_double2(dt[m].x * inv_sigma, dt[m].y * inv_sigma);
    s_u0[m] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  double2 acc[MAXQ];
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) acc[q] = make_double2(0.0, 0.0);

  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp; j < m_pad;
       j += warps_total) {
    float *row = Gp + j * k_pad;
    if (j >= m_atoms) {  // padding atom: zero operator row
      for (int k = lane; k < k_pad; k += 32) row[k] = 0.f;
      continue;
    }
    const double2 vj = v0[j];
    double bre = 0.0, bim = 0.0;
    float amax = 0.f;
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      const int m = lane + 32 * q;
      if (m < n_r) {
        double gr = 0.0, gi = 0.0;
        if (ell_idx != nullptr) {
          for (int l = 0; l < ell_width; ++l) {
            const int32_t p = ell_idx[j * ell_width + l];
            if (p < 0) break;
            const double w = ell_w[j * ell_width + l];
            const double2 f = Ft[(int64_t)p * n_r + m];
            gr += w * f.x;
            gi += w * f.y;
          }
        } else {
          const double2 g = Gd[(int64_t)m * m_atoms + j];
          gr = g.x;
          gi = g.y;
        }
        gr *= inv_sigma;
        gi *= inv_sigma;
        row[m] = (float)gr;
        row[n_r + m] = (float)gi;
        amax = fmaxf(amax, fmaxf(fabsf((float)gr), fabsf((float)gi)));
        const double2 dm = s_d[m];
        // conj(g) * d
        bre += gr * dm.x + gi * dm.y;
        bim += gr * dm.y - gi * dm.x;
        // g * v0_j
        acc[q].x += gr * vj.x - gi * vj.y;
        acc[q].y += gr * vj.y + gi * vj.x;
      }
    }
    for (int k = 2 * n_r + lane; k < k_pad; k += 32) row[k] = 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      bre += __shfl_xor_sync(0xffffffffu, bre, o);
      bim += __shfl_xor_sync(0xffffffffu, bim, o);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    if (lane == 0) {
      double2 bj = b[j];
      bj.x += bre;
      bj.y += bim;
      b[j] = bj;
      if (maxbits != nullptr) atomicMax(maxbits, __float_as_uint(amax));
      // running max_j |b_j| for the lambda rule (order-free, so deterministic)
      if (bmax != nullptr)
        atomicMax(bmax, (unsigned long long)__double_as_longlong(hypot(bj.x, bj.y)));
    }
  }
  // Fixed-order reduction of the per-lane u0 partials across the CTA's warps.
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    if (warp == w) {
#pragma unroll
      for (int q = 0; q < MAXQ; ++q) {
        const int m = lane + 32 * q;
        if (m < n_r) {
          s_u0[m].x += acc[q].x;
          s_u0[m].y += acc[q].y;
        }
      }
    }
    __syncthreads();
  }
  for (int m = threadIdx.x; m < n_r; m += blockDim.x)
    u0part[(int64_t)blockIdx.x * n_r + m] = s_u0[m];
}

// ---------------------------------------------------------------------------
// K~ partials: Kpart[s][m1][m2] = sum_{j in split s} g_m1j conj(g_m2j).
// 32x32 output block per CTA, 256 threads, 4 outputs each; 32-atom chunks
// staged through shared memory; fp32 products within a chunk, fp64 across.
__global__ void __launch_bounds__(256)
k_kgram(const float *__restrict__ Gp, int64_t m_atoms, int n_r, int k_pad,
        int64_t atoms_per_split, double2 *__restrict__ Kpart) {
  __shared__ float2 s1[32][33];
  __shared__ float2 s2[32][33];
  const int nb = (n_r + 31) / 32;
  const int m1b = blockIdx.x / nb, m2b = blockIdx.x % nb;
  const int split = blockIdx.y;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t j0 = (int64_t)split * atoms_per_split;
  const int64_t j1 = min(m_atoms, j0 + atoms_per_split);
  double accr[4] = {0, 0, 0, 0}, acci[4] = {0, 0, 0, 0};
  for (int64_t jc = j0; jc < j1; jc += 32) {
    // load 32 atoms x 32 samples for both blocks
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
      const int jj = e >> 5, mm = e & 31;
      const int64_t j = jc + jj;
      float2 v1 = make_float2(0.f, 0.f), v2 = make_float2(0.f, 0.f);
      if (j < j1) {
        const float *row = Gp + j * k_pad;
        const int a = m1b * 32 + mm, c = m2b * 32 + mm;
        if (a < n_r) v1 = make_float2(row[a], row[n_r + a]);
        if (c < n_r) v2 = make_float2(row[c], row[n_r + c]);
      }
      s1[jj][mm] = v1;
      s2[jj][mm] = v2;
    }
    __syncthreads();
    float pr[4] = {0, 0, 0, 0}, pi[4] = {0, 0, 0, 0};
#pragma unroll 8
    for (int jj = 0; jj < 32; ++jj) {
      const float2 c2 = s2[jj][tx];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 a = s1[jj][ty + 8 * i];
        // a * conj(c2)
        pr[i] += a.x * c2.x + a.y * c2.y;
        pi[i] += a.y * c2.x - a.x * c2.y;
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      accr[i] += pr[i];
      acci[i] += pi[i];
    }
    __syncthreads();
  }
  const int c = m2b * 32 + tx;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int a = m1b * 32 + ty + 8 * i;
    if (a < n_r && c < n_r)
      Kpart[((int64_t)split * n_r + a) * n_r + c] = make_double2(accr[i], acci[i]);
  }
}

// ---------------------------------------------------------------------------
// Pixel-space Lipschitz operator (geometric pulses).  With Q = H H^T (static,
// sparse, pixel x pixel) the N_r x N_r matrix of the power iteration is
//   K~ = G~ G~^H = F Q F^H / sigma^2,
// a reduction over N pixels instead of M atoms, evaluated in fp64 from the
// fp64 F (tighter than the fp32 G~ the Gram update consumes).
//   k_fq:       W[p][m] = sum_{p'} Q[p][p'] Ft[p'][m]          (CSR rows of Q)
//   k_kgram_px: Kpart[s][m1][m2] = sum_{p in split s} Ft[p][m1] conj(W[p][m2])
//               on the upper 32x32 blocks; k_kreduce mirrors and scales.
__global__ void k_fq(const int64_t *__restrict__ qptr, const int32_t *__restrict__ qcol,
                     const double *__restrict__ qval, const double2 *__restrict__ Ft, int64_t n,
                     int n_r, double2 *__restrict__ W) {
  Ft += blockIdx.y * n * n_r;
  W += blockIdx.y * n * n_r;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * n_r;
       idx += (int64_t)gridDim.x * blockDim.x) {
  const int64_t p = idx / n_r;
  const int m = (int)(idx - p * n_r);
  double re = 0.0, im = 0.0;
  const int64_t k0 = qptr[p], k1 = qptr[p + 1];
  int64_t k = k0;
  // four nonzeros' loads in flight, accumulated in the same (row) order
  for (; k + 4 <= k1; k += 4) {
    double q[4];
    double2 f[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      q[u] = qval[k + u];
      f[u] = Ft[(int64_t)qcol[k + u] * n_r + m];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      re += q[u] * f[u].x;
      im += q[u] * f[u].y;
    }
  }
  for (; k < k1; ++k) {
    const double q = qval[k];
    const double2 f = Ft[(int64_t)qcol[k] * n_r + m];
    re += q * f.x;
    im += q * f.y;
  }
  W[idx] = make_double2(re, im);
  }
}

__global__ void __launch_bounds__(256)
k_kgram_px(const double2 *__restrict__ Ft, const double2 *__restrict__ W, int64_t n, int n_r,
           int64_t px_per_split, double2 *__restrict__ Kpart) {
  __shared__ double2 s1[32][33];
  __shared__ double2 s2[32][33];
  const int nb = (n_r + 31) / 32;
  // blockIdx.x enumerates upper block pairs (m1b <= m2b) row-major
  int rem = blockIdx.x, m1b = 0;
  while (rem >= nb - m1b) {
    rem -= nb - m1b;
    ++m1b;
  }
  const int m2b = m1b + rem;
  const int split = blockIdx.y;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  Ft += blockIdx.z * n * n_r;  // batched scenes: grid z
  W += blockIdx.z * n * n_r;
  Kpart += blockIdx.z * gridDim.y * (int64_t)n_r * n_r;
  const int64_t p0 = (int64_t)split * px_per_split;
  const int64_t p1 = min(n, p0 + px_per_split);
  double accr[4] = {0, 0, 0, 0}, acci[4] = {0, 0, 0, 0};
  for (int64_t pc = p0; pc < p1; pc += 32) {
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
      const int pp = e >> 5, mm = e & 31;
      const int64_t p = pc + pp;
      double2 v1 = make_double2(0.0, 0.0), v2 = make_double2(0.0, 0.0);
      if (p < p1) {
        const int a = m1b * 32 + mm, c = m2b * 32 + mm;
        if (a < n_r) v1 = Ft[p * n_r + a];
        if (c < n_r) v2 = W[p * n_r + c];
      }
      s1[pp][mm] = v1;
      s2[pp][mm] = v2;
    }
    __syncthreads();
#pragma unroll 4
    for (int pp = 0; pp < 32; ++pp) {
      const double2 w = s2[pp][tx];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double2 f = s1[pp][ty + 8 * i];
        accr[i] += f.x * w.x + f.y * w.y;  // f * conj(w)
        acci[i] += f.y * w.x - f.x * w.y;
      }
    }
    __syncthreads();
  }
  const int c = m2b * 32 + tx;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int a = m1b * 32 + ty + 8 * i;
    if (a < n_r && c < n_r)
      Kpart[((int64_t)split * n_r + a) * n_r + c] = make_double2(accr[i], acci[i]);
  }
}

// K~ = scale * sum_s Kpart[s] (fixed order), mirrored from the upper blocks
// when upper_only; u0 = sum_c u0part[c]; Kf = fp32 copy of K~.
__global__ void k_kreduce(const double2 *__restrict__ Kpart, int nsplit,
                          const double2 *__restrict__ u0part, int nu0,
                          int n_r, int upper_only, double scale_arg, double2 *__restrict__ K,
                          float2 *__restrict__ Kf, double2 *__restrict__ u0,
                          const double *__restrict__ sig, int64_t in_stride) {
  __shared__ double2 red[8][33];
  {  // batched scenes: grid y
    const int64_t sc = blockIdx.y;
    Kpart += sc * nsplit * (int64_t)n_r * n_r;
    u0part += sc * nu0 * (int64_t)n_r;
    K += sc * (int64_t)n_r * n_r;
    Kf += sc * (int64_t)n_r * n_r;
    u0 += sc * n_r;
    if (sig) sig += sc * in_stride;
  }
  const double scale = sig ? sig[0] * sig[0] : scale_arg;  // 1/sigma^2 from the device scalars
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t idx = blockIdx.x * 32LL + tx;
  const int64_t nn = (int64_t)n_r * n_r;
  const int a = (int)(idx / n_r), c = (int)(idx % n_r);
  const bool mirror = upper_only && (a / 32 > c / 32);
  double2 s = make_double2(0.0, 0.0);
  if (idx < nn) {
    const int64_t src = mirror ? (int64_t)c * n_r + a : idx;
    for (int k = ty; k < nsplit; k += 8) {
      const double2 v = Kpart[(int64_t)k * nn + src];
      s.x += v.x;
      s.y += v.y;
    }
  }
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && idx < nn) {
    double2 t = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      t.x += red[k][tx].x;
      t.y += red[k][tx].y;
    }
    t.x *= scale;
    t.y *= scale;
    if (mirror) t.y = -t.y;
    K[idx] = t;
    Kf[idx] = make_float2((float)t.x, (float)t.y);
  }
  // u0 = sum_c u0part[c]: the blocks past the K~ range, 32 entries x 8 lanes each
  const int64_t kblocks = (nn + 31) / 32;
  if (blockIdx.x >= kblocks) {
    const int64_t m = (blockIdx.x - kblocks) * 32LL + tx;
    double2 su = make_double2(0.0, 0.0);
    if (m < n_r)
      for (int cc = ty; cc < nu0; cc += 8) {
        const double2 v = u0part[(int64_t)cc * n_r + m];
        su.x += v.x;
        su.y += v.y;
      }
    __syncthreads();
    red[ty][tx] = su;
    __syncthreads();
    if (ty == 0 && m < n_r) {
      double2 t = make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        t.x += red[k][tx].x;
        t.y += red[k][tx].y;
      }
      u0[m] = t;
    }
  }
}

// ---------------------------------------------------------------------------
// Block-wide fp64 sum with a fixed reduction tree (1024 threads max).
__device__ double block_sum(double v, double *red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  double t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.0;
  if (warp == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// Power iteration of solver.py:139-175 in N_r space:
//   u_k = G~ v_k, lam_k = |u_k|^2, |X v_k| = sqrt(u_k^H K~ u_k),
//   u_{k+1} = K~ u_k / |X v_k|.
// Identical iterate sequence, stopping rule |dlam| <= tol*max(|lam|,1e-300),
// geometric-tail bias (solver.py:166-172) and non-convergence result
// (solver.py:175).  Then accumulate()'s L update with the Frobenius fallback
// (solver.py:194-205): |dA|_F = |K~|_F.  Two kernels: k_power_cl (N_r <= 256,
// K~ fp64 across a cluster of up to 8 CTAs) and k_power_cluster (N_r <= 512).

// Reduce-scatter of V per-lane values over the 32 lanes of a warp.
template <int V>
__device__ __forceinline__ double butterfly_sum(double (&v)[V], int lane, int &idx) {
  // reduce-scatter V values over 32 lanes; returns this lane's value, idx its index
  idx = 0;
  int n = V;
#pragma unroll
  for (int off = 16; off >= 1; off >>= 1) {
    if (n > 1) {
      const int half = n >> 1;
      const bool up = lane & off;
#pragma unroll
      for (int k = 0; k < V / 2; ++k) {
        if (k < half) {
          const double send = up ? v[k] : v[k + half];
          const double keep = up ? v[k + half] : v[k];
          v[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      if (up) idx += half;
      n = half;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
    }
  }
  return v[0];
}

// ---------------------------------------------------------------------------
// Cluster power iteration (any N_r <= 512): the same sequence and stopping
// rule as above (solver.py:139-175 in N_r space), with the matvec rows
// spread over a thread-block cluster of PC CTAs (8, or 16 for N_r > 256).
// CTA r owns RL = 8*RW rows of K~ (fp32, dynamic shared memory); each
// iteration every CTA pushes its slice of w = K~ u and its partial Re(u^H w)
// into all CTAs' shared memory (DSMEM), then one cluster barrier; w is
// double-buffered so that is the only barrier.  All CTAs sum the same partials
// in the same order, so every thread takes the same decisions.  fp64
// arithmetic throughout.
namespace cgc = cooperative_groups;
constexpr int kPCMax = 16;

template <int RW, int C>
__global__ void __launch_bounds__(256, 1)
k_power_cluster(const double2 *__restrict__ K, const float2 *__restrict__ Kf,
                const double2 *__restrict__ u0, int n_r, double rel_tol, int max_iter,
                double *__restrict__ L, long long *__restrict__ counters,
                double *__restrict__ diag, int apply) {
  constexpr int RL = RW * 8;  // rows per CTA
  extern __shared__ __align__(16) unsigned char pc_smem[];
  float2 *sK = reinterpret_cast<float2 *>(pc_smem);  // RL x n_r
  __shared__ double2 sw[2][512];
  __shared__ double snw[2][kPCMax * 8];
  __shared__ double sfro[kPCMax * 8];
  cgc::cluster_group cluster = cgc::this_cluster();
  const int PC = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row0 = rank * RL;
  for (int e = tid; e < RL * n_r; e += 256) {
    const int r = e / n_r, c = e % n_r;
    sK[r * n_r + c] = (row0 + r < n_r) ? Kf[(int64_t)(row0 + r) * n_r + c] : make_float2(0.f, 0.f);
  }
  for (int m = tid; m < 512; m += 256) sw[1][m] = (m < n_r) ? u0[m] : make_double2(0.0, 0.0);
  double fro = 0.0;
  for (int e = tid; e < RL * n_r; e += 256) {
    const int r = row0 + e / n_r;
    if (r < n_r) {
      const double2 v = K[(int64_t)r * n_r + e % n_r];
      fro += v.x * v.x + v.y * v.y;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
  cluster.sync();  // every CTA of the cluster is running before the first remote store
  if (lane == 0)
    for (int q = 0; q < PC; ++q) cluster.map_shared_rank(&sfro[0], q)[rank * 8 + warp] = fro;
  cluster.sync();
  fro = 0.0;
  for (int i = 0; i < PC * 8; ++i) fro += sfro[i];
  fro = sqrt(fro);

  double scale = 1.0;
  double lam_prev = 0.0, delta_prev = 0.0, result = 0.0;
  bool have_prev = false, have_dprev = false;
  int converged = 0, iters = 0;
  for (int it = 0; it < max_iter; ++it) {
    const int src = (it + 1) & 1, dst = it & 1;
    double2 uc[C];
    double unorm = 0.0;
#pragma unroll
    for (int i = 0; i < C; ++i) {
      const int c = lane + 32 * i;
      const double2 x = (c < n_r) ? sw[src][c] : make_double2(0.0, 0.0);
      uc[i] = make_double2(x.x * scale, x.y * scale);
      unorm += uc[i].x * uc[i].x + uc[i].y * uc[i].y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) unorm += __shfl_xor_sync(0xffffffffu, unorm, o);
    const double lam = unorm;
    double v[2 * RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      const int lr = warp * RW + r;  // local row
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int i = 0; i < C; ++i) {
        const int c = lane + 32 * i;
        if (c < n_r) {
          const float2 k = sK[lr * n_r + c];
          re += (double)k.x * uc[i].x - (double)k.y * uc[i].y;
          im += (double)k.x * uc[i].y + (double)k.y * uc[i].x;
        }
      }
      v[2 * r] = re;
      v[2 * r + 1] = im;
    }
    int idx;
    const double mine = butterfly_sum<2 * RW>(v, lane, idx);
    const int row = row0 + warp * RW + (idx >> 1);
    double part = 0.0;
    if ((lane & ((32 / (2 * RW)) - 1)) == 0 && row < n_r) {
      const double2 uu = sw[src][row];
      part = (idx & 1) ? uu.y * scale * mine : uu.x * scale * mine;
      for (int q = 0; q < PC; ++q) {
        double *dstp = reinterpret_cast<double *>(cluster.map_shared_rank(&sw[dst][row], q));
        dstp[idx & 1] = mine;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane < PC) cluster.map_shared_rank(&snw[dst][0], lane)[rank * 8 + warp] = part;
    cluster.sync();
    double nw2 = 0.0;
    for (int i = 0; i < PC * 8; ++i) nw2 += snw[dst][i];
    const double norm_w = sqrt(fmax(nw2, 0.0));
    iters = it + 1;
    if (norm_w == 0.0) {
      result = 0.0;
      converged = 1;
      break;
    }
    scale = 1.0 / norm_w;
    if (have_prev) {
      const double delta = lam - lam_prev;
      if (fabs(delta) <= rel_tol * fmax(fabs(lam), 1e-300)) {
        double tail = 0.0;
        if (have_dprev && fabs(delta_prev) > fabs(delta) && fabs(delta) > 0.0) {
          const double q = delta / delta_prev;
          if (q > 0.0 && q < 1.0) tail = delta * q / (1.0 - q);
        }
        result = lam + tail + fabs(delta);
        converged = 1;
        break;
      }
      delta_prev = delta;
      have_dprev = true;
    }
    lam_prev = lam;
    have_prev = true;
  }
  if (!converged) result = have_prev ? lam_prev : 0.0;
  if (rank == 0 && tid == 0) {
    double inc = result;
    if (apply) {
      if (!converged) {
        inc = fro;
        counters[1] += 1;
      }
      L[0] += fmax(inc, 0.0);
      counters[0] += 1;
    }
    diag[0] = result;
    diag[1] = (double)iters;
    diag[2] = (double)converged;
    diag[3] = fro;
  }
  cluster.sync();  // no CTA may exit while peers can still write its shared memory
}

template <int RW, int C>
static sf_status launch_power_cluster(int pc, const double2 *K, const float2 *Kf,
                                      const double2 *u0, int n_r, double rel_tol, int max_iter,
                                      double *L, long long *counters, double *diag, int apply,
                                      cudaStream_t st) {
  const size_t dyn = (size_t)RW * 8 * n_r * sizeof(float2);
  static std::atomic<uint64_t> set{0};
  if (attr_pending(set)) {
    SF_CUDA_TRY(cudaFuncSetAttribute(k_power_cluster<RW, C>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    SF_CUDA_TRY(cudaFuncSetAttribute(k_power_cluster<RW, C>,
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_done(set);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pc);
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = pc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  count_launch();
  SF_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_power_cluster<RW, C>, K, Kf, u0, n_r, rel_tol, max_iter,
                                 L, counters, diag, apply));
  return SF_OK;
}

// ---------------------------------------------------------------------------
// Cluster power iteration, latency-optimised (N_r <= 256; the default).
// Same iterate sequence and stopping rule as solver.py:139-175 in N_r space.
// K~ stays fp64 in distributed shared memory: the cluster's PC CTAs own
// RL = 4*NW consecutive rows each (PC * RL = NP = 32*C padded rows), warp w of
// a CTA owns 4 rows, lane l the columns l + 32 i.  Per iteration:
//   s_k  = stored vector (u_k = a_k s_k, a_k = 1/|X v_{k-1}|, a_0 = 1)
//   w_k  = a_k K~ s_k                         (4 rows per warp, fp64 FMA)
//   part = Re(u_k^H w_k) = a_k Re(s_k^H w_k),  wsq = |w_k|^2
// each warp pushes its w rows and (part, wsq) into every CTA's shared memory,
// one cluster barrier, then every warp reduces the PC*NW (part, wsq) pairs
// with the same xor butterfly (identical bits everywhere), so
//   |X v_k| = sqrt(sum part),  s_{k+1} = w_k,  a_{k+1} = 1/|X v_k|,
//   lam_{k+1} = |u_{k+1}|^2 = sum wsq * a_{k+1}^2.
// The scale is applied to the matvec OUTPUT, so the next matvec starts right
// after the barrier, off the sqrt/divide chain; one barrier per iteration.
// DSMEM push with transaction accounting: 16 bytes into CTA `rank`'s copy of
// `local`, completing 16 bytes of tx on that CTA's copy of `bar`.
__device__ __forceinline__ void st_async_d2(const void *local, const uint64_t *bar, int rank,
                                            double a, double b) {
  const uint32_t la = (uint32_t)__cvta_generic_to_shared(local);
  const uint32_t lb = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t ra, rb;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(la), "r"(rank));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(rb) : "r"(lb), "r"(rank));
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(ra),
               "d"(a), "d"(b), "r"(rb)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}

// Single-CTA N_r <= 64 variant (C = 2, NW = 16): two CTAs per SM (<= 64
// registers) so a batch of scenes (cfg2: one CTA per scene) runs twice as many
// power iterations at once.
template <int C, int NW, int V>
__global__ void __launch_bounds__(32 * NW, (C == 2 && NW == 16) ? 2 : 1)
k_power_cl(const double2 *__restrict__ K, const double2 *__restrict__ u0, int n_r,
           double rel_tol, int max_iter, double *__restrict__ L, long long *__restrict__ counters,
           double *__restrict__ diag, int apply) {
  constexpr int NP = 32 * C, RL = 4 * NW, PC = NP / RL, NT = 32 * NW;
  static_assert(PC * NW <= 64, "partials exceed one pair of lanes");
  extern __shared__ __align__(16) unsigned char pl_smem[];
  double2 *sK = reinterpret_cast<double2 *>(pl_smem);  // RL x NP
  __shared__ double2 sw[2][NP];
  __shared__ double2 snw[2][64];
  __shared__ double sfro[64];
  __shared__ __align__(8) uint64_t mb[2];  // V == 3: per-buffer arrival barriers
  cgc::cluster_group cluster = cgc::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int row0 = rank * RL;
  {  // batched scenes: one cluster per scene
    const int64_t sc = blockIdx.x / PC;
    K += sc * (int64_t)n_r * n_r;
    u0 += sc * n_r;
    diag += sc * 8;
  }
  if (V == 3 && tid == 0) {
    bulk::mbar_init(&mb[0], 1);
    bulk::mbar_init(&mb[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  double fro = 0.0;
  for (int e = tid; e < RL * NP; e += NT) {
    const int r = row0 + e / NP, c = e % NP;
    double2 v = make_double2(0.0, 0.0);
    if (r < n_r && c < n_r) v = K[(int64_t)r * n_r + c];
    sK[e] = v;
    fro += v.x * v.x + v.y * v.y;
  }
  for (int m = tid; m < NP; m += NT) sw[1][m] = (m < n_r) ? u0[m] : make_double2(0.0, 0.0);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) fro += __shfl_xor_sync(0xffffffffu, fro, o);
  cluster.sync();  // every CTA of the cluster is running before the first remote store
  if (lane < PC) cluster.map_shared_rank(&sfro[0], lane)[rank * NW + warp] = fro;
  cluster.sync();
  // every thread: identical fixed-order butterflies
  double f = (lane < PC * NW ? sfro[lane] : 0.0) + (lane + 32 < PC * NW ? sfro[lane + 32] : 0.0);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
  fro = sqrt(f);
  double lam = 0.0;  // lam_0 = |u_0|^2
#pragma unroll
  for (int i = 0; i < C; ++i) {
    const double2 x = sw[1][lane + 32 * i];
    lam += x.x * x.x + x.y * x.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lam += __shfl_xor_sync(0xffffffffu, lam, o);

  double scale = 1.0;
  double lam_prev = 0.0, delta_prev = 0.0, result = 0.0;
  bool have_prev = false, have_dprev = false;
  int converged = 0, iters = 0;
  const double2 *Kw = sK + (warp * 4) * NP + lane;
  for (int it = 0; it < max_iter; ++it) {
    const int src = (it + 1) & 1, dst = it & 1;
    if (V == 3 && tid == 0) bulk::arrive_expect_tx(&mb[dst], NP * 16);
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = 0.0;
#pragma unroll
    for (int i = 0; i < C; ++i) {
      const double2 x = sw[src][lane + 32 * i];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const double2 k = Kw[r * NP + 32 * i];
        v[2 * r] = fma(k.x, x.x, v[2 * r]);
        v[2 * r] = fma(-k.y, x.y, v[2 * r]);
        v[2 * r + 1] = fma(k.x, x.y, v[2 * r + 1]);
        v[2 * r + 1] = fma(k.y, x.x, v[2 * r + 1]);
      }
    }
    int idx;
    const double w = butterfly_sum<8>(v, lane, idx) * scale;  // lanes 4q..4q+3 hold index q
    const double wo = __shfl_xor_sync(0xffffffffu, w, 4);      // the other half of the pair
    double part = 0.0, wsq = 0.0;
    if (V == 3) {
      // push w; every CTA then forms Re(s^H w) and |w|^2 from the full vectors
      if ((lane & 7) == 0) {
        const int row = row0 + warp * 4 + (idx >> 1);
#pragma unroll 4
        for (int q = 0; q < PC; ++q) st_async_d2(&sw[dst][row], &mb[dst], q, w, wo);
      }
      mbar_wait_cluster(&mb[dst], (it >> 1) & 1);
#pragma unroll
      for (int i = 0; i < C; ++i) {
        const double2 x = sw[src][lane + 32 * i], y = sw[dst][lane + 32 * i];
        part = fma(x.x, y.x, fma(x.y, y.y, part));
        wsq = fma(y.x, y.x, fma(y.y, y.y, wsq));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        part += __shfl_xor_sync(0xffffffffu, part, o);
        wsq += __shfl_xor_sync(0xffffffffu, wsq, o);
      }
      part *= scale;
    } else if ((lane & 7) == 0) {  // idx even: (re, im) = (w, wo) of row warp*4 + idx/2
      const int row = row0 + warp * 4 + (idx >> 1);
      const double2 x = sw[src][row];
      part = scale * (x.x * w + x.y * wo);
      wsq = w * w + wo * wo;
      const double2 val = make_double2(w, wo);
      {
#pragma unroll 4
        for (int q = 0; q < PC; ++q) *cluster.map_shared_rank(&sw[dst][row], q) = val;
      }
    }
    double2 t0 = make_double2(part, wsq);
    if (V != 3) {
      part += __shfl_xor_sync(0xffffffffu, part, 8);
      wsq += __shfl_xor_sync(0xffffffffu, wsq, 8);
      part += __shfl_xor_sync(0xffffffffu, part, 16);
      wsq += __shfl_xor_sync(0xffffffffu, wsq, 16);
      part = __shfl_sync(0xffffffffu, part, 0);  // the sums sit in lanes 0, 8, 16, 24
      wsq = __shfl_sync(0xffffffffu, wsq, 0);
      if (lane < PC)
        *cluster.map_shared_rank(&snw[dst][rank * NW + warp], lane) = make_double2(part, wsq);
      if (V == 0) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
        asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
      } else {
        cluster.sync();
      }
      t0 = make_double2(0.0, 0.0);
      if (lane < PC * NW) t0 = snw[dst][lane];
      if (lane + 32 < PC * NW) {
        const double2 t1 = snw[dst][lane + 32];
        t0.x += t1.x;
        t0.y += t1.y;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        t0.x += __shfl_xor_sync(0xffffffffu, t0.x, o);
        t0.y += __shfl_xor_sync(0xffffffffu, t0.y, o);
      }
    }
    const double norm_w = sqrt(fmax(t0.x, 0.0));
    iters = it + 1;
    if (norm_w == 0.0) {
      result = 0.0;
      converged = 1;
      break;
    }
    if (have_prev) {
      const double delta = lam - lam_prev;
      if (fabs(delta) <= rel_tol * fmax(fabs(lam), 1e-300)) {
        double tail = 0.0;
        if (have_dprev && fabs(delta_prev) > fabs(delta) && fabs(delta) > 0.0) {
          const double q = delta / delta_prev;
          if (q > 0.0 && q < 1.0) tail = delta * q / (1.0 - q);
        }
        result = lam + tail + fabs(delta);
        converged = 1;
        break;
      }
      delta_prev = delta;
      have_dprev = true;
    }
    lam_prev = lam;
    have_prev = true;
    scale = 1.0 / norm_w;
    lam = t0.y * scale * scale;
  }
  if (!converged) result = have_prev ? lam_prev : 0.0;
  if (rank == 0 && tid == 0) {
    double inc = result;
    if (apply) {
      if (!converged) {
        inc = fro;
        counters[1] += 1;
      }
      L[0] += fmax(inc, 0.0);
      counters[0] += 1;
    }
    diag[0] = result;
    diag[1] = (double)iters;
    diag[2] = (double)converged;
    diag[3] = fro;
  }
  cluster.sync();  // no CTA may exit while peers can still write its shared memory
}

template <int C, int NW, int V = 0>
static sf_status launch_power_cl(const double2 *K, const double2 *u0, int n_r, double rel_tol,
                                 int max_iter, double *L, long long *counters, double *diag,
                                 int apply, cudaStream_t st, int batch = 1) {
  constexpr int NP = 32 * C, RL = 4 * NW, PC = NP / RL;
  const size_t dyn = (size_t)RL * NP * sizeof(double2);
  static std::atomic<uint64_t> set{0};
  if (attr_pending(set)) {
    SF_CUDA_TRY(cudaFuncSetAttribute(k_power_cl<C, NW, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)dyn));
    if (PC > 8)
      SF_CUDA_TRY(cudaFuncSetAttribute(k_power_cl<C, NW, V>,
                                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr_done(set);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(PC * batch);
  cfg.blockDim = dim3(32 * NW);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  SF_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_power_cl<C, NW, V>, K, u0, n_r, rel_tol, max_iter, L,
                                 counters, diag, apply));
  SF_LAUNCH_CHECK();
  return SF_OK;
}

// ---------------------------------------------------------------------------
// counter_unit_complex_vector(n, salt) of rng.py:28-37 (SplitMix64,
// rng.py:14-25), unnormalised; the norm is applied by k_scale_by_norm.
__device__ inline uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ inline double counter_uniform(uint64_t seed, uint64_t index) {
  const uint64_t mixed = splitmix64(seed * 0x9E3779B97F4A7C15ull + index + 1ull);
  return (double)(mixed >> 11) * 0x1.0p-53;
}
__global__ void k_start_vector(int64_t n, uint64_t salt, double2 *__restrict__ v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  v[i] = make_double2(counter_uniform(salt, 2 * i) - 0.5,
                      counter_uniform(salt, 2 * i + 1) - 0.5);
}
__global__ void __launch_bounds__(1024)
k_normalize(int64_t n, double2 *__restrict__ v) {
  __shared__ double red[33];
  double part = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    part += v[i].x * v[i].x + v[i].y * v[i].y;
  const double nrm = sqrt(block_sum(part, red));
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
    v[i] = make_double2(v[i].x / nrm, v[i].y / nrm);
}

// ---------------------------------------------------------------------------
// Pulse simulator (harness.py:221-234 without the noise): d_k[m] = sum_p
// exp(-j w_m tau_kp) rho_p for a batch of platform positions.  Delays and
// phases are formed exactly as k_pixel_delays / k_delay_phase form them; one
// CTA per (frequency, pulse) sums its pixels with a fixed-order block tree.
__global__ void __launch_bounds__(256)
k_simulate_echo(const double *__restrict__ omega, int n_r, const double *__restrict__ gammas,
                const double *__restrict__ xyz, const double2 *__restrict__ rho, int64_t n,
                double2 *__restrict__ d) {
  __shared__ double red_re[256], red_im[256];
  const int m = blockIdx.x, k = blockIdx.y;
  const double gx = gammas[3 * k], gy = gammas[3 * k + 1], gz = gammas[3 * k + 2];
  const double w = omega[m];
  double re = 0.0, im = 0.0;
  for (int64_t p = threadIdx.x; p < n; p += 256) {
    const double2 r = rho[p];
    if (r.x == 0.0 && r.y == 0.0) continue;
    const double dx = __dsub_rn(xyz[3 * p + 0], gx);
    const double dy = __dsub_rn(xyz[3 * p + 1], gy);
    const double dz = __dsub_rn(xyz[3 * p + 2], gz);
    const double dist = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)),
                                             __dmul_rn(dz, dz)));
    const double tau = __dmul_rn(2.0 / kSpeedOfLight, dist);
    double sn, cs;
    sincos(__dmul_rn(w, tau), &sn, &cs);
    // (cs - j sn) (r.x + j r.y)
    re += cs * r.x + sn * r.y;
    im += cs * r.y - sn * r.x;
  }
  red_re[threadIdx.x] = re;
  red_im[threadIdx.x] = im;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      red_re[threadIdx.x] += red_re[threadIdx.x + o];
      red_im[threadIdx.x] += red_im[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) d[(int64_t)k * n_r + m] = make_double2(red_re[0], red_im[0]);
}

sf_status launch_simulate_echo(const double *omega, int n_r, const double *gammas, int n_pulses,
                               const double *xyz, const double2 *rho, int64_t n, double2 *d,
                               cudaStream_t st) {
  if (n_pulses < 1 || n_r < 1) return SF_OK;
  k_simulate_echo<<<dim3(n_r, n_pulses), 256, 0, st>>>(omega, n_r, gammas, xyz, rho, n, d);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

// ---------------------------------------------------------------------------
// Host launchers.
sf_status launch_pixel_delays(const double *xyz, int64_t n, const double *g,
                              double *tau, int *zero_flag, cudaStream_t st, int batch,
                              int64_t in_stride) {
  const int bs = 256;
  k_pixel_delays<<<dim3((unsigned)((n + bs - 1) / bs), batch), bs, 0, st>>>(xyz, n, g, tau,
                                                                            zero_flag, in_stride);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_forward_t(const double *omega, int n_r, const double *tau,
                           int64_t n, double2 *Ft, cudaStream_t st) {
  const int bs = 256;
  const int64_t tot = n * n_r;
  k_forward_t<<<(unsigned)((tot + bs - 1) / bs), bs, 0, st>>>(omega, n_r, tau, n, Ft);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_delay_phase(const double *omega, int n_r, const double *tau,
                             int64_t n, double2 *F, cudaStream_t st) {
  const int bs = 256;
  const int64_t tot = n * n_r;
  k_delay_phase<<<(unsigned)((tot + bs - 1) / bs), bs, 0, st>>>(omega, n_r, tau, n, F);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_compose(const ComposeArgs &a, cudaStream_t st) {
  const int q = (a.n_r + 31) / 32;
  dim3 grid(a.grid), block(256);
#define SF_COMPOSE_CASE(Q)                                                    \
  case Q:                                                                     \
    k_compose<Q><<<grid, block, 0, st>>>(a.Ft, a.ell_idx, a.ell_w,            \
                                         a.ell_width, a.Gd, a.m_atoms,        \
                                         a.m_pad, a.n_r, a.k_pad,             \
                                         a.inv_sigma, a.dt, a.v0, a.Gp, a.b, a.u0part, a.maxbits, a.bmax);                           \
    break;
  switch (q) {
    SF_COMPOSE_CASE(1)
    SF_COMPOSE_CASE(2)
    SF_COMPOSE_CASE(4)
    SF_COMPOSE_CASE(8)
    SF_COMPOSE_CASE(16)
    default:
      if (q == 3) {
        k_compose<4><<<grid, block, 0, st>>>(a.Ft, a.ell_idx, a.ell_w, a.ell_width, a.Gd,
                                             a.m_atoms, a.m_pad, a.n_r, a.k_pad,
                                             a.inv_sigma, a.dt, a.v0, a.Gp, a.b, a.u0part, a.maxbits, a.bmax);
      } else if (q <= 8) {
        k_compose<8><<<grid, block, 0, st>>>(a.Ft, a.ell_idx, a.ell_w, a.ell_width, a.Gd,
                                             a.m_atoms, a.m_pad, a.n_r, a.k_pad,
                                             a.inv_sigma, a.dt, a.v0, a.Gp, a.b, a.u0part, a.maxbits, a.bmax);
      } else if (q <= 16) {
        k_compose<16><<<grid, block, 0, st>>>(a.Ft, a.ell_idx, a.ell_w, a.ell_width, a.Gd,
                                              a.m_atoms, a.m_pad, a.n_r, a.k_pad,
                                              a.inv_sigma, a.dt, a.v0, a.Gp, a.b, a.u0part, a.maxbits, a.bmax);
      } else {
        return fail(SF_EINVAL, "n_freq above 512 is not supported");
      }
  }
#undef SF_COMPOSE_CASE
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_kgram(const float *Gp, int64_t m_atoms, int n_r, int k_pad,
                       int nsplit, double2 *Kpart, cudaStream_t st) {
  const int nb = (n_r + 31) / 32;
  const int64_t per = ((m_atoms + nsplit - 1) / nsplit + 31) / 32 * 32;
  dim3 grid(nb * nb, nsplit);
  k_kgram<<<grid, 256, 0, st>>>(Gp, m_atoms, n_r, k_pad, per, Kpart);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_fq(const int64_t *qptr, const int32_t *qcol, const double *qval,
                    const double2 *Ft, int64_t n, int n_r, double2 *W, cudaStream_t st,
                    int batch) {
  const int64_t tot = n * n_r;
  const int bs = 256;
  const int64_t g = (tot + bs - 1) / bs;
  k_fq<<<dim3((unsigned)g, batch), bs, 0, st>>>(qptr, qcol, qval, Ft, n, n_r, W);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_kgram_px(const double2 *Ft, const double2 *W, int64_t n, int n_r, int nsplit,
                          double2 *Kpart, cudaStream_t st, int batch) {
  const int64_t per = ((n + nsplit - 1) / nsplit + 31) / 32 * 32;
  const int nb = (n_r + 31) / 32;
  dim3 grid(nb * (nb + 1) / 2, nsplit, batch);
  k_kgram_px<<<grid, 256, 0, st>>>(Ft, W, n, n_r, per, Kpart);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_kreduce(const double2 *Kpart, int nsplit, const double2 *u0part,
                         int nu0, int n_r, int upper_only, double scale, double2 *K, float2 *Kf,
                         double2 *u0, cudaStream_t st, const double *sig, int batch,
                         int64_t in_stride) {
  const int64_t nn = (int64_t)n_r * n_r;
  const unsigned blocks = (unsigned)((nn + 31) / 32 + (n_r + 31) / 32);
  k_kreduce<<<dim3(blocks, batch), 256, 0, st>>>(Kpart, nsplit, u0part, nu0, n_r, upper_only,
                                                 scale, K, Kf, u0, sig, in_stride);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_power_iter(const double2 *K, const float2 *Kf, const double2 *u0,
                            int n_r, double rel_tol, int max_iter, double *L,
                            long long *counters, double *diag, cudaStream_t st, int apply, int batch) {
  // N_r <= 256: k_power_cl, K~ fp64 in distributed shared memory (one CTA up
  // to N_r = 64, a cluster of 4 / 8 CTAs above); N_r <= 512: the 16-CTA
  // cluster kernel with K~ rows in fp32.  Measured variants (single-CTA fp32,
  // 16-CTA clusters at N_r <= 256, one-CTA 1024-thread) were slower, DESIGN.md.
  if (n_r <= 256) {
    if (n_r <= 32)
      return launch_power_cl<1, 8>(K, u0, n_r, rel_tol, max_iter, L, counters, diag, apply, st,
                                   batch);
    if (n_r <= 64)
      return launch_power_cl<2, 16>(K, u0, n_r, rel_tol, max_iter, L, counters, diag, apply, st,
                                    batch);
    if (n_r <= 128)
      return launch_power_cl<4, 4>(K, u0, n_r, rel_tol, max_iter, L, counters, diag, apply, st,
                                   batch);
    return launch_power_cl<8, 8>(K, u0, n_r, rel_tol, max_iter, L, counters, diag, apply, st,
                                 batch);
  }
  if (batch > 1) return fail(SF_EUNSUPPORTED, "batched scenes need n_freq <= 256");
  return launch_power_cluster<4, 16>(16, K, Kf, u0, n_r, rel_tol, max_iter, L, counters, diag,
                                     apply, st);
}

sf_status launch_start_vector(int64_t n, uint64_t salt, double2 *v, cudaStream_t st) {
  const int bs = 256;
  k_start_vector<<<(unsigned)((n + bs - 1) / bs), bs, 0, st>>>(n, salt, v);
  SF_LAUNCH_CHECK();
  k_normalize<<<1, 1024, 0, st>>>(n, v);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

}  // namespace sf
