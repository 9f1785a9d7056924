// sf_pixel.cu -- pixel-space sufficient statistics (the default for geometric pulses).
//
// Every geometric pulse has G_k = F_k H with the same static dictionary H
// (dictionary.py:151-157), so the reference's atom-space statistics factor
// exactly through pixel space:
//   A_n = sum_k G_k^H G_k / s_k^2 = H^T B_n H,   B_n = sum_k F_k^H F_k / s_k^2  (N x N)
//   b_n = sum_k G_k^H d_k / s_k^2 = H^T beta_n,  beta_n = sum_k F_k^H d_k / s_k^2
//   Re(A) z - Re(b) = H^T (Re(B) (H z) - Re(beta))          (H real, z real)
// so the engine keeps Re(B) (packed upper-triangle fp32 tiles) and beta, and
// the per-pulse update and FISTA matvec run on N pixels instead of M atoms.
// The spectrum of dA = G^H G / s^2 is untouched (power iteration on
// K~ = F Q F^H / s^2, sf_geom.cu).
//
//   k_forward_pix  F (fp64, pixel-major), packed P = [Re F~ | Im F~] rows (fp32),
//                  beta += F~^H d~, u0 += F~ (H v0) partials, max|F~| for f16x3
//   k_hv0          H v0 (once per engine)
//   k_bupdate      b = H^T beta, running max|b|
//   k_hz           x = H z            (pixel-major CSR of the ELL dictionary)
//   k_pix_reduce   y_pix = sum of the GEMV partial slots
//   k_atom_step    g = H^T y_pix - Re(b); shrink + momentum (kernels.py:90-97)
//   k_pix_to_atom  dense H^T Re(B) H readback (tests / materialisation only)
#include <string>

#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {

// the K~ build's operand format (sf_ktc.cu): 2^e scaling that puts max|x| in
// [2^13, 2^14), and 8 values -> scaled fp16 hi / lo 16-byte stores
__device__ __forceinline__ int slab_scale_exp(float mx) {
  if (!(mx > 0.f)) return 0;
  int ex;
  frexpf(mx, &ex);
  return 14 - ex;
}
__device__ __forceinline__ void slab_put8(__half *hi, __half *lo, const float *x, float scale) {
  __align__(16) __half h[8], l[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float v = x[i] * scale;
    h[i] = __float2half_rn(v);
    l[i] = __float2half_rn(v - __half2float(h[i]));
  }
  *reinterpret_cast<uint4 *>(hi) = *reinterpret_cast<const uint4 *>(h);
  *reinterpret_cast<uint4 *>(lo) = *reinterpret_cast<const uint4 *>(l);
}

template <int MAXQ>
__global__ void __launch_bounds__(256)
k_forward_pix(const double *__restrict__ omega, int n_r, const double *__restrict__ tau,
              int64_t n, int64_t n_pad, int k_pad, double inv_sigma_arg,
              const double *__restrict__ sig, const double2 *__restrict__ d,
              const double2 *__restrict__ hv0,
              double2 *__restrict__ Ft, float *__restrict__ Gp, double2 *__restrict__ dbeta,
              double2 *__restrict__ u0part, unsigned *__restrict__ maxbits, int64_t in_stride,
              FwdSlabs sl) {
  extern __shared__ __align__(16) float s_tile[];  // slab mode: [8 pixels][k_pad]
  __shared__ double2 s_d[512];
  __shared__ double s_w[512];
  __shared__ double2 s_u0[512];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  {  // batched scenes: one grid row per scene, inputs at sc * in_stride
    const int64_t sc = blockIdx.y;
    omega += sc * in_stride;
    if (sig) sig += sc * in_stride;
    d = reinterpret_cast<const double2 *>(reinterpret_cast<const double *>(d) + sc * in_stride);
    tau += sc * n;
    if (Ft) Ft += sc * n * n_r;
    if (Gp) Gp += sc * n_pad * k_pad;
    if (sl.xs) {
      sl.xs += sc * sl.xs_stride;
      sl.exps += 2 * sc;
    }
    dbeta += sc * n;
    u0part += sc * gridDim.x * n_r;
    maxbits += sc;
  }
  const double inv_sigma = sig ? sig[0] : inv_sigma_arg;  // sig = {1/sigma, sigma^2} (device)
  for (int m = threadIdx.x; m < n_r; m += blockDim.x) {
    s_d[m] = make_double2(d[m].x * inv_sigma, d[m].y * inv_sigma);
    s_w[m] = omega[m];
    s_u0[m] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  double2 acc[MAXQ];
#pragma unroll
  for (int q = 0; q < MAXQ; ++q) acc[q] = make_double2(0.0, 0.0);
  const int64_t warps_total = (int64_t)gridDim.x * (blockDim.x >> 5);
  // Panel mode: one pixel per warp, rows of Gp.  Slab mode (sl.xs): one Morton
  // group of 8 pixels per CTA (warp w = slot 8 g + w), the rows staged in shared
  // memory and written out as the K~ build's scaled fp16 hi/lo slabs
  // ([128 columns][8 pixels] per column block) -- the fp32 panel never exists.
  const bool slab = sl.xs != nullptr;
  int sl_ex = 0;
  if (slab) {
    // |F~| <= 1/sigma exactly, so the scale is known before the data
    const float mx = (float)inv_sigma;
    sl_ex = slab_scale_exp(mx);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      sl.exps[0] = sl_ex;
      sl.exps[1] = slab_scale_exp(sl.qrow_max * mx);
    }
  }
  const float sl_scale = ldexpf(1.f, sl_ex);
  const int64_t n_items = slab ? sl.ngrp : n_pad;
  for (int64_t it = slab ? (int64_t)blockIdx.x : (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;
       it < n_items; it += slab ? (int64_t)gridDim.x : warps_total) {
    const int64_t p = slab ? (int64_t)sl.grp_pix[8 * it + warp] : it;
    float *row = slab ? s_tile + (int64_t)warp * k_pad : Gp + p * k_pad;
    if (p < 0 || p >= n) {
      for (int k = lane; k < k_pad; k += 32) row[k] = 0.f;
    } else {
    const double tp = tau[p];
    const double2 hv = hv0[p];
    double bre = 0.0, bim = 0.0;
    float amax = 0.f;
#pragma unroll
    for (int q = 0; q < MAXQ; ++q) {
      const int m = lane + 32 * q;
      if (m < n_r) {
        double s, c;
        sincos(__dmul_rn(s_w[m], tp), &s, &c);  // kernels.py:29 / geometry.py:105
        if (Ft) Ft[p * n_r + m] = make_double2(c, -s);  // (only the SIMT K~ path reads F)
        const double fr = c * inv_sigma, fi = -s * inv_sigma;
        row[m] = (float)fr;
        row[n_r + m] = (float)fi;
        amax = fmaxf(amax, fmaxf(fabsf((float)fr), fabsf((float)fi)));
        const double2 dm = s_d[m];
        bre += fr * dm.x + fi * dm.y;  // conj(f~) d~
        bim += fr * dm.y - fi * dm.x;
        acc[q].x += fr * hv.x - fi * hv.y;  // f~ (H v0)_p
        acc[q].y += fr * hv.y + fi * hv.x;
      }
    }
    for (int k = 2 * n_r + lane; k < k_pad; k += 32) row[k] = 0.f;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      bre += __shfl_xor_sync(0xffffffffu, bre, o);
      bim += __shfl_xor_sync(0xffffffffu, bim, o);
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    }
    if (lane == 0) {
      dbeta[p] = make_double2(bre, bim);  // this pulse's F~^H d~, folded in order by k_fold
      atomicMax(maxbits, __float_as_uint(amax));
    }
    }
    if (slab) {
      __syncthreads();  // the group's eight rows are staged
      __half *xh = sl.xs, *xl = sl.xs + sl.slab_stride;
      for (int col = threadIdx.x; col < sl.nb * 128; col += blockDim.x) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = col < k_pad ? s_tile[j * k_pad + col] : 0.f;
        const int64_t o = ((int64_t)(col >> 7) * sl.ngrp + it) * 1024 + (int64_t)(col & 127) * 8;
        slab_put8(xh + o, xl + o, v, sl_scale);
      }
      __syncthreads();
    }
  }
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

// In-order fold of one pipelined pulse into the state: beta += dbeta, and the
// accumulate() L update with the Frobenius fallback (solver.py:194-205) from
// the power-iteration record {result, iterations, converged, |dA|_F}.
// Also folds the back-projection image (baseline.py:23-33): F^H d = sigma^2 dbeta.
__global__ void k_fold(const double2 *__restrict__ dbeta, double2 *__restrict__ beta, int64_t n,
                       const double *__restrict__ pdiag, double *__restrict__ L,
                       long long *__restrict__ counters, double *__restrict__ diag,
                       double sigma2_arg, const double *__restrict__ sig,
                       double2 *__restrict__ bp, int64_t in_stride) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  {  // batched scenes: grid y
    const int64_t sc = blockIdx.y;
    dbeta += sc * n;
    beta += sc * n;
    bp += sc * n;
    pdiag += sc * 8;
    L += sc;
    counters += sc * 2;
    diag += sc * 8;
    if (sig) sig += sc * in_stride;
  }
  const double sigma2 = sig ? sig[1] : sigma2_arg;
  if (p < n) {
    double2 b = beta[p];
    const double2 db = dbeta[p];
    b.x += db.x;
    b.y += db.y;
    beta[p] = b;
    double2 s = bp[p];
    s.x += sigma2 * db.x;
    s.y += sigma2 * db.y;
    bp[p] = s;
  }
  if (p == 0) {
    const double result = pdiag[0], converged = pdiag[2], fro = pdiag[3];
    double inc = result;
    if (converged == 0.0) {
      inc = fro;
      counters[1] += 1;
    }
    L[0] += fmax(inc, 0.0);
    counters[0] += 1;
    for (int i = 0; i < 4; ++i) diag[i] = pdiag[i];
  }
}

sf_status launch_fold(const double2 *dbeta, double2 *beta, int64_t n, const double *pdiag,
                      double *L, long long *counters, double *diag, double sigma2, double2 *bp,
                      cudaStream_t st, const double *sig, int batch, int64_t in_stride) {
  const int bs = 256;
  k_fold<<<dim3((unsigned)((n + bs - 1) / bs), batch), bs, 0, st>>>(
      dbeta, beta, n, pdiag, L, counters, diag, sigma2, sig, bp, in_stride);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

// (H v)_p for complex v through the pixel-major CSR (fixed atom order).
__global__ void k_hv0(const int64_t *__restrict__ ptr, const int32_t *__restrict__ atom,
                      const double *__restrict__ w, int64_t n, const double2 *__restrict__ v,
                      double2 *__restrict__ out) {
  const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (p >= n) return;
  double re = 0.0, im = 0.0;
  for (int64_t k = ptr[p]; k < ptr[p + 1]; ++k) {
    const double2 x = v[atom[k]];
    re += w[k] * x.x;
    im += w[k] * x.y;
  }
  out[p] = make_double2(re, im);
}

// b_j = sum_l w_jl beta[idx_jl]; running max_j |b_j| (ordered fp64 bits).
__global__ void k_bupdate(const int32_t *__restrict__ idx, const double *__restrict__ wt, int width,
                          int64_t m, const double2 *__restrict__ beta, double2 *__restrict__ b,
                          unsigned long long *__restrict__ bmax, int64_t n_pix) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  beta += blockIdx.y * n_pix;  // batched scenes: grid y
  b += blockIdx.y * m;
  bmax += blockIdx.y;
  double mx = 0.0;
  if (j < m) {
    double re = 0.0, im = 0.0;
    for (int l = 0; l < width; ++l) {
      const int32_t p = idx[j * width + l];
      if (p < 0) break;
      const double2 x = beta[p];
      re += wt[j * width + l] * x.x;
      im += wt[j * width + l] * x.y;
    }
    b[j] = make_double2(re, im);
    mx = hypot(re, im);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(bmax, (unsigned long long)__double_as_longlong(mx));
}

// x = H z (fp32 out for the GEMV); one warp per pixel, lanes over the
// pixel's CSR entries, fixed shuffle tree; zero on padding pixels.  The CSR
// arrays are engine constants, so a lane's first two entries are loaded
// before griddepcontrol.wait: only the z gathers follow the producer of z.
__global__ void k_hz(const int64_t *__restrict__ ptr, const int32_t *__restrict__ atom,
                     const double *__restrict__ w, int64_t n, int64_t n_pad,
                     const double *__restrict__ z, float *__restrict__ x, int64_t zstride,
                     int64_t xstride) {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  z += blockIdx.y * zstride;  // batched scenes: grid y
  x += blockIdx.y * xstride;
  const int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  int64_t k0 = 0, k1 = 0;
  int32_t a0 = 0, a1 = 0;
  double w0 = 0.0, w1 = 0.0;
  if (p < n) {
    k0 = ptr[p];
    k1 = ptr[p + 1];
    const int64_t k = k0 + lane;
    if (k < k1) a0 = atom[k], w0 = w[k];
    if (k + 32 < k1) a1 = atom[k + 32], w1 = w[k + 32];
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (p >= n_pad) return;
  double s = 0.0;
  if (p < n) {
    int64_t k = k0 + lane;
    if (k + 32 < k1) {  // two entries per lane in flight (same order as before)
      s += w0 * z[a0];
      s += w1 * z[a1];
      for (k += 64; k + 32 < k1; k += 64) {
        const int32_t b0 = atom[k], b1 = atom[k + 32];
        const double v0 = w[k], v1 = w[k + 32];
        s += v0 * z[b0];
        s += v1 * z[b1];
      }
      if (k < k1) s += w[k] * z[atom[k]];
    } else if (k < k1) {
      s += w0 * z[a0];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) x[p] = (float)s;
}

// k_fista_setup + k_fista_init + the first k_hz of a one-scene FISTA call as
// block roles of one launch (see PrologueArgs).  Block 0: the step scalars and
// momentum weights (k_fista_setup, solver.py:220-225 / kernels.py:87); blocks
// 1..init_blocks: z = c_prev = c0 (k_fista_init); the rest: x = H c0 with
// k_hz's exact lane order and shuffle tree (z = c0 at step 0), so every
// output is bitwise the three-kernel result.
__global__ void __launch_bounds__(256) k_fista_prologue(PrologueArgs a) {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int blk = blockIdx.x;
  if (blk == 0) {
    if (threadIdx.x == 0) {
      const double mx = __longlong_as_double((long long)*a.bmax);
      const double tau = 1.0 / a.L[0];
      const double lmb = (a.lam > 0.0) ? a.lam : a.lam_rel * mx;
      a.scal[0] = tau;
      a.scal[1] = lmb * tau;
      a.scal[2] = lmb;
      double t = a.t0;
      for (int k = 0; k < a.steps; ++k) {
        const double tn = __dmul_rn(
            0.5, __dadd_rn(1.0, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(__dmul_rn(4.0, t), t)))));
        a.wv[k] = __ddiv_rn(__dsub_rn(t, 1.0), tn);
        t = tn;
      }
    }
    return;
  }
  if (blk <= a.init_blocks) {
    const int64_t i = (blk - 1) * 256LL + threadIdx.x;
    if (i < a.m_pad) {
      const double v = (i < a.m_atoms) ? a.c0[i] : 0.0;
      a.zd[i] = v;
      a.cprev[i] = v;
    }
    return;
  }
  const int64_t p = ((blk - 1 - a.init_blocks) * 256LL + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= a.n_pad) return;
  double s = 0.0;
  if (p < a.n) {
    const int64_t k0 = a.ptr[p], k1 = a.ptr[p + 1];
    int64_t k = k0 + lane;
    if (k + 32 < k1) {
      s += a.w[k] * a.c0[a.atom[k]];
      s += a.w[k + 32] * a.c0[a.atom[k + 32]];
      for (k += 64; k + 32 < k1; k += 64) {
        const int32_t b0 = a.atom[k], b1 = a.atom[k + 32];
        const double v0 = a.w[k], v1 = a.w[k + 32];
        s += v0 * a.c0[b0];
        s += v1 * a.c0[b1];
      }
      if (k < k1) s += a.w[k] * a.c0[a.atom[k]];
    } else if (k < k1) {
      s += a.w[k] * a.c0[a.atom[k]];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) a.x[p] = (float)s;
}

const void *fista_prologue_kernel() { return (const void *)k_fista_prologue; }

bool fista_prologue_ok(int64_t n_pad, int batch) {
  const char *v = getenv("SF_FISTA_PROLOGUE");  // per call: tests compare both paths
  return !(v && v[0] == '0') && batch == 1 && n_pad * batch < 32768;  // k_hz regime
}

PrologueArgs make_prologue_args(const double *L, const unsigned long long *bmax, double lam,
                                double lam_rel, double *scal, double t0, int steps, double *wv,
                                const double *c0, int64_t m_atoms, int64_t m_pad, double *zd,
                                double *cprev, const int64_t *ptr, const int32_t *atom,
                                const double *w, int64_t n, int64_t n_pad, float *x) {
  PrologueArgs a;
  a.L = L;
  a.bmax = bmax;
  a.lam = lam;
  a.lam_rel = lam_rel;
  a.scal = scal;
  a.t0 = t0;
  a.steps = steps;
  a.wv = wv;
  a.c0 = c0;
  a.m_atoms = m_atoms;
  a.m_pad = m_pad;
  a.zd = zd;
  a.cprev = cprev;
  a.ptr = ptr;
  a.atom = atom;
  a.w = w;
  a.n = n;
  a.n_pad = n_pad;
  a.x = x;
  a.init_blocks = (int)((m_pad + 255) / 256);
  a.hz_blocks = (int)((n_pad * 32 + 255) / 256);
  return a;
}

sf_status launch_fista_prologue(const PrologueArgs &a, cudaStream_t st) {
  k_fista_prologue<<<1 + a.init_blocks + a.hz_blocks, 256, 0, st>>>(a);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

// x = H z with one thread per (scene, pixel), lanes over consecutive pixels,
// from the entry-major transpose of the CSR (coalesced index/weight loads; the
// z gathers of neighbouring pixels hit neighbouring atoms).  Bitwise equal to
// k_hz: k_hz's lane l sums entries l, l+32, ... in order into its own partial
// and the xor-butterfly 16, 8, 4, 2, 1 combines them; here slot t[l] gets the
// same in-order sum and lane 0's butterfly chain t[i] += t[i + o] (o = 16..1)
// is replayed in registers (IEEE addition is commutative, so every butterfly
// lane holds lane 0's value).  Batched engines (cfg2): 101 -> ~30 us a step.
template <int E>
__global__ void __launch_bounds__(256)
k_hz_ell(const int32_t *__restrict__ atomT, const double *__restrict__ wT, int ents, int64_t n,
         int64_t n_pad, const double *__restrict__ z, float *__restrict__ x, int64_t zstride,
         int64_t xstride) {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  z += blockIdx.y * zstride;
  x += blockIdx.y * xstride;
  const int64_t p = blockIdx.x * 256LL + threadIdx.x;
  constexpr int EP = E <= 32 ? E : 1;  // entries whose indices are loaded before the wait
  int32_t a[EP];
  double w[EP];
#pragma unroll
  for (int e = 0; e < EP; ++e) {  // engine constants
    a[e] = (p < n && e < ents) ? atomT[e * n_pad + p] : -1;
    w[e] = (a[e] >= 0) ? wT[e * n_pad + p] : 0.0;
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (p >= n_pad) return;
  double t[32];
#pragma unroll
  for (int l = 0; l < 32; ++l) t[l] = 0.0;
  if (E <= 32) {
#pragma unroll
    for (int e = 0; e < EP; ++e)
      if (a[e] >= 0) t[e & 31] += w[e] * z[a[e]];
  } else if (p < n) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int32_t ae = e < ents ? atomT[e * n_pad + p] : -1;
      if (ae >= 0) t[e & 31] += wT[e * n_pad + p] * z[ae];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < o; ++i) t[i] += t[i + o];
  x[p] = (float)t[0];
}

sf_status launch_hz_ell(const int32_t *atomT, const double *wT, int ents, int64_t n, int64_t n_pad,
                        const double *z, float *x, cudaStream_t st, int batch, int64_t zstride,
                        int64_t xstride) {
  const dim3 g((unsigned)((n_pad + 255) / 256), batch);
  cudaError_t ce;
  if (ents <= 32)
    ce = launch_pdl(k_hz_ell<32>, g, dim3(256), 0, st, atomT, wT, ents, n, n_pad, z, x, zstride,
                    xstride);
  else if (ents <= 64)
    ce = launch_pdl(k_hz_ell<64>, g, dim3(256), 0, st, atomT, wT, ents, n, n_pad, z, x, zstride,
                    xstride);
  else
    return fail(SF_EINVAL, "k_hz_ell: more than 64 atoms per pixel");
  if (ce != cudaSuccess) return fail(SF_ECUDA, std::string("k_hz_ell: ") + cudaGetErrorString(ce));
  SF_LAUNCH_CHECK();
  return SF_OK;
}

// x = H z with G lanes per pixel (32/G pixels per warp), bit-identical to
// k_hz: lane h forms the per-lane partial sums s_j (j = h, h+G, ...: entries
// j, j+32, j+64, ... in order) that k_hz's lanes j would hold, combines them
// with k_hz's xor-butterfly levels 16..G locally, then shuffles G/2..1.
template <int G>
__global__ void k_hz_packed(const int64_t *__restrict__ ptr, const int32_t *__restrict__ atom,
                            const double *__restrict__ w, int64_t n, int64_t n_pad,
                            const double *__restrict__ z, float *__restrict__ x, int64_t zstride,
                            int64_t xstride) {
  constexpr int M = 32 / G;
  pdl_enter();
  z += blockIdx.y * zstride;  // batched scenes: grid y
  x += blockIdx.y * xstride;
  const int64_t p = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G;
  const int h = threadIdx.x & (G - 1);
  double v[M];
#pragma unroll
  for (int m = 0; m < M; ++m) v[m] = 0.0;
  if (p < n) {
    const int64_t k0 = ptr[p], k1 = ptr[p + 1];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      int64_t k = k0 + h + m * G;
      double s = 0.0;
      for (; k + 32 < k1; k += 64) {
        const int32_t a0 = atom[k], a1 = atom[k + 32];
        const double w0 = w[k], w1 = w[k + 32];
        s += w0 * z[a0];
        s += w1 * z[a1];
      }
      if (k < k1) s += w[k] * z[atom[k]];
      v[m] = s;
    }
  }
#pragma unroll
  for (int o = 16; o >= G; o >>= 1) {
#pragma unroll
    for (int m = 0; m < o / G; ++m) v[m] += v[m + o / G];
  }
  double t = v[0];
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (h == 0 && p < n_pad) x[p] = (float)t;
}

// y_pix = sum over the nt partial slots of each pixel (fixed order, fp64).
// Block = 32 pixels x 8 slot lanes; each slot lane sums every 8th slot,
// then the 8 lane sums are added in order.
__global__ void __launch_bounds__(256)
k_pix_reduce(const float *__restrict__ P, int nt, int64_t n_pad, double *__restrict__ ypix,
             PeerSlots peers, size_t peer_off) {
  pdl_enter();
  P += blockIdx.y * (int64_t)nt * nt * kTile;  // batched scenes: grid y
  ypix += blockIdx.y * n_pad;
  __shared__ double red[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t i = blockIdx.x * 32LL + tx;
  double s = 0.0;
  if (i < n_pad) {
    const int64_t blk = i / kTile;
    const int r = (int)(i - blk * kTile);
    const float *src = P + blk * (int64_t)nt * kTile + r;
    for (int k = ty; k < nt; k += 8) s += (double)src[(int64_t)k * kTile];
  }
  red[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && i < n_pad) {
    double y = 0.0;
#pragma unroll
    for (int t = 0; t < 8; ++t) y += red[t][tx];
    if (peers.world > 0) {
      // sharded over a peer-memory group: the rank's partial goes straight
      // into its slot on every rank (stores over NVLink; sf_shard.cu)
      for (int r = 0; r < peers.world; ++r) peers.p[r][peer_off + i] = y;
    } else {
      ypix[i] = y;
    }
  }
}

// g_j = (H^T y_pix)_j - Re(b_j); then the reference step (kernels.py:90-97).
// WMAX >= width: every ELL load is issued before the first use.
template <int WMAX>
__global__ void k_atom_step(const int32_t *__restrict__ idx, const double *__restrict__ wt, int width,
                            int64_t m, const double *__restrict__ ypix,
                            const double2 *__restrict__ b, double *__restrict__ zd,
                            double *__restrict__ cprev, const double *__restrict__ scal,
                            const double *__restrict__ wv, int kstep, double *__restrict__ c_out,
                            int64_t m_pad, int64_t n_pad) {
  // The ELL table and b are constant during the FISTA call (b was written
  // before the call's first kernel), so they are loaded before
  // griddepcontrol.wait; y_pix, z, c_prev and the step scalars after it.
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  {  // batched scenes: grid y
    const int64_t sc = blockIdx.y;
    ypix += sc * n_pad;
    b += sc * m;
    zd += sc * m_pad;
    cprev += sc * m_pad;
    scal += sc * 4;
    if (c_out) c_out += sc * m;
  }
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= m) {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    return;
  }
  int32_t pi[WMAX];
  double wi[WMAX], yv[WMAX];
#pragma unroll
  for (int l = 0; l < WMAX; ++l) {
    pi[l] = (l < width) ? idx[j * width + l] : -1;
    wi[l] = (l < width) ? wt[j * width + l] : 0.0;
  }
  const double bre = b[j].x;
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  const double w = wv[kstep];
#pragma unroll
  for (int l = 0; l < WMAX; ++l) yv[l] = (pi[l] >= 0) ? ypix[pi[l]] : 0.0;
  double y = 0.0;
#pragma unroll
  for (int l = 0; l < WMAX; ++l)
    if (pi[l] >= 0) y += wi[l] * yv[l];
  const double tau = scal[0], thresh = scal[1];
  const double z = zd[j];
  const double u = z - tau * (y - bre);
  double ci;
  if (u > thresh) ci = u - thresh;
  else if (u < -thresh) ci = u + thresh;
  else ci = 0.0;
  const double zn = ci + w * (ci - cprev[j]);
  cprev[j] = ci;
  zd[j] = zn;
  if (c_out != nullptr) c_out[j] = ci;
}


// Dense Re(A) = H^T Re(B) H from the pixel tile store (readback only).
__global__ void k_pix_to_atom(const float *__restrict__ B, int ntp, const int32_t *__restrict__ idx,
                              const double *__restrict__ wt, int width, int64_t m,
                              double *__restrict__ A) {
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= m * m) return;
  const int64_t j1 = e / m, j2 = e % m;
  double s = 0.0;
  for (int l1 = 0; l1 < width; ++l1) {
    const int32_t p1 = idx[j1 * width + l1];
    if (p1 < 0) break;
    for (int l2 = 0; l2 < width; ++l2) {
      const int32_t p2 = idx[j2 * width + l2];
      if (p2 < 0) break;
      // symmetric store: element (a, c) with a <= c, diagonal tiles upper half
      int a = p1, c = p2;
      if (a > c) {
        const int t = a;
        a = c;
        c = t;
      }
      const int I = a / kTile, J = c / kTile;
      const int r = a % kTile, cc = c % kTile;
      const int64_t t = (int64_t)I * ntp - (int64_t)I * (I - 1) / 2 + (J - I);
      s += wt[j1 * width + l1] * wt[j2 * width + l2] *
           (double)B[t * kTileElems + tile_offset(r, cc)];
    }
  }
  A[e] = s;
}



// Batched scenes: scatter omega [n_r] | gammas [B][3] | d [B][n_r] c128 |
// sigma2 [B] into each scene's input block (one CTA per scene).
__global__ void k_stage_batch(const double *__restrict__ raw, int n_r, int B, int64_t off_d,
                              int64_t off_g, int64_t off_s, int64_t stride,
                              double *__restrict__ in) {
  const int sc = blockIdx.x;
  const double *g = raw + n_r + 3 * (int64_t)sc;
  const double *d = raw + n_r + 3 * (int64_t)B + 2 * (int64_t)n_r * sc;
  const double s2 = raw[n_r + 3 * (int64_t)B + 2 * (int64_t)n_r * B + sc];
  double *o = in + sc * stride;
  for (int i = threadIdx.x; i < n_r; i += blockDim.x) o[i] = raw[i];
  for (int i = threadIdx.x; i < 2 * n_r; i += blockDim.x) o[off_d + i] = d[i];
  if (threadIdx.x < 3) o[off_g + threadIdx.x] = g[threadIdx.x];
  if (threadIdx.x == 0) {
    o[off_s] = __ddiv_rn(1.0, __dsqrt_rn(s2));  // == the host's 1.0 / sqrt(sigma2)
    o[off_s + 1] = s2;
  }
}

sf_status launch_stage_batch(const double *raw, int n_r, int B, int64_t off_d, int64_t off_g,
                             int64_t off_s, int64_t stride, double *in, cudaStream_t st) {
  k_stage_batch<<<B, 128, 0, st>>>(raw, n_r, B, off_d, off_g, off_s, stride, in);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

// ---------------------------------------------------------------------------
sf_status launch_forward_pix(const PixelForwardArgs &a, cudaStream_t st) {
  const int q = (a.n_r + 31) / 32;
  dim3 grid(a.grid, a.batch), block(256);
  const size_t dsm = a.slabs.xs ? (size_t)8 * a.k_pad * sizeof(float) : 0;
#define SF_FWD(Q)                                                                          \
  do {                                                                                     \
    if (dsm > 16384) {                                                                     \
      static std::atomic<uint64_t> set{0};                                                 \
      if (attr_pending(set)) {                                                             \
        SF_CUDA_TRY(cudaFuncSetAttribute(k_forward_pix<Q>,                                 \
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                         8 * 1024 * (int)sizeof(float)));                  \
        attr_done(set);                                                                    \
      }                                                                                    \
    }                                                                                      \
    k_forward_pix<Q><<<grid, block, dsm, st>>>(a.omega, a.n_r, a.tau, a.n, a.n_pad,        \
                                               a.k_pad, a.inv_sigma, a.sig, a.d, a.hv0,    \
                                               a.Ft, a.Gp, a.dbeta, a.u0part, a.maxbits,   \
                                               a.in_stride, a.slabs);                      \
  } while (0)
  if (q <= 1) SF_FWD(1);
  else if (q <= 2) SF_FWD(2);
  else if (q <= 4) SF_FWD(4);
  else if (q <= 8) SF_FWD(8);
  else if (q <= 16) SF_FWD(16);
  else return fail(SF_EINVAL, "n_freq above 512 is not supported");
#undef SF_FWD
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_hv0(const int64_t *ptr, const int32_t *atom, const double *w, int64_t n,
                     const double2 *v, double2 *out, cudaStream_t st) {
  const int bs = 256;
  k_hv0<<<(unsigned)((n + bs - 1) / bs), bs, 0, st>>>(ptr, atom, w, n, v, out);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_bupdate(const int32_t *idx, const double *w, int width, int64_t m,
                         const double2 *beta, double2 *b, unsigned long long *bmax,
                         cudaStream_t st, int batch, int64_t n_pix) {
  const int bs = 256;
  k_bupdate<<<dim3((unsigned)((m + bs - 1) / bs), batch), bs, 0, st>>>(idx, w, width, m, beta, b,
                                                                       bmax, n_pix);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_hz(const int64_t *ptr, const int32_t *atom, const double *w, int64_t n,
                    int64_t n_pad, const double *z, float *x, cudaStream_t st, int batch,
                    int64_t zstride, int64_t xstride) {
  const int bs = 256;
  cudaError_t ce;
  if (n_pad * batch >= 32768) {  // throughput regime: 4 pixels per warp (bit-identical sums)
    const int64_t threads = n_pad * 8;
    ce = launch_pdl(k_hz_packed<8>, dim3((unsigned)((threads + bs - 1) / bs), batch), dim3(bs), 0,
                    st, ptr, atom, w, n, n_pad, z, x, zstride, xstride);
  } else {
    const int64_t threads = n_pad * 32;
    ce = launch_pdl(k_hz, dim3((unsigned)((threads + bs - 1) / bs), batch), dim3(bs), 0, st, ptr,
                    atom, w, n, n_pad, z, x, zstride, xstride);
  }
  if (ce != cudaSuccess) return fail(SF_ECUDA, std::string("k_hz: ") + cudaGetErrorString(ce));
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_pix_reduce(const float *P, int nt, int64_t n_pad, double *ypix, cudaStream_t st,
                            int batch, const PeerSlots *peers, size_t peer_off) {
  cudaError_t ce = launch_pdl(k_pix_reduce, dim3((unsigned)((n_pad + 31) / 32), batch), dim3(256),
                              0, st, P, nt, n_pad, ypix, peers ? *peers : PeerSlots(), peer_off);
  if (ce != cudaSuccess)
    return fail(SF_ECUDA, std::string("k_pix_reduce: ") + cudaGetErrorString(ce));
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_atom_step(const int32_t *idx, const double *w, int width, int64_t m,
                           const double *ypix, const double2 *b, double *zd, double *cprev,
                           const double *scal, const double *wv, int kstep, double *c_out,
                           cudaStream_t st, int batch, int64_t m_pad, int64_t n_pad) {
  const int bs = 256;
  const dim3 g((unsigned)((m + bs - 1) / bs), batch);
  cudaError_t ce;
  if (width <= 4)
    ce = launch_pdl(k_atom_step<4>, dim3(g), dim3(bs), 0, st, idx, w, width, m, ypix, b, zd, cprev,
                    scal, wv, kstep, c_out, m_pad, n_pad);
  else if (width <= 8)
    ce = launch_pdl(k_atom_step<8>, dim3(g), dim3(bs), 0, st, idx, w, width, m, ypix, b, zd, cprev,
                    scal, wv, kstep, c_out, m_pad, n_pad);
  else if (width <= 16)
    ce = launch_pdl(k_atom_step<16>, dim3(g), dim3(bs), 0, st, idx, w, width, m, ypix, b, zd,
                    cprev, scal, wv, kstep, c_out, m_pad, n_pad);
  else
    return fail(SF_EUNSUPPORTED, "pixel-space FISTA supports atoms of at most 16 pixels");
  if (ce != cudaSuccess)
    return fail(SF_ECUDA, std::string("k_atom_step: ") + cudaGetErrorString(ce));
  SF_LAUNCH_CHECK();
  return SF_OK;
}

bool is_atom_step_kernel(const void *f) {
  return f == (const void *)k_atom_step<4> || f == (const void *)k_atom_step<8> ||
         f == (const void *)k_atom_step<16>;
}

sf_status launch_pix_to_atom(const float *B, int ntp, const int32_t *idx, const double *w,
                             int width, int64_t m, double *A, cudaStream_t st) {
  const int64_t tot = m * m;
  const int bs = 256;
  k_pix_to_atom<<<(unsigned)((tot + bs - 1) / bs), bs, 0, st>>>(B, ntp, idx, w, width, m, A);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

}  // namespace sf
