// sf_step_fused.cu -- atom step + H z of a FISTA step as ONE kernel.
//
// Reference: kernels.py:90-97 (shrink + momentum) in pixel space,
// g = H^T (Re(B) x - Re(beta)).  The unfused chain runs k_atom_step and k_hz
// as two dependent kernels; on B200 a dependent kernel boundary costs ~4 us
// (tools/gridsync_bench.cu), which makes the small-scene FISTA step
// launch-bound.  Here the pixels are cut into G spatially compact patches
// (Morton order of the pixel lattice) and CTA c:
//
//   1. gathers y_pix (k_pix_reduce's output) at its footprint pixels,
//   2. runs the shrink + momentum update (k_atom_step's arithmetic) for EVERY
//      atom touching its own pixels -- atoms on a patch border are updated by
//      each neighbouring CTA, redundantly and bit-identically; only the owner
//      CTA stores the new state --
//   3. forms x = H z at its own pixels from those fresh values (k_hz's order).
//
// The atom state (z, c_prev) ping-pongs between two buffers per step, since
// non-owner CTAs read the previous state while the owner writes the next.
// Measured on cfg1 (B200): see DESIGN.md section 5.
#include <stdlib.h>

#include <algorithm>
#include <string>
#include <vector>

#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {

// Everything the kernel reads that is constant for the FISTA call -- the
// patch plan, the dictionary entries, b -- is loaded BEFORE
// griddepcontrol.wait (registers: up to kAP atoms per thread, two H z
// entries per lane and pixel), so after the producer (k_pix_reduce) completes
// only the y_pix and (z, c_prev) gathers remain on the critical path: one L2
// round trip, then shared-memory work.  Atoms beyond kAP * 256 per patch take
// the general loop (plan data read after the wait).
template <int WMAX, int kAP>
__global__ void __launch_bounds__(256, kAP == 1 ? 3 : 2)
k_step_fused(const FusedStepArgs a, const double *__restrict__ zin,
             const double *__restrict__ cin, double *__restrict__ zout,
             double *__restrict__ cout_, int kstep, double *__restrict__ c_out) {
  extern __shared__ __align__(16) unsigned char fs_smem[];
  double *yf = reinterpret_cast<double *>(fs_smem);  // [max_foot]
  double *zn = yf + a.max_foot;                      // [max_need]
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int c = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int f0 = a.foot_off[c], nf = a.foot_off[c + 1] - f0;
  const int q0 = a.need_off[c], nq = a.need_off[c + 1] - q0;
  // ---- constant data, before the wait
  int32_t jv[kAP];
  int lf[kAP][WMAX];
  double wl[kAP][WMAX], bre[kAP];
  bool own[kAP];
#pragma unroll
  for (int r = 0; r < kAP; ++r) {
    const int i = tid + 256 * r;
    jv[r] = -1;
    bre[r] = 0.0;
    own[r] = false;
#pragma unroll
    for (int l = 0; l < WMAX; ++l) lf[r][l] = -1, wl[r][l] = 0.0;
    if (i < nq) {
      const int q = q0 + i;
      jv[r] = a.need_atom[q];
#pragma unroll
      for (int l = 0; l < WMAX; ++l) {
        lf[r][l] = (l < a.width) ? a.need_lf[(int64_t)q * a.width + l] : -1;
        wl[r][l] = (l < a.width) ? a.need_wl[(int64_t)q * a.width + l] : 0.0;
      }
      bre[r] = a.b[jv[r]].x;
      own[r] = a.need_owner[q] != 0;
    }
  }
  int32_t fid[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) fid[r] = (tid + 256 * r < nf) ? a.foot_list[f0 + tid + 256 * r] : -1;
  // H z entries of this warp's first two own pixels: k0, k1 and two per lane
  const int p0 = a.pix_off[c], np = a.pix_off[c + 1] - p0;
  const int e0 = a.ent_off[c];
  int hk0[2] = {0, 0}, hk1[2] = {0, 0}, hl[2][2] = {{0, 0}, {0, 0}};
  double hw[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int qq = warp + 8 * r;
    if (qq < np) {
      hk0[r] = a.pe_off[p0 + c + qq];
      hk1[r] = a.pe_off[p0 + c + qq + 1];
      const int k = hk0[r] + lane;
      if (k < hk1[r]) hl[r][0] = a.ent_local[e0 + k], hw[r][0] = a.ent_w[e0 + k];
      if (k + 32 < hk1[r]) hl[r][1] = a.ent_local[e0 + k + 32], hw[r][1] = a.ent_w[e0 + k + 32];
    }
  }
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  // ---- y at the footprint pixels (summed once per pixel by k_pix_reduce)
  // and this thread's (z, c_prev): independent gathers, one L2 round trip
  double yv[2], zv[kAP], cv[kAP];
#pragma unroll
  for (int r = 0; r < 2; ++r) yv[r] = (fid[r] >= 0) ? a.ypix[fid[r]] : 0.0;
#pragma unroll
  for (int r = 0; r < kAP; ++r) {
    zv[r] = (jv[r] >= 0) ? zin[jv[r]] : 0.0;
    cv[r] = (jv[r] >= 0) ? cin[jv[r]] : 0.0;
  }
#pragma unroll
  for (int r = 0; r < 2; ++r)
    if (fid[r] >= 0) yf[tid + 256 * r] = yv[r];
  for (int f = tid + 512; f < nf; f += 256) yf[f] = a.ypix[a.foot_list[f0 + f]];
  const double tau = a.scal[0], thresh = a.scal[1];
  const double w = a.wv[kstep];
  __syncthreads();
  // ---- atom update for every atom touching this CTA's pixels (k_atom_step)
#pragma unroll
  for (int r = 0; r < kAP; ++r) {
    if (jv[r] < 0) continue;
    const int i = tid + 256 * r;
    double y = 0.0;
#pragma unroll
    for (int l = 0; l < WMAX; ++l)
      if (lf[r][l] >= 0) y += wl[r][l] * yf[lf[r][l]];
    const double u = zv[r] - tau * (y - bre[r]);
    double ci;
    if (u > thresh) ci = u - thresh;
    else if (u < -thresh) ci = u + thresh;
    else ci = 0.0;
    const double znew = ci + w * (ci - cv[r]);
    zn[i] = znew;
    if (own[r]) {
      zout[jv[r]] = znew;
      cout_[jv[r]] = ci;
      if (c_out != nullptr) c_out[jv[r]] = ci;
    }
  }
  for (int i = tid + 256 * kAP; i < nq; i += 256) {  // general path
    const int q = q0 + i;
    const int32_t j = a.need_atom[q];
    int lg[WMAX];
    double wg[WMAX];
#pragma unroll
    for (int l = 0; l < WMAX; ++l) {
      lg[l] = (l < a.width) ? a.need_lf[(int64_t)q * a.width + l] : -1;
      wg[l] = (l < a.width) ? a.need_wl[(int64_t)q * a.width + l] : 0.0;
    }
    const double z = zin[j], cp = cin[j], bj = a.b[j].x;
    double y = 0.0;
#pragma unroll
    for (int l = 0; l < WMAX; ++l)
      if (lg[l] >= 0) y += wg[l] * yf[lg[l]];
    const double u = z - tau * (y - bj);
    double ci;
    if (u > thresh) ci = u - thresh;
    else if (u < -thresh) ci = u + thresh;
    else ci = 0.0;
    const double znew = ci + w * (ci - cp);
    zn[i] = znew;
    if (a.need_owner[q]) {
      zout[j] = znew;
      cout_[j] = ci;
      if (c_out != nullptr) c_out[j] = ci;
    }
  }
  if (c_out != nullptr) return;  // last step: no H z needed
  __syncthreads();
  // ---- x = H z at the own pixels (k_hz's order), z from shared memory
#pragma unroll
  for (int r = 0; r < 2; ++r) {  // the prefetched pixels
    const int qq = warp + 8 * r;
    if (qq >= np) break;
    const int k0 = hk0[r], k1 = hk1[r];
    double s = 0.0;
    int k = k0 + lane;
    if (k + 32 < k1) {
      s += hw[r][0] * zn[hl[r][0]];
      s += hw[r][1] * zn[hl[r][1]];
      for (k += 64; k + 32 < k1; k += 64) {
        const double z0 = zn[a.ent_local[e0 + k]], z1 = zn[a.ent_local[e0 + k + 32]];
        s += a.ent_w[e0 + k] * z0;
        s += a.ent_w[e0 + k + 32] * z1;
      }
      if (k < k1) s += a.ent_w[e0 + k] * zn[a.ent_local[e0 + k]];
    } else if (k < k1) {
      s += hw[r][0] * zn[hl[r][0]];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) a.x[a.pix_list[p0 + qq]] = (float)s;
  }
  for (int qq = warp + 16; qq < np; qq += 8) {  // general path
    const int k0 = a.pe_off[p0 + c + qq], k1 = a.pe_off[p0 + c + qq + 1];
    double s = 0.0;
    int k = k0 + lane;
    for (; k + 32 < k1; k += 64) {
      const double z0 = zn[a.ent_local[e0 + k]], z1 = zn[a.ent_local[e0 + k + 32]];
      s += a.ent_w[e0 + k] * z0;
      s += a.ent_w[e0 + k + 32] * z1;
    }
    if (k < k1) s += a.ent_w[e0 + k] * zn[a.ent_local[e0 + k]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) a.x[a.pix_list[p0 + qq]] = (float)s;
  }
}

sf_status launch_step_fused(const FusedStepArgs &a, const double *zin, const double *cin,
                            double *zout, double *cout_, int kstep, double *c_out,
                            cudaStream_t st) {
  const size_t dyn = (size_t)(a.max_foot + a.max_need) * sizeof(double);
  cudaError_t ce;
#define SF_FS(W, AP)                                                                          \
  do {                                                                                        \
    static size_t set_for = 0;                                                                \
    if (dyn > 48 * 1024 && set_for < dyn) {                                                   \
      SF_CUDA_TRY(cudaFuncSetAttribute(k_step_fused<W, AP>,                                   \
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn)); \
      set_for = dyn;                                                                          \
    }                                                                                         \
    ce = launch_pdl(k_step_fused<W, AP>, dim3(a.G), dim3(256), dyn, st, a, zin, cin, zout,    \
                    cout_, kstep, c_out);                                                     \
  } while (0)
  // SF_FUSED_AP (A/B): atoms per thread prefetched before the wait (1 or 2)
  static const int ap = getenv("SF_FUSED_AP") ? atoi(getenv("SF_FUSED_AP")) : 2;
  if (a.width <= 4) {
    if (ap == 1) SF_FS(4, 1); else SF_FS(4, 2);
  } else if (a.width <= 8) {
    if (ap == 1) SF_FS(8, 1); else SF_FS(8, 2);
  } else if (a.width <= 16) {
    if (ap == 1) SF_FS(16, 1); else SF_FS(16, 2);
  } else {
    return fail(SF_EUNSUPPORTED, "fused FISTA step supports atoms of at most 16 pixels");
  }
#undef SF_FS
  if (ce != cudaSuccess) return fail(SF_ECUDA, std::string("k_step_fused: ") + cudaGetErrorString(ce));
  SF_LAUNCH_CHECK();
  return SF_OK;
}

// ---- host: patch plan ---------------------------------------------------------
static uint32_t spread16(uint32_t v) {
  v &= 0xFFFF;
  v = (v | (v << 8)) & 0x00FF00FF;
  v = (v | (v << 4)) & 0x0F0F0F0F;
  v = (v | (v << 2)) & 0x33333333;
  v = (v | (v << 1)) & 0x55555555;
  return v;
}

sf_status build_fused_plan(const double *xyz, int64_t n, const int32_t *ell_idx,
                           const double *ell_w, int64_t m, int width, const int64_t *csr_ptr,
                           const int32_t *csr_atom, const double *csr_w, int G,
                           FusedPlanHost &out) {
  if (n < 1 || G < 1 || n >= (1LL << 31) || m >= (1LL << 31))
    return fail(SF_EINVAL, "fused FISTA plan: sizes out of range");
  auto ranks = [&](int axis) {
    std::vector<double> u(n);
    for (int64_t p = 0; p < n; ++p) u[p] = xyz[3 * p + axis];
    std::vector<double> s(u);
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    std::vector<uint32_t> r(n);
    for (int64_t p = 0; p < n; ++p) r[p] = (uint32_t)(std::lower_bound(s.begin(), s.end(), u[p]) - s.begin());
    return r;
  };
  const std::vector<uint32_t> rx = ranks(0), ry = ranks(1);
  std::vector<std::pair<uint64_t, int64_t>> key(n);
  for (int64_t p = 0; p < n; ++p)
    key[p] = {((uint64_t)(spread16(ry[p]) << 1 | spread16(rx[p])) << 32) | (uint64_t)p, p};
  std::sort(key.begin(), key.end());
  std::vector<int32_t> patch(n);
  for (int64_t k = 0; k < n; ++k) patch[key[k].second] = (int32_t)((k * G) / n);
  // owner: the patch of the atom's middle pixel
  std::vector<int32_t> owner(m);
  for (int64_t j = 0; j < m; ++j) {
    int nv = 0;
    while (nv < width && ell_idx[j * width + nv] >= 0) ++nv;
    owner[j] = nv ? patch[ell_idx[j * width + nv / 2]] : (int32_t)(j % G);
  }
  // own pixels per patch
  out.G = G;
  out.pix_off.assign(G + 1, 0);
  for (int64_t p = 0; p < n; ++p) out.pix_off[patch[p] + 1]++;
  for (int c = 0; c < G; ++c) out.pix_off[c + 1] += out.pix_off[c];
  out.pix_list.assign(n, 0);
  {
    std::vector<int32_t> fill(out.pix_off.begin(), out.pix_off.end() - 1);
    for (int64_t p = 0; p < n; ++p) out.pix_list[fill[patch[p]]++] = (int32_t)p;
  }
  // needed atoms per patch: every atom touching an own pixel, plus owned atoms
  std::vector<std::vector<int32_t>> need(G);
  for (int64_t j = 0; j < m; ++j) {
    need[owner[j]].push_back((int32_t)j);
    for (int l = 0; l < width; ++l) {
      const int32_t p = ell_idx[j * width + l];
      if (p >= 0 && patch[p] != owner[j]) need[patch[p]].push_back((int32_t)j);
    }
  }
  out.need_off.assign(G + 1, 0);
  out.need_atom.clear();
  out.need_owner.clear();
  out.need_lf.clear();
  out.need_wl.clear();
  out.foot_off.assign(G + 1, 0);
  out.foot_list.clear();
  out.ent_off.assign(G + 1, 0);
  out.pe_off.assign((size_t)n + G, 0);
  out.ent_local.clear();
  out.ent_w.clear();
  out.max_foot = out.max_need = 0;
  std::vector<int32_t> fp;
  for (int c = 0; c < G; ++c) {
    auto &nd = need[c];
    std::sort(nd.begin(), nd.end());
    nd.erase(std::unique(nd.begin(), nd.end()), nd.end());
    if (nd.size() > 32767) return fail(SF_EUNSUPPORTED, "fused FISTA plan: patch too large");
    fp.clear();
    for (int32_t j : nd)
      for (int l = 0; l < width; ++l)
        if (ell_idx[(int64_t)j * width + l] >= 0) fp.push_back(ell_idx[(int64_t)j * width + l]);
    std::sort(fp.begin(), fp.end());
    fp.erase(std::unique(fp.begin(), fp.end()), fp.end());
    if (fp.size() > 32767) return fail(SF_EUNSUPPORTED, "fused FISTA plan: footprint too large");
    for (int32_t j : nd) {
      out.need_atom.push_back(j);
      out.need_owner.push_back(owner[j] == c ? 1 : 0);
      for (int l = 0; l < width; ++l) {
        const int32_t p = ell_idx[(int64_t)j * width + l];
        out.need_lf.push_back(
            p >= 0 ? (int16_t)(std::lower_bound(fp.begin(), fp.end(), p) - fp.begin()) : (int16_t)-1);
        out.need_wl.push_back(ell_w[(int64_t)j * width + l]);
      }
    }
    out.need_off[c + 1] = (int32_t)out.need_atom.size();
    out.foot_list.insert(out.foot_list.end(), fp.begin(), fp.end());
    out.foot_off[c + 1] = (int32_t)out.foot_list.size();
    out.max_foot = std::max(out.max_foot, (int)fp.size());
    out.max_need = std::max(out.max_need, (int)nd.size());
    // H z entries of the own pixels in global CSR order, atoms as local indices
    int local = 0;
    for (int q = out.pix_off[c]; q < out.pix_off[c + 1]; ++q) {
      out.pe_off[(size_t)q + c] = local;
      const int32_t p = out.pix_list[q];
      for (int64_t k = csr_ptr[p]; k < csr_ptr[p + 1]; ++k) {
        const int32_t j = csr_atom[k];
        out.ent_local.push_back((int16_t)(std::lower_bound(nd.begin(), nd.end(), j) - nd.begin()));
        out.ent_w.push_back(csr_w[k]);
        ++local;
      }
    }
    out.pe_off[(size_t)out.pix_off[c + 1] + c] = local;
    out.ent_off[c + 1] = out.ent_off[c] + local;
  }
  return SF_OK;
}

}  // namespace sf

// ---------------------------------------------------------------------------
// W = Q F~ (pixel x pixel sparse Q = H H^T times the fp64 forward operator),
// spatially tiled.  The row-per-thread k_fq reads one F~ row (N_r complex)
// from L2 per nonzero of Q: ~nnz(Q) N_r 16 bytes per pulse (411 MB at cfg1).
// Here a CTA owns a tile of up to 64 pixels (a Morton run) and one chunk of
// MC columns: it stages the F~ rows of the tile's Q-neighbourhood (the union
// of the rows' column indices) once in shared memory and forms every output
// of the tile from there, in k_fq's per-row summation order (bitwise equal).
namespace sf {

template <int MC>
__global__ void __launch_bounds__(256)
k_fq_tiled(const QTileArgs a, const double2 *__restrict__ Ft, int n_r, double2 *__restrict__ W) {
  extern __shared__ __align__(16) double2 sF[];  // [union][MC]
  const int t = blockIdx.x, m0 = blockIdx.y * MC;
  const int u0 = a.union_off[t], nu = a.union_off[t + 1] - u0;
  for (int e = threadIdx.x; e < nu * MC; e += 256) {
    const int u = e / MC, mm = e % MC;
    const int m = m0 + mm;
    sF[e] = (m < n_r) ? Ft[(int64_t)a.union_list[u0 + u] * n_r + m] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int q0 = a.pix_off[t], np = a.pix_off[t + 1] - q0;
  constexpr int PPS = 256 / MC;  // pixels per sweep
  const int mm = threadIdx.x % MC;
  const int m = m0 + mm;
  for (int q = threadIdx.x / MC; q < np; q += PPS) {
    const int k0 = a.ent_off[q0 + q], k1 = a.ent_off[q0 + q + 1];
    double re = 0.0, im = 0.0;
    for (int k = k0; k < k1; ++k) {
      const double qv = a.ent_q[k];
      const double2 f = sF[a.ent_u[k] * MC + mm];
      re += qv * f.x;
      im += qv * f.y;
    }
    if (m < n_r) W[(int64_t)a.pix_list[q0 + q] * n_r + m] = make_double2(re, im);
  }
}

// Same tiles, outputs register-blocked over m: 8 threads per pixel, thread g
// owns columns m0 + g + 8 r (r < MR), so for every r the 8 threads of a
// pixel read one contiguous 128-byte row segment (conflict-free) and each
// entry's (q, local index) load is shared by MR outputs.  Per output the
// entries are summed in k_fq's row order (bitwise equal).
template <int MR>
__global__ void __launch_bounds__(256, 2)
k_fq_tiled2(const QTileArgs a, const double2 *__restrict__ Ft, int n_r, double2 *__restrict__ W) {
  constexpr int MC = 8 * MR;
  extern __shared__ __align__(16) double2 sF[];  // [union][MC]
  const int t = blockIdx.x, m0 = blockIdx.y * MC;
  const int u0 = a.union_off[t], nu = a.union_off[t + 1] - u0;
  for (int e = threadIdx.x; e < nu * MC; e += 256) {
    const int u = e / MC, mm = e % MC;
    const int m = m0 + mm;
    sF[e] = (m < n_r) ? Ft[(int64_t)a.union_list[u0 + u] * n_r + m] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const int q0 = a.pix_off[t], np = a.pix_off[t + 1] - q0;
  const int g = threadIdx.x & 7;
  for (int q = threadIdx.x >> 3; q < np; q += 32) {
    const int k0 = a.ent_off[q0 + q], k1 = a.ent_off[q0 + q + 1];
    double re[MR], im[MR];
#pragma unroll
    for (int r = 0; r < MR; ++r) re[r] = im[r] = 0.0;
    int k = k0;
    for (; k + 2 <= k1; k += 2) {
      const double qa = a.ent_q[k], qb = a.ent_q[k + 1];
      const double2 *fa = sF + a.ent_u[k] * MC + g, *fb = sF + a.ent_u[k + 1] * MC + g;
      double2 va[MR], vb[MR];
#pragma unroll
      for (int r = 0; r < MR; ++r) va[r] = fa[8 * r], vb[r] = fb[8 * r];
#pragma unroll
      for (int r = 0; r < MR; ++r) {
        re[r] += qa * va[r].x;
        im[r] += qa * va[r].y;
        re[r] += qb * vb[r].x;
        im[r] += qb * vb[r].y;
      }
    }
    if (k < k1) {
      const double qa = a.ent_q[k];
      const double2 *fa = sF + a.ent_u[k] * MC + g;
#pragma unroll
      for (int r = 0; r < MR; ++r) {
        const double2 v = fa[8 * r];
        re[r] += qa * v.x;
        im[r] += qa * v.y;
      }
    }
    double2 *dst = W + (int64_t)a.pix_list[q0 + q] * n_r;
#pragma unroll
    for (int r = 0; r < MR; ++r) {
      const int m = m0 + g + 8 * r;
      if (m < n_r) dst[m] = make_double2(re[r], im[r]);
    }
  }
}

sf_status launch_fq_tiled2(const QTileArgs &a, const double2 *Ft, int n_r, double2 *W,
                           cudaStream_t st) {
  const int MC = a.mc;  // 16 (MR 2) or 8 (MR 1)
  const size_t dyn = (size_t)a.max_union * MC * sizeof(double2);
  dim3 grid((unsigned)a.tiles, (unsigned)((n_r + MC - 1) / MC));
  static size_t set2 = 0, set1 = 0;
  if (MC == 16) {
    if (dyn > set2) {
      SF_CUDA_TRY(cudaFuncSetAttribute(k_fq_tiled2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)dyn));
      set2 = dyn;
    }
    k_fq_tiled2<2><<<grid, 256, dyn, st>>>(a, Ft, n_r, W);
  } else {
    if (dyn > set1) {
      SF_CUDA_TRY(cudaFuncSetAttribute(k_fq_tiled2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)dyn));
      set1 = dyn;
    }
    k_fq_tiled2<1><<<grid, 256, dyn, st>>>(a, Ft, n_r, W);
  }
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_fq_tiled(const QTileArgs &a, const double2 *Ft, int n_r, double2 *W,
                          cudaStream_t st) {
  if (a.v2) return launch_fq_tiled2(a, Ft, n_r, W, st);
  const int MC = a.mc;
  const size_t dyn = (size_t)a.max_union * MC * sizeof(double2);
  dim3 grid((unsigned)a.tiles, (unsigned)((n_r + MC - 1) / MC));
  static size_t set8 = 0, set16 = 0;
  if (MC == 16) {
    if (dyn > set16) {
      SF_CUDA_TRY(cudaFuncSetAttribute(k_fq_tiled<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)dyn));
      set16 = dyn;
    }
    k_fq_tiled<16><<<grid, 256, dyn, st>>>(a, Ft, n_r, W);
  } else {
    if (dyn > set8) {
      SF_CUDA_TRY(cudaFuncSetAttribute(k_fq_tiled<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)dyn));
      set8 = dyn;
    }
    k_fq_tiled<8><<<grid, 256, dyn, st>>>(a, Ft, n_r, W);
  }
  SF_LAUNCH_CHECK();
  return SF_OK;
}

// Tiles of <= 64 pixels along the Morton order of the pixel lattice.
sf_status build_q_tiles(const double *xyz, int64_t n, const int64_t *qptr, const int32_t *qcol,
                        const double *qval, QTileHost &out) {
  if (n < 1 || n >= (1LL << 31)) return fail(SF_EINVAL, "Q tiles: size out of range");
  auto ranks = [&](int axis) {
    std::vector<double> u(n);
    for (int64_t p = 0; p < n; ++p) u[p] = xyz[3 * p + axis];
    std::vector<double> s(u);
    std::sort(s.begin(), s.end());
    s.erase(std::unique(s.begin(), s.end()), s.end());
    std::vector<uint32_t> r(n);
    for (int64_t p = 0; p < n; ++p)
      r[p] = (uint32_t)(std::lower_bound(s.begin(), s.end(), u[p]) - s.begin());
    return r;
  };
  const std::vector<uint32_t> rx = ranks(0), ry = ranks(1);
  std::vector<std::pair<uint64_t, int64_t>> key(n);
  for (int64_t p = 0; p < n; ++p)
    key[p] = {((uint64_t)(spread16(ry[p]) << 1 | spread16(rx[p])) << 32) | (uint64_t)p, p};
  std::sort(key.begin(), key.end());
  const int TP = 64;
  const int tiles = (int)((n + TP - 1) / TP);
  out.tiles = tiles;
  out.pix_off.assign(tiles + 1, 0);
  out.union_off.assign(tiles + 1, 0);
  out.pix_list.clear();
  out.union_list.clear();
  out.ent_off.assign(1, 0);
  out.ent_u.clear();
  out.ent_q.clear();
  out.max_union = 0;
  std::vector<int32_t> un;
  for (int t = 0; t < tiles; ++t) {
    const int64_t k0 = (int64_t)t * TP, k1 = std::min<int64_t>(n, k0 + TP);
    un.clear();
    for (int64_t k = k0; k < k1; ++k) {
      const int64_t p = key[k].second;
      for (int64_t e = qptr[p]; e < qptr[p + 1]; ++e) un.push_back(qcol[e]);
    }
    std::sort(un.begin(), un.end());
    un.erase(std::unique(un.begin(), un.end()), un.end());
    if (un.size() > 32767) return fail(SF_EUNSUPPORTED, "Q tiles: neighbourhood too large");
    for (int64_t k = k0; k < k1; ++k) {
      const int64_t p = key[k].second;
      out.pix_list.push_back((int32_t)p);
      for (int64_t e = qptr[p]; e < qptr[p + 1]; ++e) {
        out.ent_u.push_back((int16_t)(std::lower_bound(un.begin(), un.end(), qcol[e]) - un.begin()));
        out.ent_q.push_back(qval[e]);
      }
      out.ent_off.push_back((int32_t)out.ent_u.size());
    }
    out.union_list.insert(out.union_list.end(), un.begin(), un.end());
    out.pix_off[t + 1] = (int32_t)out.pix_list.size();
    out.union_off[t + 1] = (int32_t)out.union_list.size();
    out.max_union = std::max(out.max_union, (int)un.size());
  }
  out.mc = ((size_t)out.max_union * 16 * sizeof(double2) <= 100 * 1024) ? 16 : 8;
  if ((size_t)out.max_union * out.mc * sizeof(double2) > 200 * 1024)
    return fail(SF_EUNSUPPORTED, "Q tiles: neighbourhood too large for shared memory");
  return SF_OK;
}

}  // namespace sf
