// sf_fista_chip.cu -- one-launch FISTA for pixel-space statistics whose tile
// store fits on chip (the L2-resident regime, e.g. BASELINE cfg1).
//
// Reference: solver.py:209-226 (online_fista_pulse), kernels.py:78-103.  Per
// step g = H^T (Re(B) (H z) - Re(beta)); the 4-kernel chain (k_gemv_sym ->
// k_pix_reduce -> k_atom_step -> k_hz) is latency-bound there: four dependent
// launches per step.  This cooperative kernel runs all steps of a pulse with
// three grid barriers per step and keeps Re(B) ON CHIP:
//
//   * one CTA per SM (512 threads = two 256-thread groups); CTA c owns tiles
//     c, c+G, c+2G, ...; the first `smem_tiles` of them are copied into shared
//     memory once per launch (64 KiB each) and re-read from there every step,
//     the rest stream from L2.  Each group runs gemv_tile_compute (the same
//     thread mapping and summation order as k_gemv_sym) on alternate tiles.
//   * pixels are cut into G spatially compact patches (Morton order of the
//     pixel grid); CTA c owns the atoms anchored in its patch and the pixels of
//     its patch.  After the matvec barrier it sums the partial slots of its
//     atoms' footprint pixels into shared memory (k_pix_reduce's order), runs
//     the shrink + momentum step for its atoms (k_atom_step's arithmetic),
//     barrier, then H z for its own pixels (k_hz's order), barrier.
//
// Every reduction keeps the 4-kernel chain's order, so the iterates are
// bitwise identical to it (tests/test_gpu_parity.py checks this).  Data
// produced inside the launch (P, x, zd) is read with ld.global.cg (L2), never
// through the non-coherent L1.
#include <cooperative_groups.h>

#include <algorithm>
#include <string>
#include <vector>

#include "sf_common.cuh"
#include "sf_kernels.cuh"
#include "sf_gemv_tile.cuh"

namespace sf {

namespace cg = cooperative_groups;

namespace {

__device__ __forceinline__ void chip_hz(const ChipFistaArgs &a, int c) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int p0 = a.pix_off[c], np = a.pix_off[c + 1] - p0;
  for (int q = warp; q < np; q += 16) {
    const int32_t p = a.pix_list[p0 + q];
    double s = 0.0;
    const int64_t k0 = a.csr_ptr[p], k1 = a.csr_ptr[p + 1];
    int64_t k = k0 + lane;
    for (; k + 32 < k1; k += 64) {  // k_hz's order: entries lane, lane+32, lane+64, ...
      const int32_t a0 = a.csr_atom[k], a1 = a.csr_atom[k + 32];
      const double w0 = a.csr_w[k], w1 = a.csr_w[k + 32];
      s += w0 * __ldcg(a.zd + a0);
      s += w1 * __ldcg(a.zd + a1);
    }
    if (k < k1) s += a.csr_w[k] * __ldcg(a.zd + a.csr_atom[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) a.x[p] = (float)s;
  }
}

__device__ __forceinline__ void chip_mark(const ChipFistaArgs &a, int &n) {
  if (a.trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[n] = t;
  }
  ++n;
}

}  // namespace

__global__ void __launch_bounds__(512, 1) k_fista_chip(const ChipFistaArgs a) {
  extern __shared__ __align__(16) unsigned char chip_smem[];
  float4 *st = reinterpret_cast<float4 *>(chip_smem);
  double *yf = reinterpret_cast<double *>(chip_smem + (size_t)a.smem_tiles * kTileElems * 4);
  __shared__ float s_row[2][8][kTile];
  __shared__ float s_col[2][kTile];
  cg::grid_group grid = cg::this_grid();
  const int c = blockIdx.x, G = gridDim.x, tid = threadIdx.x, grp = tid >> 8;
  const int lane = tid & 31, gw = (tid & 255) >> 5;
  int tn = 0;
  chip_mark(a, tn);

  // this CTA's resident tiles (constant during the launch)
  for (int kk = 0; kk < a.smem_tiles; ++kk) {
    const int64_t t = c + (int64_t)G * kk;
    if (t >= a.n_tiles) break;
    const int2 ij = a.tiles[t];
    const float4 *src =
        reinterpret_cast<const float4 *>(a.B + tri_index(ij.x, ij.y, a.nt) * kTileElems);
    for (int e = tid; e < kTileElems / 4; e += 512) st[kk * (kTileElems / 4) + e] = src[e];
  }
  // k_fista_setup's scalars (solver.py:220-225)
  const double mx = __longlong_as_double((long long)*a.bmax);
  const double tau = 1.0 / a.L[0];
  const double lmb = (a.lam > 0.0) ? a.lam : a.lam_rel * mx;
  const double thresh = lmb * tau;
  if (a.first && c == 0 && tid == 0) {
    a.scal[0] = tau;
    a.scal[1] = thresh;
    a.scal[2] = lmb;
  }
  const int q0 = a.atom_off[c], q1 = a.atom_off[c + 1];
  if (a.first) {
    for (int q = q0 + tid; q < q1; q += 512) {
      const int32_t j = a.atom_list[q];
      const double v = a.c0[j];
      a.zd[j] = v;
      a.cprev[j] = v;
    }
    if (c == 0)
      for (int64_t p = a.n + tid; p < a.n_pad; p += 512) a.x[p] = 0.f;
    grid.sync();
    chip_hz(a, c);
    grid.sync();
  } else {
    __syncthreads();
  }
  chip_mark(a, tn);
  const int f0 = a.foot_off[c], nf = a.foot_off[c + 1] - f0;
  for (int k = 0; k < a.steps; ++k) {
    // ---- y partial slots = Re(B) x over this CTA's tiles
    for (int kk = grp;; kk += 2) {
      const int64_t t = c + (int64_t)G * kk;
      if (t >= a.n_tiles) break;
      float4 v[4][4];
      if (kk < a.smem_tiles) {
        const float4 *T = st + kk * (kTileElems / 4);
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
          for (int i = 0; i < 4; ++i) v[s4][i] = T[(gw + 8 * s4) * kTile + lane + 32 * i];
      } else {
        const int2 ij = a.tiles[t];
        const float4 *T =
            reinterpret_cast<const float4 *>(a.B + tri_index(ij.x, ij.y, a.nt) * kTileElems);
#pragma unroll
        for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            v[s4][i] = __ldg(T + (int64_t)(gw + 8 * s4) * kTile + lane + 32 * i);
      }
      const int2 ij = a.tiles[t];
      if (grp == 0)
        gemv_tile_compute<1>(v, ij.x, ij.y, a.x, a.P, a.nt, 1, s_row[0], s_col[0]);
      else
        gemv_tile_compute<2>(v, ij.x, ij.y, a.x, a.P, a.nt, 1, s_row[1], s_col[1]);
    }
    chip_mark(a, tn);
    grid.sync();
    chip_mark(a, tn);
    // ---- y at this CTA's footprint pixels: k_pix_reduce's order (slot lane g
    // sums slots g, g+8, ...; the eight lane sums are added in order)
    for (int e = tid; e < ((nf + 63) >> 6) * 512; e += 512) {
      const int fi = e >> 3, g8 = e & 7;
      double s = 0.0;
      if (fi < nf) {
        const int32_t p = a.foot_list[f0 + fi];
        const float *src = a.P + (int64_t)(p / kTile) * a.nt * kTile + (p % kTile);
        for (int q = g8; q < a.nt; q += 8) s += (double)__ldcg(src + (int64_t)q * kTile);
      }
      double part[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) part[u] = __shfl_sync(0xffffffffu, s, (lane & ~7) + u);
      if (g8 == 0 && fi < nf) {
        double y = 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) y += part[u];
        yf[fi] = y;
      }
    }
    __syncthreads();
    // ---- shrink + momentum for this CTA's atoms (k_atom_step, kernels.py:90-97)
    const double w = a.w[k];
    const bool last = a.last && (k == a.steps - 1);
    for (int q = q0 + tid; q < q1; q += 512) {
      const int32_t j = a.atom_list[q];
      double y = 0.0;
      for (int l = 0; l < a.width; ++l) {
        const int32_t pi = a.ell_idx[(int64_t)j * a.width + l];
        const double wi = a.ell_w[(int64_t)j * a.width + l];
        const int lf = a.atom_lf[(int64_t)q * a.width + l];
        if (pi >= 0) y += wi * yf[lf];
      }
      const double z = __ldcg(a.zd + j);
      const double u = z - tau * (y - a.b[j].x);
      double ci;
      if (u > thresh) ci = u - thresh;
      else if (u < -thresh) ci = u + thresh;
      else ci = 0.0;
      const double zn = ci + w * (ci - __ldcg(a.cprev + j));
      a.cprev[j] = ci;
      a.zd[j] = zn;
      if (last) a.c_out[j] = ci;
    }
    chip_mark(a, tn);
    if (last) break;
    grid.sync();
    chip_mark(a, tn);
    chip_hz(a, c);
    chip_mark(a, tn);
    grid.sync();
    chip_mark(a, tn);
  }
}

sf_status launch_fista_chip(const ChipFistaArgs &a, int grid, cudaStream_t st) {
  const size_t dyn = (size_t)a.smem_tiles * kTileElems * 4 + (size_t)a.max_foot * sizeof(double);
  static size_t set_for = 0;
  if (set_for < dyn) {
    SF_CUDA_TRY(cudaFuncSetAttribute(k_fista_chip, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)dyn));
    set_for = dyn;
  }
  void *args[] = {const_cast<ChipFistaArgs *>(&a)};
  cudaError_t e =
      cudaLaunchCooperativeKernel((const void *)k_fista_chip, dim3(grid), dim3(512), args, dyn, st);
  count_launch();
  if (e != cudaSuccess)
    return fail(SF_ECUDA, std::string("cooperative on-chip FISTA launch: ") + cudaGetErrorString(e));
  return SF_OK;
}

int fista_chip_fits(int device, int smem_tiles, int max_foot) {
  const size_t dyn = (size_t)smem_tiles * kTileElems * 4 + (size_t)max_foot * sizeof(double);
  if (cudaFuncSetAttribute(k_fista_chip, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn) !=
      cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fista_chip, 512, dyn) !=
      cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  (void)device;
  return per_sm;
}

// ---- host: patch plan ----------------------------------------------------------
static uint32_t spread_bits(uint32_t v) {
  v &= 0xFFFF;
  v = (v | (v << 8)) & 0x00FF00FF;
  v = (v | (v << 4)) & 0x0F0F0F0F;
  v = (v | (v << 2)) & 0x33333333;
  v = (v | (v << 1)) & 0x55555555;
  return v;
}

sf_status build_chip_plan(const double *xyz, int64_t n, const int32_t *ell_idx, int64_t m,
                          int width, int G, ChipPlanHost &out) {
  if (n < 1 || G < 1 || n >= (1LL << 31) || m >= (1LL << 31))
    return fail(SF_EINVAL, "on-chip FISTA plan: sizes out of range");
  // Morton order of the pixel lattice (coordinate ranks), cut into G runs
  auto ranks = [&](int axis) {
    std::vector<double> v(n);
    for (int64_t p = 0; p < n; ++p) v[p] = xyz[3 * p + axis];
    std::vector<double> u(v);
    std::sort(u.begin(), u.end());
    u.erase(std::unique(u.begin(), u.end()), u.end());
    std::vector<uint32_t> r(n);
    for (int64_t p = 0; p < n; ++p)
      r[p] = (uint32_t)(std::lower_bound(u.begin(), u.end(), v[p]) - u.begin());
    return r;
  };
  const std::vector<uint32_t> rx = ranks(0), ry = ranks(1);
  std::vector<std::pair<uint64_t, int32_t>> key(n);
  for (int64_t p = 0; p < n; ++p)
    key[p] = {((uint64_t)(spread_bits(ry[p]) << 1 | spread_bits(rx[p])) << 32) | (uint64_t)p,
              (int32_t)p};
  std::sort(key.begin(), key.end());
  std::vector<int32_t> patch(n);
  for (int64_t k = 0; k < n; ++k) patch[key[k].second] = (int32_t)((k * G) / n);
  // atom owner: patch of its middle valid pixel
  std::vector<int32_t> owner(m);
  for (int64_t j = 0; j < m; ++j) {
    int nv = 0;
    while (nv < width && ell_idx[j * width + nv] >= 0) ++nv;
    owner[j] = nv ? patch[ell_idx[j * width + nv / 2]] : (int32_t)(j % G);
  }
  out.pix_off.assign(G + 1, 0);
  out.atom_off.assign(G + 1, 0);
  for (int64_t p = 0; p < n; ++p) out.pix_off[patch[p] + 1]++;
  for (int64_t j = 0; j < m; ++j) out.atom_off[owner[j] + 1]++;
  for (int c = 0; c < G; ++c) {
    out.pix_off[c + 1] += out.pix_off[c];
    out.atom_off[c + 1] += out.atom_off[c];
  }
  out.pix_list.assign(n, 0);
  out.atom_list.assign(m, 0);
  {
    std::vector<int32_t> fill(out.pix_off.begin(), out.pix_off.end() - 1);
    for (int64_t p = 0; p < n; ++p) out.pix_list[fill[patch[p]]++] = (int32_t)p;
    std::vector<int32_t> fa(out.atom_off.begin(), out.atom_off.end() - 1);
    for (int64_t j = 0; j < m; ++j) out.atom_list[fa[owner[j]]++] = (int32_t)j;
  }
  out.foot_off.assign(G + 1, 0);
  out.foot_list.clear();
  out.atom_lf.assign((size_t)m * width, (int16_t)-1);
  out.max_foot = 0;
  std::vector<int32_t> fp;
  for (int c = 0; c < G; ++c) {
    fp.clear();
    for (int q = out.atom_off[c]; q < out.atom_off[c + 1]; ++q) {
      const int32_t j = out.atom_list[q];
      for (int l = 0; l < width; ++l)
        if (ell_idx[(int64_t)j * width + l] >= 0) fp.push_back(ell_idx[(int64_t)j * width + l]);
    }
    std::sort(fp.begin(), fp.end());
    fp.erase(std::unique(fp.begin(), fp.end()), fp.end());
    if (fp.size() > 32767) return fail(SF_EUNSUPPORTED, "on-chip FISTA plan: footprint too large");
    for (int q = out.atom_off[c]; q < out.atom_off[c + 1]; ++q) {
      const int32_t j = out.atom_list[q];
      for (int l = 0; l < width; ++l) {
        const int32_t p = ell_idx[(int64_t)j * width + l];
        if (p >= 0)
          out.atom_lf[(size_t)q * width + l] =
              (int16_t)(std::lower_bound(fp.begin(), fp.end(), p) - fp.begin());
      }
    }
    out.foot_list.insert(out.foot_list.end(), fp.begin(), fp.end());
    out.foot_off[c + 1] = (int32_t)out.foot_list.size();
    out.max_foot = std::max(out.max_foot, (int)fp.size());
  }
  return SF_OK;
}

}  // namespace sf
