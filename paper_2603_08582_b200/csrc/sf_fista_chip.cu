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

__device__ __forceinline__ void chip_mark(const ChipFistaArgs &a, int &n) {
  if (a.trace != nullptr && threadIdx.x == 0 && n < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[blockIdx.x * 64 + n] = t;
  }
  ++n;
}

// shared-memory carve-up of the per-CTA index data (after the resident tiles)
struct ChipSmem {
  double *ent_w, *atom_wl, *z, *cprev, *bre, *yf;
  int32_t *ent_atom, *foot, *atom_id, *pe;
  int16_t *atom_lf;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~(size_t)15; }

__device__ __forceinline__ ChipSmem chip_carve(unsigned char *base, const ChipFistaArgs &a) {
  ChipSmem m;
  size_t o = 0;
  auto take = [&](size_t bytes) {
    unsigned char *p = base + o;
    o += align16(bytes);
    return p;
  };
  m.ent_w = reinterpret_cast<double *>(take((size_t)a.max_ent * 8));
  m.atom_wl = reinterpret_cast<double *>(take((size_t)a.max_atoms * a.width * 8));
  m.z = reinterpret_cast<double *>(take((size_t)a.max_atoms * 8));
  m.cprev = reinterpret_cast<double *>(take((size_t)a.max_atoms * 8));
  m.bre = reinterpret_cast<double *>(take((size_t)a.max_atoms * 8));
  m.yf = reinterpret_cast<double *>(take((size_t)a.max_foot * 8));
  m.ent_atom = reinterpret_cast<int32_t *>(take((size_t)a.max_ent * 4));
  m.foot = reinterpret_cast<int32_t *>(take((size_t)a.max_foot * 4));
  m.atom_id = reinterpret_cast<int32_t *>(take((size_t)a.max_atoms * 4));
  m.pe = reinterpret_cast<int32_t *>(take((size_t)(a.max_pix + 1) * 4));
  m.atom_lf = reinterpret_cast<int16_t *>(take((size_t)a.max_atoms * a.width * 2));
  return m;
}

// x = H z at this CTA's own pixels, k_hz's summation order; entries in shared
// memory, z gathered from global (one dependent level)
__device__ __forceinline__ void chip_hz(const ChipFistaArgs &a, const ChipSmem &m, int p0, int np) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = warp; q < np; q += 16) {
    const int32_t p = a.pix_list[p0 + q];
    const int k0 = m.pe[q], k1 = m.pe[q + 1];
    double s = 0.0;
    int k = k0 + lane;
    for (; k + 32 < k1; k += 64) {
      const double z0 = __ldcg(a.zd + m.ent_atom[k]), z1 = __ldcg(a.zd + m.ent_atom[k + 32]);
      s += m.ent_w[k] * z0;
      s += m.ent_w[k + 32] * z1;
    }
    if (k < k1) s += m.ent_w[k] * __ldcg(a.zd + m.ent_atom[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) a.x[p] = (float)s;
  }
}

}  // namespace

__global__ void __launch_bounds__(512, 1) k_fista_chip(const ChipFistaArgs a) {
  extern __shared__ __align__(16) unsigned char chip_smem[];
  float4 *st = reinterpret_cast<float4 *>(chip_smem);
  const ChipSmem m = chip_carve(chip_smem + (size_t)a.smem_tiles * kTileElems * 4, a);
  __shared__ float s_row[2][8][kTile];
  __shared__ float s_col[2][kTile];
  cg::grid_group grid = cg::this_grid();
  const int c = blockIdx.x, G = gridDim.x, tid = threadIdx.x, grp = tid >> 8;
  const int lane = tid & 31, gw = (tid & 255) >> 5;
  int tn = 0;
  chip_mark(a, tn);

  // ---- once per launch: resident tiles and this CTA's index data
  for (int kk = 0; kk < a.smem_tiles; ++kk) {
    const int64_t t = c + (int64_t)G * kk;
    if (t >= a.n_tiles) break;
    const int2 ij = a.tiles[t];
    const float4 *src =
        reinterpret_cast<const float4 *>(a.B + tri_index(ij.x, ij.y, a.nt) * kTileElems);
    for (int e = tid; e < kTileElems / 4; e += 512) st[kk * (kTileElems / 4) + e] = src[e];
  }
  const int p0 = a.pix_off[c], np = a.pix_off[c + 1] - p0;
  const int q0 = a.atom_off[c], na = a.atom_off[c + 1] - q0;
  const int f0 = a.foot_off[c], nf = a.foot_off[c + 1] - f0;
  const int e0 = a.ent_off[c], ne = a.ent_off[c + 1] - e0;
  for (int i = tid; i < ne; i += 512) {
    m.ent_w[i] = a.ent_w[e0 + i];
    m.ent_atom[i] = a.ent_atom[e0 + i];
  }
  for (int i = tid; i <= np; i += 512) m.pe[i] = a.pe_off[p0 + c + i];
  for (int i = tid; i < nf; i += 512) m.foot[i] = a.foot_list[f0 + i];
  for (int i = tid; i < na * a.width; i += 512) {
    m.atom_wl[i] = a.atom_wl[(int64_t)q0 * a.width + i];
    m.atom_lf[i] = a.atom_lf[(int64_t)q0 * a.width + i];
  }
  for (int i = tid; i < na; i += 512) {
    const int32_t j = a.atom_list[q0 + i];
    m.atom_id[i] = j;
    m.bre[i] = a.b[j].x;
    const double z = a.first ? a.c0[j] : a.zd[j];
    m.z[i] = z;
    m.cprev[i] = a.first ? z : a.cprev[j];
    if (a.first) a.zd[j] = z;
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
  if (a.first) {
    if (c == 0)
      for (int64_t p = a.n + tid; p < a.n_pad; p += 512) a.x[p] = 0.f;
    grid.sync();
    chip_hz(a, m, p0, np);
    grid.sync();
  } else {
    __syncthreads();
  }
  chip_mark(a, tn);
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
    // ---- y at the footprint pixels: k_pix_reduce's order (slot lane g sums
    // slots g, g+8, ... in order; the eight lane sums are added in order).
    // Four (pixel, slot lane) pairs per thread, all slot loads issued first.
    for (int base = 0; base < nf * 8; base += 2048) {
      const float *src[4];
      bool ok[4];
      double sacc[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int e = base + tid + 512 * r;
        ok[r] = e < nf * 8;
        const int32_t p = ok[r] ? m.foot[e >> 3] : 0;
        src[r] = a.P + (int64_t)(p / kTile) * a.nt * kTile + (p % kTile);
        sacc[r] = 0.0;
      }
      const int g8 = tid & 7;
#pragma unroll 4
      for (int q = g8; q < a.nt; q += 8) {
        float v[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) v[r] = ok[r] ? __ldcg(src[r] + (int64_t)q * kTile) : 0.f;
#pragma unroll
        for (int r = 0; r < 4; ++r) sacc[r] += (double)v[r];
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        double part[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) part[u] = __shfl_sync(0xffffffffu, sacc[r], (lane & ~7) + u);
        const int e = base + tid + 512 * r;
        if (g8 == 0 && e < nf * 8) {
          double y = 0.0;
#pragma unroll
          for (int u = 0; u < 8; ++u) y += part[u];
          m.yf[e >> 3] = y;
        }
      }
    }
    __syncthreads();
    // ---- shrink + momentum for this CTA's atoms (k_atom_step, kernels.py:90-97)
    const double w = a.w[k];
    const bool last = a.last && (k == a.steps - 1);
    for (int i = tid; i < na; i += 512) {
      double y = 0.0;
      for (int l = 0; l < a.width; ++l) {
        const int lf = m.atom_lf[i * a.width + l];
        if (lf >= 0) y += m.atom_wl[i * a.width + l] * m.yf[lf];
      }
      const double z = m.z[i];
      const double u = z - tau * (y - m.bre[i]);
      double ci;
      if (u > thresh) ci = u - thresh;
      else if (u < -thresh) ci = u + thresh;
      else ci = 0.0;
      const double zn = ci + w * (ci - m.cprev[i]);
      m.cprev[i] = ci;
      m.z[i] = zn;
      const int32_t j = m.atom_id[i];
      a.zd[j] = zn;
      if (last) {
        a.c_out[j] = ci;
        a.cprev[j] = ci;
      } else if (k == a.steps - 1) {
        a.cprev[j] = ci;  // continuation chunk picks the state up from global
      }
    }
    chip_mark(a, tn);
    if (last) break;
    grid.sync();
    chip_mark(a, tn);
    chip_hz(a, m, p0, np);
    chip_mark(a, tn);
    grid.sync();
    chip_mark(a, tn);
  }
}

size_t chip_index_smem(int max_foot, int max_atoms, int max_pix, int max_ent, int width) {
  return align16((size_t)max_ent * 8) + align16((size_t)max_atoms * width * 8) +
         3 * align16((size_t)max_atoms * 8) + align16((size_t)max_foot * 8) +
         align16((size_t)max_ent * 4) + align16((size_t)max_foot * 4) +
         align16((size_t)max_atoms * 4) + align16((size_t)(max_pix + 1) * 4) +
         align16((size_t)max_atoms * width * 2);
}

sf_status launch_fista_chip(const ChipFistaArgs &a, int grid, cudaStream_t st) {
  const size_t dyn = (size_t)a.smem_tiles * kTileElems * 4 +
                     chip_index_smem(a.max_foot, a.max_atoms, a.max_pix, a.max_ent, a.width);
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

int fista_chip_fits(int device, int smem_tiles, size_t index_bytes) {
  const size_t dyn = (size_t)smem_tiles * kTileElems * 4 + index_bytes;
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

sf_status build_chip_plan(const double *xyz, int64_t n, const int32_t *ell_idx,
                          const double *ell_w, int64_t m, int width, const int64_t *csr_ptr,
                          const int32_t *csr_atom, const double *csr_w, int G, ChipPlanHost &out) {
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
  out.atom_wl.assign((size_t)m * width, 0.0);
  for (int64_t q = 0; q < m; ++q)
    for (int l = 0; l < width; ++l)
      out.atom_wl[(size_t)q * width + l] = ell_w[(int64_t)out.atom_list[q] * width + l];
  // H z entries of each CTA's own pixels, in global CSR order
  out.ent_off.assign(G + 1, 0);
  out.pe_off.assign((size_t)n + G, 0);
  out.ent_atom.clear();
  out.ent_w.clear();
  out.max_atoms = out.max_pix = out.max_ent = 0;
  for (int c = 0; c < G; ++c) {
    int local = 0;
    for (int q = out.pix_off[c]; q < out.pix_off[c + 1]; ++q) {
      out.pe_off[(size_t)q + c] = local;
      const int32_t p = out.pix_list[q];
      for (int64_t k = csr_ptr[p]; k < csr_ptr[p + 1]; ++k) {
        out.ent_atom.push_back(csr_atom[k]);
        out.ent_w.push_back(csr_w[k]);
        ++local;
      }
    }
    out.pe_off[(size_t)out.pix_off[c + 1] + c] = local;
    out.ent_off[c + 1] = out.ent_off[c] + local;
    out.max_ent = std::max(out.max_ent, local);
    out.max_pix = std::max(out.max_pix, out.pix_off[c + 1] - out.pix_off[c]);
    out.max_atoms = std::max(out.max_atoms, out.atom_off[c + 1] - out.atom_off[c]);
  }
  return SF_OK;
}

}  // namespace sf
