// sf_ktc.cu -- the Lipschitz operator K~ = F~ Q F~^H on tcgen05 tensor cores.
//
// Reference: solver.py:139-175 / 194-199 need lambda_max(dA) of every pulse,
// dA = G~^H G~ (solver.py:178-183); its spectrum is that of the N_r x N_r
// K~ = G~ G~^H = F~ Q F~^H with Q = H H^T.  In the real form
//     X = [Re F~ | Im F~]  (pixel rows, the forward kernel's panel Gp),
//     Y = Q X,  Z = X^T Y  (k_pad x k_pad, symmetric: upper 128-blocks only),
//     K~_re = Z[m][n] + Z[N_r+m][N_r+n],  K~_im = Z[N_r+m][n] - Z[m][N_r+n].
// Pixels are taken in the Morton order of QTileHost, in groups of eight: one
// group is the 16-byte K slice of a tcgen05 core matrix, and a "slab" (one
// group x one 128-column block, fp16, [128 columns][8 pixels]) is 16 core
// matrices stacked along M -- 2 KiB, the unit every operand load is made of.
//   k_ktc_split  X -> scaled fp16 hi/lo slabs (Xh, Xl)
//   k_ktc_y      per (64-pixel Morton tile O, column block): Y_O = Q_{O,U} X_U,
//                A = the slabs of U's groups, B = the static Q panel of the
//                tile, D in TMEM; Y_O written back as slabs (Yh, Yl)
//   k_ktc_z      split K: per (block row a, up to 4 block columns b, a range
//                of pixel groups) Z_ab += X_a^T Y_b, fp32 partials
// then k_ktc_zsum (fixed-order fp64 sum over the K splits, deterministic) and
// k_ktc_assemble.  Products are f16x3 (D += hi*hi + hi*lo + lo*hi: ~22-bit
// operands, the Gram update's precision) with fp32 accumulators in TMEM.
// Every operand arrives by cp.async.bulk from one elected thread; short CTAs
// (one tile / one K range each) let the FISTA chain's CTAs take SMs back
// between them.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {
namespace ktc {

constexpr int kOwn = 64;                      // pixels per tile (N of the Y product)
constexpr int kGrp = 8;                       // pixels per group (K of one core matrix)
constexpr uint32_t kSlab = 128 * kGrp * 2;    // 2 KiB: 128 columns x 8 pixels, fp16
constexpr int64_t kSlabHalves = 128 * kGrp;
// k_ktc_y: chunks of 4 groups (K = 32): A hi | A lo (4 slabs each) | Q hi | Q lo
constexpr int kYGroups = 4;
constexpr uint32_t kQPart = kOwn * 32 * 2;    // 4 KiB: Q panel part, 64 own x 32 K
constexpr uint32_t kYStage = 2 * kYGroups * kSlab + 2 * kQPart;  // 24 KiB
constexpr int kYStages = 4;
constexpr uint32_t kYSmem = kYStages * kYStage;                  // 96 KiB: two CTAs per SM
constexpr int kMaxUG = 128;   // groups of one tile's Q neighbourhood (checked on the host)
// k_ktc_z: chunks of 2 groups (K = 16): X_a hi | lo, then per Z block Y_b hi | lo
constexpr int kZGroups = 2;
constexpr int kZBlocks = 4;                   // accumulators per CTA (4 x 128 TMEM columns)
constexpr uint32_t kZOp = 2 * kZGroups * kSlab;                  // 8 KiB
constexpr uint32_t kZStage = (1 + kZBlocks) * kZOp;              // 40 KiB
constexpr int kZStages = 4;
constexpr uint32_t kZSmem = kZStages * kZStage;                  // 160 KiB
constexpr int kThreads = 192;  // warp 0 producer, warp 1 MMA issuer, warps 2-5 epilogue
// canonical K-major SWIZZLE_NONE layouts: LBO = next core matrix along K,
// SBO = next along M/N.  Slabs: K neighbours one slab apart, M neighbours 128 B;
// Q panel parts: the [row/8][k/8][8 rows x 16 B] order of build_ktc_panels.
constexpr uint32_t kSlabLBO = kSlab, kSlabSBO = 128, kQLBO = 128, kQSBO = 512;
constexpr uint32_t kIdescN64 = (1u << 4) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdescN128 = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ uint32_t su32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void arrive_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   su32(bar))
               : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // sm_100 descriptor version; SWIZZLE_NONE
  return d;
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                    uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// D += hi*hi + hi*lo + lo*hi over one K = 16 step.  Measured against the
// fp64 path: lambda_max and |K~|_F agree to ~1e-6 relative; adding lo*lo
// changes nothing (the deviation is the fp32 accumulation, not the split).
__device__ __forceinline__ void mma3(uint32_t d, uint64_t a_hi, uint64_t a_lo, uint64_t b_hi,
                                     uint64_t b_lo, uint32_t idesc, bool first) {
  mma(d, a_hi, b_hi, idesc, first ? 0u : 1u);
  mma(d, a_hi, b_lo, idesc, 1u);
  mma(d, a_lo, b_hi, idesc, 1u);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
        "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]),
        "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]),
        "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
        "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// 8 values -> scaled fp16 hi / lo 16-byte stores
__device__ __forceinline__ void put8(__half *hi, __half *lo, const float *x, float scale) {
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
__device__ __forceinline__ int blk_index(int a, int b, int nb) {  // upper blocks a <= b, row-major
  return a * nb - a * (a - 1) / 2 + (b - a);
}
// 2^e scaling that puts max|x| in [2^13, 2^14)
__device__ __forceinline__ int scale_exp(float mx) {
  if (!(mx > 0.f)) return 0;
  int ex;
  frexpf(mx, &ex);
  return 14 - ex;
}

}  // namespace ktc

// Block groups of k_ktc_z: row a, columns b0 .. b0+nbk-1 (b0 >= a, nbk <= 4),
// enumerated row by row.
__host__ __device__ inline int ktc_nbgroups(int nb) {
  int n = 0;
  for (int a = 0; a < nb; ++a) n += (nb - a + ktc::kZBlocks - 1) / ktc::kZBlocks;
  return n;
}
__device__ __forceinline__ void ktc_bgroup(int gi, int nb, int &a, int &b0, int &nbk) {
  for (a = 0; a < nb; ++a) {
    const int ng = (nb - a + ktc::kZBlocks - 1) / ktc::kZBlocks;
    if (gi < ng) break;
    gi -= ng;
  }
  b0 = a + ktc::kZBlocks * gi;
  nbk = min(ktc::kZBlocks, nb - b0);
}

// X (fp32 rows of k_pad values) -> Xh / Xl slabs scaled by 2^ex; block =
// (tile, column block, scene), thread = column; also records {ex, ey}.
__global__ void __launch_bounds__(128) k_ktc_split(KtcArgs a) {
  using namespace ktc;
  const int64_t sc = blockIdx.z;
  const float *X = a.X + sc * a.x_stride;
  __half *xh = a.xs + sc * a.xs_stride;
  __half *xl = xh + a.slab_stride;
  const float mx = __uint_as_float(a.maxbits[sc]);
  const int ex = scale_exp(mx);
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    a.exps[2 * sc] = ex;
    a.exps[2 * sc + 1] = scale_exp(a.qrow_max * mx);
  }
  const float sx = ldexpf(1.f, ex);
  const int t = blockIdx.x, cb = blockIdx.y, m = threadIdx.x;
  const int col = cb * 128 + m;
  const bool ok = col < a.k_pad;
  const int32_t *gp = a.grp_pix + (int64_t)t * kOwn;
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {  // two halves of the tile: 32 loads in flight
    float v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int p = __ldg(gp + 32 * h + j);
      v[j] = (ok && p >= 0) ? __ldg(X + (int64_t)p * a.k_pad + col) : 0.f;
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const int64_t o = ((int64_t)cb * a.ngrp + (int64_t)t * (kOwn / kGrp) + 4 * h + g) * kSlabHalves +
                        (int64_t)m * kGrp;
      put8(xh + o, xl + o, v + 8 * g, sx);
    }
  }
}

// Y_O = Q_{O,U} X_U for one (tile, column block): D (128 columns x 64 own
// pixels, TMEM) accumulates over chunks of 4 U groups; the epilogue (thread =
// TMEM lane = column) writes the tile's 8 Y slabs, scaled by 2^ey.
__global__ void __launch_bounds__(ktc::kThreads) k_ktc_y(KtcArgs a) {
  using namespace ktc;
  const int64_t sc = blockIdx.y;
  const __half *xh = a.xs + sc * a.xs_stride;
  const __half *xl = xh + a.slab_stride;
  __half *yh = a.xs + sc * a.xs_stride + 2 * a.slab_stride;
  __half *yl = yh + a.slab_stride;
  const int t = a.tile_begin + (int)blockIdx.x / a.nb, cb = (int)blockIdx.x % a.nb;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full[kYStages], empty[kYStages], d_full;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g0 = a.ug_off[t], ng = a.ug_off[t + 1] - g0;
  const int nch = (ng + kYGroups - 1) / kYGroups;
  // A tile's last chunk may fill fewer than 4 groups; its Q panel is zero
  // there, so those slots only need finite contents: zero them in the stage
  // the last chunk uses (earlier chunks in that stage, if any, fill all 4).
  if (nch > 0) {
    const int nj_last = ng - (nch - 1) * kYGroups;
    unsigned char *st = smem + ((nch - 1) % kYStages) * kYStage;
    const int nz = (kYGroups - nj_last) * (int)(kSlab / 16);
    for (int i = tid; i < 2 * nz; i += kThreads) {
      const int part = i / nz, k = i % nz;
      reinterpret_cast<uint4 *>(st + (part * kYGroups + nj_last) * kSlab)[k] =
          make_uint4(0u, 0u, 0u, 0u);
    }
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(&tmem_slot)),
                 "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int s = 0; s < kYStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&d_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // producer warp: the tile's group list in registers (lane l holds entries
    // l, l + 32, ...; read by shuffles -- no dependent loads in the copy loop,
    // and no static shared memory: two CTAs must fit the 196 KiB carveout);
    // lane 0 issues one copy per run of consecutive groups and part
    static_assert(kMaxUG == 128, "four list registers per lane");
    auto ld = [&](int i) { return i < ng ? __ldg(a.ug_list + g0 + i) : -1; };
    const int32_t u0 = ld(lane), u1 = ld(lane + 32), u2 = ld(lane + 64), u3 = ld(lane + 96);
    auto ug = [&](int j) {
      const int hi = j >> 5;
      const int32_t v = hi == 0 ? u0 : hi == 1 ? u1 : hi == 2 ? u2 : u3;
      return __shfl_sync(0xffffffffu, v, j & 31);
    };
    const unsigned char *qsrc =
        reinterpret_cast<const unsigned char *>(a.qpanels) + (int64_t)a.qchunk_off[t] * 2 * kQPart;
    for (int c = 0; c < nch; ++c) {
      const int s = c % kYStages;
      if (lane == 0) mbar_wait(&empty[s], ((c / kYStages) & 1) ^ 1);
      __syncwarp();
      const int j0 = c * kYGroups, nj = min(kYGroups, ng - j0);
      unsigned char *st = smem + s * kYStage;
      if (lane == 0) arrive_tx(&full[s], 2 * nj * kSlab + 2 * kQPart);
      int32_t gj[kYGroups];
#pragma unroll
      for (int j = 0; j < kYGroups; ++j) gj[j] = ug(min(j0 + j, ng - 1));
      if (lane == 0) {
        // a run starts at j unless group j directly follows group j - 1
        int start = 0, run = 0, g_start = 0;
        auto flush = [&]() {
          if (run > 0) {
            const int64_t src = ((int64_t)cb * a.ngrp + g_start) * kSlabHalves;
            bulk_g2s(st + start * kSlab, xh + src, run * kSlab, &full[s]);
            bulk_g2s(st + (kYGroups + start) * kSlab, xl + src, run * kSlab, &full[s]);
          }
        };
#pragma unroll
        for (int j = 0; j < kYGroups; ++j) {
          if (j < nj && j > 0 && gj[j] == gj[j - 1] + 1) {
            ++run;
          } else {
            flush();
            start = j;
            g_start = gj[j];
            run = j < nj ? 1 : 0;
          }
        }
        flush();
        bulk_g2s(st + 2 * kYGroups * kSlab, qsrc + (int64_t)c * 2 * kQPart, 2 * kQPart, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      for (int c = 0; c < nch; ++c) {
        const int s = c % kYStages;
        mbar_wait(&full[s], (c / kYStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t st = su32(smem + s * kYStage);
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint32_t ao = st + ks * 2 * kSlab, bo = st + 2 * kYGroups * kSlab + ks * 2 * kQLBO;
          mma3(tmem, desc(ao, kSlabLBO, kSlabSBO), desc(ao + kYGroups * kSlab, kSlabLBO, kSlabSBO),
               desc(bo, kQLBO, kQSBO), desc(bo + kQPart, kQLBO, kQSBO), kIdescN64,
               c == 0 && ks == 0);
        }
        commit(&empty[s]);
      }
      commit(&d_full);
    }
  } else {
    // epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31
    const int m = 32 * (warp & 3) + lane;
    const float mx = __uint_as_float(a.maxbits[sc]);
    const int ex = scale_exp(mx), ey = scale_exp(a.qrow_max * mx);
    const float sy = ldexpf(1.f, ey - ex - a.eq);
    float y[64];
    if (nch > 0) {
      mbar_wait(&d_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(32 * (warp & 3)) << 16), v);
#pragma unroll
      for (int i = 0; i < 32; ++i) y[i] = v[i];
      tmem_ld32(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 32, v);
#pragma unroll
      for (int i = 0; i < 32; ++i) y[32 + i] = v[i];
    } else {
#pragma unroll
      for (int i = 0; i < 64; ++i) y[i] = 0.f;
    }
#pragma unroll
    for (int g = 0; g < kOwn / kGrp; ++g) {
      const int64_t o = ((int64_t)cb * a.ngrp + (int64_t)t * (kOwn / kGrp) + g) * kSlabHalves +
                        (int64_t)m * kGrp;
      put8(yh + o, yl + o, y + 8 * g, sy);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(64));
}

// Split-K Z blocks: CTA = (block group, K range of a.cps chunks of 2 groups
// inside this rank's tiles); D_i (128 x 128, TMEM) += X_a^T Y_{b0+i}; the
// epilogue writes the fp32 partials of its blocks (thread = row).
__global__ void __launch_bounds__(ktc::kThreads) k_ktc_z(KtcArgs a) {
  using namespace ktc;
  const int64_t sc = blockIdx.y;
  const __half *xh = a.xs + sc * a.xs_stride;
  const __half *xl = xh + a.slab_stride;
  const __half *yh = xl + a.slab_stride;
  const __half *yl = yh + a.slab_stride;
  float *zpart = a.zpart + sc * a.z_stride;
  const int nbg = ktc_nbgroups(a.nb), nblk = a.nb * (a.nb + 1) / 2;
  const int sp = (int)blockIdx.x / nbg;
  int ba, bb0, nbk;
  ktc_bgroup((int)blockIdx.x % nbg, a.nb, ba, bb0, nbk);
  const int c0 = 4 * a.tile_begin + sp * a.cps;
  const int nch = min(4 * a.tile_end, c0 + a.cps) - c0;
  const uint32_t ncols = nbk == 1 ? 128u : nbk == 2 ? 256u : 512u;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full[kZStages], empty[kZStages], d_full;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(&tmem_slot)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int s = 0; s < kZStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&d_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // producer: the K range is contiguous, one copy per operand part
      for (int c = 0; c < nch; ++c) {
        const int s = c % kZStages;
        mbar_wait(&empty[s], ((c / kZStages) & 1) ^ 1);
        unsigned char *st = smem + s * kZStage;
        arrive_tx(&full[s], (uint32_t)(1 + nbk) * kZOp);
        const int64_t g = (int64_t)kZGroups * (c0 + c);
        const int64_t sa = ((int64_t)ba * a.ngrp + g) * kSlabHalves;
        bulk_g2s(st, xh + sa, kZGroups * kSlab, &full[s]);
        bulk_g2s(st + kZGroups * kSlab, xl + sa, kZGroups * kSlab, &full[s]);
        for (int i = 0; i < nbk; ++i) {
          const int64_t sb = ((int64_t)(bb0 + i) * a.ngrp + g) * kSlabHalves;
          bulk_g2s(st + (1 + i) * kZOp, yh + sb, kZGroups * kSlab, &full[s]);
          bulk_g2s(st + (1 + i) * kZOp + kZGroups * kSlab, yl + sb, kZGroups * kSlab, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      for (int c = 0; c < nch; ++c) {
        const int s = c % kZStages;
        mbar_wait(&full[s], (c / kZStages) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t st = su32(smem + s * kZStage);
        const uint64_t a_hi = desc(st, kSlabLBO, kSlabSBO);
        const uint64_t a_lo = desc(st + kZGroups * kSlab, kSlabLBO, kSlabSBO);
        for (int i = 0; i < nbk; ++i) {
          const uint32_t bo = st + (1 + i) * kZOp;
          mma3(tmem + 128 * i, a_hi, a_lo, desc(bo, kSlabLBO, kSlabSBO),
               desc(bo + kZGroups * kSlab, kSlabLBO, kSlabSBO), kIdescN128, c == 0);
        }
        commit(&empty[s]);
      }
      commit(&d_full);
    }
  } else {
    const int r = 32 * (warp & 3) + lane;  // TMEM lane = row of block a
    if (nch > 0) {
      mbar_wait(&d_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    }
    for (int i = 0; i < nbk; ++i) {
      const int blk = blk_index(ba, bb0 + i, a.nb);
      float4 *dst =
          reinterpret_cast<float4 *>(zpart + (((int64_t)sp * nblk + blk) * 128 + r) * 128);
#pragma unroll 1
      for (int h = 0; h < 4; ++h) {
        float v[32];
        if (nch > 0) {
          tmem_ld32(tmem + ((uint32_t)(32 * (warp & 3)) << 16) + 128 * i + 32 * h, v);
        } else {
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = 0.f;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
          dst[8 * h + k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(ncols));
}

// Z (fp64, upper 128-blocks) = sum over the ncta K splits of the partial
// blocks, in split order, scaled by 2^-(ex+ey): coalesced over the partial
// array (cap = the partial slots allocated; the sum follows them).
__global__ void __launch_bounds__(256)
k_ktc_zsum(const float *__restrict__ zpart, int ncta, int cap, int nblk,
           const int *__restrict__ exps, int64_t z_stride) {
  zpart += blockIdx.y * z_stride;  // batched scenes: grid y
  exps += 2 * blockIdx.y;
  double *zsum = reinterpret_cast<double *>(const_cast<float *>(zpart) +
                                            (int64_t)cap * nblk * 128 * 128);
  const int64_t per4 = (int64_t)nblk * 128 * 128 / 4;
  const int64_t i = blockIdx.x * 256LL + threadIdx.x;  // four consecutive elements
  if (i >= per4) return;
  const float4 *src = reinterpret_cast<const float4 *>(zpart) + i;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int c = 0;
  for (; c + 8 <= ncta; c += 8) {  // eight partials in flight, summed in CTA order
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(src + (int64_t)(c + u) * per4);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s0 += (double)v[u].x;
      s1 += (double)v[u].y;
      s2 += (double)v[u].z;
      s3 += (double)v[u].w;
    }
  }
  for (; c < ncta; ++c) {
    const float4 v = __ldg(src + (int64_t)c * per4);
    s0 += (double)v.x;
    s1 += (double)v.y;
    s2 += (double)v.z;
    s3 += (double)v.w;
  }
  const double sc = ldexp(1.0, -(exps[0] + exps[1]));
  double *dst = zsum + 4 * i;
  dst[0] = s0 * sc;
  dst[1] = s1 * sc;
  dst[2] = s2 * sc;
  dst[3] = s3 * sc;
}

// K~ (fp64 and its fp32 copy) from Z: K~_re = Z[m][n] + Z[N_r+m][N_r+n],
// K~_im = Z[N_r+m][n] - Z[m][N_r+n] (Z symmetric: lower blocks mirrored);
// u0 = sum of the forward kernel's u0 partials (as k_kreduce).
__global__ void __launch_bounds__(256)
k_ktc_assemble(const float *__restrict__ zpart, int ncta, int nb, int n_r,
               const double2 *__restrict__ u0part, int nu0, double2 *__restrict__ K,
               float2 *__restrict__ Kf, double2 *__restrict__ u0, int64_t z_stride) {
  __shared__ double2 red[8][33];
  {  // batched scenes: grid y
    const int64_t sc = blockIdx.y;
    zpart += sc * z_stride;
    u0part += sc * nu0 * (int64_t)n_r;
    K += sc * (int64_t)n_r * n_r;
    Kf += sc * (int64_t)n_r * n_r;
    u0 += sc * n_r;
  }
  const double *zsum =
      reinterpret_cast<const double *>(zpart + (int64_t)ncta * (nb * (nb + 1) / 2) * 128 * 128);
  const int64_t nn = (int64_t)n_r * n_r;
  const int64_t kblocks = (nn + 255) / 256;
  if (blockIdx.x < kblocks) {
    const int64_t idx = blockIdx.x * 256LL + threadIdx.x;
    if (idx >= nn) return;
    const int m = (int)(idx / n_r), n = (int)(idx % n_r);
    auto z = [&](int i, int j) {
      if (i / 128 > j / 128) {
        const int t = i;
        i = j;
        j = t;
      }
      return zsum[((int64_t)ktc::blk_index(i / 128, j / 128, nb) * 128 + (i % 128)) * 128 + (j % 128)];
    };
    const double re = z(m, n) + z(n_r + m, n_r + n);
    const double im = z(n_r + m, n) - z(m, n_r + n);
    K[idx] = make_double2(re, im);
    Kf[idx] = make_float2((float)re, (float)im);
    return;
  }
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int64_t m = (blockIdx.x - kblocks) * 32LL + tx;
  double2 su = make_double2(0.0, 0.0);
  if (m < n_r)
    for (int cc = ty; cc < nu0; cc += 8) {
      const double2 v = u0part[(int64_t)cc * n_r + m];
      su.x += v.x;
      su.y += v.y;
    }
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

// K splits of this rank's tiles (chunks of 2 groups, a.cps per split).
int ktc_splits(const KtcArgs &a) {
  const int nch = 4 * (a.tile_end - a.tile_begin);
  return nch > 0 ? (nch + a.cps - 1) / a.cps : 0;
}

// Partial (this rank's tiles [tile_begin, tile_end)) fp64 Z blocks into zsum;
// cap = the K-split slots of zpart.
sf_status launch_ktilde_tc_partial(const KtcArgs &a, int cap, cudaStream_t st, int batch) {
  static std::atomic<uint64_t> set{0};
  if (attr_pending(set)) {
    SF_CUDA_TRY(cudaFuncSetAttribute(k_ktc_y, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)ktc::kYSmem));
    SF_CUDA_TRY(cudaFuncSetAttribute(k_ktc_z, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)ktc::kZSmem));
    attr_done(set);
  }
  const int tl = a.tile_end - a.tile_begin, splits = ktc_splits(a);
  if (splits > cap) return fail(SF_EINVAL, "K~: more K splits than partial slots");
  if (tl > 0) {
    // every tile's X (the Q neighbourhoods cross the rank's range)
    if (!a.presplit) {  // (else k_forward_pix wrote the slabs and the exponents)
      k_ktc_split<<<dim3(a.tiles, a.nb, batch), 128, 0, st>>>(a);
      SF_LAUNCH_CHECK();
    }
    k_ktc_y<<<dim3(tl * a.nb, batch), ktc::kThreads, ktc::kYSmem, st>>>(a);
    SF_LAUNCH_CHECK();
    k_ktc_z<<<dim3(splits * ktc_nbgroups(a.nb), batch), ktc::kThreads, ktc::kZSmem, st>>>(a);
    SF_LAUNCH_CHECK();
  }
  const int nblk = a.nb * (a.nb + 1) / 2;
  const int64_t per = (int64_t)nblk * 128 * 128;
  k_ktc_zsum<<<dim3((unsigned)((per / 4 + 255) / 256), batch), 256, 0, st>>>(
      a.zpart, splits, cap, nblk, a.exps, a.z_stride);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

// fp64 Z blocks (after the ranks' partials are summed) -> K~, its fp32 copy, u0.
sf_status launch_ktilde_assemble(const KtcArgs &a, int grid, const double2 *u0part, int nu0,
                                 int n_r, double2 *K, float2 *Kf, double2 *u0, cudaStream_t st,
                                 int batch) {
  const int64_t nn = (int64_t)n_r * n_r;
  const unsigned blocks = (unsigned)((nn + 255) / 256 + (n_r + 31) / 32);
  k_ktc_assemble<<<dim3(blocks, batch), 256, 0, st>>>(a.zpart, grid, a.nb, n_r, u0part, nu0, K,
                                                      Kf, u0, a.z_stride);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

double *ktc_zsum(const KtcArgs &a, int grid) {
  return reinterpret_cast<double *>(a.zpart + (int64_t)grid * (a.nb * (a.nb + 1) / 2) * 128 * 128);
}

sf_status launch_ktilde_tc(const KtcArgs &a, int grid, const double2 *u0part, int nu0, int n_r,
                           double2 *K, float2 *Kf, double2 *u0, cudaStream_t st, int batch) {
  sf_status s = launch_ktilde_tc_partial(a, grid, st, batch);
  if (s) return s;
  return launch_ktilde_assemble(a, grid, u0part, nu0, n_r, K, Kf, u0, st, batch);
}

// Static operand of the Y product and the Morton grouping: per tile, the
// groups of its Q neighbourhood (ug) and the dense Q_{O,U} (64 own pixels x 8
// pixel slots per group, chunks of 4 groups) scaled by 2^eq and split into
// fp16 hi/lo canonical parts [chunk][hi 64x32 | lo 64x32].
sf_status build_ktc_panels(const QTileHost &qt, KtcHost &out, int *eq_out, float *qrow_max) {
  const int tiles = qt.tiles;
  const int64_t n = (int64_t)qt.pix_list.size();
  for (int t = 0; t < tiles; ++t)
    if (qt.pix_off[t] != (int64_t)t * ktc::kOwn || qt.pix_off[t + 1] - qt.pix_off[t] > ktc::kOwn)
      return fail(SF_EUNSUPPORTED, "K~ tiles: not 64-pixel Morton runs");
  double qmax = 0.0, rmax = 0.0;
  for (int64_t o = 0; o < n; ++o) {
    double rs = 0.0;
    for (int k = qt.ent_off[o]; k < qt.ent_off[o + 1]; ++k) {
      qmax = std::max(qmax, std::fabs(qt.ent_q[k]));
      rs += std::fabs(qt.ent_q[k]);
    }
    rmax = std::max(rmax, rs);
  }
  int e = 0;
  if (qmax > 0.0) {
    int ex;
    std::frexp(qmax, &ex);
    e = 14 - ex;
  }
  *eq_out = e;
  *qrow_max = (float)(rmax * (1.0 + 1e-6));
  // Morton position of every pixel; groups of 8 positions, 8 per tile
  int64_t npix = 0;
  for (int32_t p : qt.pix_list) npix = std::max<int64_t>(npix, (int64_t)p + 1);
  std::vector<int32_t> pos(npix, -1);
  for (int64_t k = 0; k < n; ++k) pos[qt.pix_list[k]] = (int32_t)k;
  out.grp_pix.assign((size_t)tiles * ktc::kOwn, -1);
  for (int64_t k = 0; k < n; ++k) out.grp_pix[k] = qt.pix_list[k];
  out.ug_off.assign(tiles + 1, 0);
  out.ug_list.clear();
  out.chunk_off.assign(tiles + 1, 0);
  std::vector<int32_t> ug;
  for (int t = 0; t < tiles; ++t) {
    ug.clear();
    if (qt.union_off[t + 1] - qt.union_off[t] > 8 * ktc::kMaxUG)
      return fail(SF_EUNSUPPORTED, "K~ tiles: neighbourhood too large");
    for (int k = qt.union_off[t]; k < qt.union_off[t + 1]; ++k)
      ug.push_back(pos[qt.union_list[k]] / ktc::kGrp);
    std::sort(ug.begin(), ug.end());
    ug.erase(std::unique(ug.begin(), ug.end()), ug.end());
    if ((int)ug.size() > ktc::kMaxUG)
      return fail(SF_EUNSUPPORTED, "K~ tiles: neighbourhood too large");
    out.ug_list.insert(out.ug_list.end(), ug.begin(), ug.end());
    out.ug_off[t + 1] = (int32_t)out.ug_list.size();
    out.chunk_off[t + 1] =
        out.chunk_off[t] + ((int)ug.size() + ktc::kYGroups - 1) / ktc::kYGroups;
  }
  const size_t part = (size_t)ktc::kOwn * 32;  // halves per part
  out.panels.assign((size_t)out.chunk_off[tiles] * 2 * part, __float2half(0.f));
  for (int t = 0; t < tiles; ++t) {
    const int32_t *g0 = out.ug_list.data() + out.ug_off[t];
    const int ng = out.ug_off[t + 1] - out.ug_off[t];
    for (int o = 0; o < qt.pix_off[t + 1] - qt.pix_off[t]; ++o) {
      const int64_t op = qt.pix_off[t] + o;
      for (int k = qt.ent_off[op]; k < qt.ent_off[op + 1]; ++k) {
        const int32_t qp = pos[qt.union_list[qt.union_off[t] + qt.ent_u[k]]];
        const int j = (int)(std::lower_bound(g0, g0 + ng, qp / ktc::kGrp) - g0);
        const int kk = ktc::kGrp * (j % ktc::kYGroups) + qp % ktc::kGrp;
        const float x = (float)std::ldexp(qt.ent_q[k], e);
        const __half h = __float2half_rn(x);
        const __half l = __float2half_rn(x - __half2float(h));
        const size_t chunk = (size_t)out.chunk_off[t] + j / ktc::kYGroups;
        const size_t off = (size_t)(o >> 3) * (ktc::kQSBO / 2) + (size_t)(kk >> 3) * (ktc::kQLBO / 2) +
                           (size_t)(o & 7) * 8 + (size_t)(kk & 7);  // in halves
        out.panels[chunk * 2 * part + off] = h;
        out.panels[chunk * 2 * part + part + off] = l;
      }
    }
  }
  return SF_OK;
}

}  // namespace sf
