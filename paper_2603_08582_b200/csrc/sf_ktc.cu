// sf_ktc.cu -- the Lipschitz operator K~ = F~ Q F~^H on tcgen05 tensor cores.
//
// Reference: solver.py:139-175 / 194-199 need lambda_max(dA) of every pulse,
// dA = G~^H G~ (solver.py:178-183); its spectrum is that of the N_r x N_r
// K~ = G~ G~^H = F~ Q F~^H with Q = H H^T.  The SIMT path
// (k_fq + k_kgram_px, fp64) costs ~80 us of the whole GPU per cfg1 pulse and
// its CTAs crowd the FISTA chain; here the same operator is two small dense
// GEMMs per Morton tile of 64 pixels, in the real form
//     X = [Re F~ | Im F~]  (pixel rows, the Gram operand panel Gp),
//     Y_O = Q_{O,U} X_U    (own pixels O of the tile, U = their Q-neighbourhood)
//     Z  += X_O^T Y_O      (k_pad x k_pad, symmetric: upper 128-blocks only)
//     K~_re = Z[m][n] + Z[N_r+m][N_r+n],  K~_im = Z[N_r+m][n] - Z[m][N_r+n].
// Both products run as tcgen05 kind::f16 MMAs on scaled fp16 hi/lo splits
// (D += hi*hi + hi*lo + lo*hi: ~22-bit operands, the Gram update's
// precision) with fp32 accumulators in TMEM; per-CTA partial Z blocks are
// summed in fp64 in a fixed order by k_ktc_reduce (deterministic).
//
// CTA = 12 warps, persistent over tiles t = blockIdx.x + k*gridDim.x:
//   warp 0        loader: bulk copies of the X rows (U or O, one 128-column
//                 block, 512 B each) into a raw ring, and of the static
//                 Q_{O,U} panel chunks into the MMA ring
//   warp 1        TMEM owner + single-thread MMA issuer
//   warps 4-7     transposers: raw rows -> scaled fp16 hi/lo in the canonical
//                 K-major layout (thread = column)
//   warps 8-11    epilogue: D1 = Y^T (TMEM) -> fp16 hi/lo B operand of the
//                 second GEMM (shared memory); finally Z partials -> global
// TMEM: D1 at columns [0, 64), the CTA's (up to three) Z blocks at
// 128 + 128 * i.  Z has nb(nb+1)/2 upper 128-blocks (nb = k_pad / 128); a
// CTA owns one group of them -- one column block b of Y, row blocks a0..a0+2
// -- and recomputes that column block of Y for its tiles.
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {
namespace ktc {

constexpr int kOwn = 64;                                // pixels per tile (N of GEMM 1)
constexpr int kKC = 32;                                 // K per ring chunk (fp16)
constexpr uint32_t kAPart = 128 * kKC * 2;              // 8 KiB: 128 rows x 32 K, one part
constexpr uint32_t kQPart = kOwn * kKC * 2;             // 4 KiB
constexpr uint32_t kStageBytes = 2 * kAPart + 2 * kQPart;  // A hi|lo, Q hi|lo
constexpr int kStages = 4;
constexpr uint32_t kB2Bytes = 2 * 2 * kAPart;           // 2 K-chunks x (hi|lo) of 128 x 32
constexpr int kRaw = 3;                                 // raw X row stages (bulk copies)
constexpr uint32_t kRawBytes = kKC * 128 * 4;           // 32 rows x 128 fp32 = 16 KiB
constexpr uint32_t kSmem = kStages * kStageBytes + kB2Bytes + kRaw * kRawBytes;
constexpr uint32_t kLBO = 128, kSBO = 512;
constexpr int kThreads = 384;
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
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((kLBO >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((kSBO >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // sm_100 descriptor version; SWIZZLE_NONE
  return d;
}
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint32_t b, uint32_t idesc,
                                    uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(desc(a)), "l"(desc(b)), "r"(idesc), "r"(acc));
}
// D += hi*hi + hi*lo + lo*hi over one 32-wide K chunk (two K=16 MMAs each).
// Measured against the fp64 path: lambda_max and |K~|_F agree to 0.8-1.8e-6
// relative, slightly low; adding lo*lo changes nothing (the deviation is the
// fp32 accumulation, not the split).
__device__ __forceinline__ void mma3(uint32_t d, uint32_t a_hi, uint32_t a_lo, uint32_t b_hi,
                                     uint32_t b_lo, uint32_t idesc, bool first) {
#pragma unroll
  for (int ks = 0; ks < kKC / 16; ++ks) {
    const uint32_t off = ks * 2 * kLBO;
    mma(d, a_hi + off, b_hi + off, idesc, (first && ks == 0) ? 0u : 1u);
    mma(d, a_hi + off, b_lo + off, idesc, 1u);
    mma(d, a_lo + off, b_hi + off, idesc, 1u);
  }
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
// canonical K-major offset of (row r, k) inside one 32-wide chunk part
__device__ __forceinline__ uint32_t coff(int r, int k) {
  return (uint32_t)(r >> 3) * kSBO + (uint32_t)(k >> 3) * kLBO + (uint32_t)(r & 7) * 16 +
         (uint32_t)(k & 7) * 2;
}
// 8 consecutive K values of row r -> hi, lo 16-byte stores
__device__ __forceinline__ void put8(unsigned char *hi_part, unsigned char *lo_part, int r, int k0,
                                     const float *x) {
  __align__(16) __half h[8], l[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    h[i] = __float2half_rn(x[i]);
    l[i] = __float2half_rn(x[i] - __half2float(h[i]));
  }
  *reinterpret_cast<uint4 *>(hi_part + coff(r, k0)) = *reinterpret_cast<const uint4 *>(h);
  *reinterpret_cast<uint4 *>(lo_part + coff(r, k0)) = *reinterpret_cast<const uint4 *>(l);
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

// Chunk kc of the unit (tile t, group): kc < nkc -> union rows kc*32..,
// column block b; else own rows ((kc-nkc)%2)*32.., column block a0+(kc-nkc)/2.
struct KtcTile {
  int u0, nu, p0, np, nkc;
};
__device__ __forceinline__ KtcTile ktc_tile(const KtcArgs &a, int t) {
  KtcTile T;
  T.u0 = a.union_off[t];
  T.nu = a.union_off[t + 1] - T.u0;
  T.p0 = a.pix_off[t];
  T.np = a.pix_off[t + 1] - T.p0;
  T.nkc = (T.nu + ktc::kKC - 1) / ktc::kKC;
  return T;
}
struct KtcChunk {
  const int32_t *rows;  // row ids of the chunk (valid entries: n)
  int n, cb;
  bool g1;
};
// Group gi of Z blocks: one column block b of Y, row blocks a0 .. a0+na-1
// (na <= 3: TMEM holds D1 + three 128-column accumulators).  Groups enumerate
// b = 0..nb-1 and, per b, a0 = 0, 3, 6, ... <= b.
__host__ __device__ inline int ktc_ngroups(int nb) {
  int n = 0;
  for (int b = 0; b < nb; ++b) n += (b + 3) / 3;
  return n;
}
__device__ __forceinline__ void ktc_group(int gi, int nb, int &b, int &a0, int &na) {
  for (b = 0; b < nb; ++b) {
    const int ng = (b + 3) / 3;
    if (gi < ng) break;
    gi -= ng;
  }
  a0 = 3 * gi;
  na = min(3, b + 1 - a0);
}
__device__ __forceinline__ KtcChunk ktc_chunk(const KtcArgs &a, const KtcTile &T, int b, int a0,
                                              int kc) {
  KtcChunk c;
  c.g1 = kc < T.nkc;
  if (c.g1) {
    c.rows = a.union_list + T.u0 + kc * ktc::kKC;
    c.n = min(ktc::kKC, T.nu - kc * ktc::kKC);
    c.cb = b;
  } else {
    const int k0 = ((kc - T.nkc) % (ktc::kOwn / ktc::kKC)) * ktc::kKC;
    c.rows = a.pix_list + T.p0 + k0;
    c.n = max(0, min(ktc::kKC, T.np - k0));
    c.cb = a0 + (kc - T.nkc) / (ktc::kOwn / ktc::kKC);
  }
  return c;
}

__global__ void __launch_bounds__(ktc::kThreads, 1) k_ktilde_tc(KtcArgs a) {
  using namespace ktc;
  {  // batched scenes: grid y
    const int64_t sc = blockIdx.y;
    a.X += sc * a.x_stride;
    a.maxbits += sc;
    a.zpart += sc * a.z_stride;
    a.exps += 2 * sc;
  }
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full[kStages], empty[kStages], raw_full[kRaw], raw_empty[kRaw], d1_full,
      b2_full, b2_free, z_full;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nb = a.nb, nblk = nb * (nb + 1) / 2;
  // CTA = (group, tile-CTA tc): tiles tc, tc + gx, ...
  const int gx = gridDim.x / a.ngroups;
  const int tc = blockIdx.x % gx;
  int gb, ga0, gna;
  ktc_group(blockIdx.x / gx, nb, gb, ga0, gna);
  const int nch2 = gna * (kOwn / kKC);  // own-row chunks per unit
  unsigned char *b2 = smem + kStages * kStageBytes;
  unsigned char *raw = b2 + kB2Bytes;
  const float mx = __uint_as_float(*a.maxbits);
  const int ex = scale_exp(mx);
  const int ey = scale_exp(a.qrow_max * mx);
  if (blockIdx.x == 0 && tid == 0) {  // per scene
    a.exps[0] = ex;
    a.exps[1] = ey;
  }

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     su32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 129);  // 128 transposers + the loader
      mbar_init(&empty[s], 1);
    }
    for (int r = 0; r < kRaw; ++r) {
      mbar_init(&raw_full[r], 1);
      mbar_init(&raw_empty[r], 128);
    }
    mbar_init(&d1_full, 1);
    mbar_init(&b2_full, 128);
    mbar_init(&b2_free, 1);
    mbar_init(&z_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // ---------------- loader (lane j copies row j of a chunk) ----------------
    uint32_t g = 0;
    for (int t = a.tile_begin + tc; t < a.tile_end; t += gx) {
      const KtcTile T = ktc_tile(a, t);
      const unsigned char *qsrc =
          reinterpret_cast<const unsigned char *>(a.qpanels) + (int64_t)a.qchunk_off[t] * 2 * kQPart;
      {
        for (int kc = 0; kc < T.nkc + nch2; ++kc, ++g) {
          const KtcChunk ch = ktc_chunk(a, T, gb, ga0, kc);
          const int ncol = max(0, min(128, a.k_pad - 128 * ch.cb));
          const int row = lane < ch.n ? ch.rows[lane] : 0;
          const int r = g % kRaw;
          mbar_wait(&raw_empty[r], ((g / kRaw) & 1) ^ 1);
          if (lane == 0) arrive_tx(&raw_full[r], (uint32_t)(ch.n * ncol * 4));
          __syncwarp();
          if (lane < ch.n)
            bulk_g2s(raw + r * kRawBytes + lane * 512, a.X + (int64_t)row * a.k_pad + 128 * ch.cb,
                     (uint32_t)(ncol * 4), &raw_full[r]);
          if (lane == 0) {
            const int s = g % kStages;
            mbar_wait(&empty[s], ((g / kStages) & 1) ^ 1);
            if (ch.g1) {
              arrive_tx(&full[s], 2 * kQPart);
              bulk_g2s(smem + s * kStageBytes + 2 * kAPart, qsrc + (int64_t)kc * 2 * kQPart,
                       2 * kQPart, &full[s]);
            } else {
              arrive(&full[s]);
            }
          }
          __syncwarp();
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t sbase = su32(smem), b2base = su32(b2);
      uint32_t g = 0, unit = 0;
      bool zfirst[3] = {true, true, true};
      for (int t = a.tile_begin + tc; t < a.tile_end; t += gx) {
        const int nkc = ktc_tile(a, t).nkc;
        {
          // GEMM 1: D1 (128 x 64) = X_U^T[c-block b] . Q_{O,U}^T
          for (int kc = 0; kc < nkc; ++kc, ++g) {
            const int s = g % kStages;
            mbar_wait(&full[s], (g / kStages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
            const uint32_t st = sbase + s * kStageBytes;
            mma3(tmem, st, st + kAPart, st + 2 * kAPart, st + 2 * kAPart + kQPart, kIdescN64,
                 kc == 0);
            commit(&empty[s]);
          }
          commit(&d1_full);
          mbar_wait(&b2_full, unit & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          // GEMM 2: Z_{a2,b} += X_O^T[c-block a2] . Y_O[c-block b], a2 = a0 + i
          for (int i = 0; i < gna; ++i) {
            const int blk = i;  // TMEM slot
            const uint32_t zd = tmem + 128 + 128 * blk;
            for (int kc2 = 0; kc2 < kOwn / kKC; ++kc2, ++g) {
              const int s = g % kStages;
              mbar_wait(&full[s], (g / kStages) & 1);
              asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
              const uint32_t st = sbase + s * kStageBytes;
              const uint32_t bb = b2base + kc2 * 2 * kAPart;
              mma3(zd, st, st + kAPart, bb, bb + kAPart, kIdescN128, zfirst[blk]);
              zfirst[blk] = false;
              commit(&empty[s]);
            }
          }
          commit(&b2_free);
          ++unit;
        }
      }
      commit(&z_full);
    }
  } else if (warp >= 4 && warp < 8) {
    // ---------------- transposers ----------------
    const int r = tid - 128;  // row of the 128-column block (= column of X)
    const float sx = ldexpf(1.f, ex);
    uint32_t g = 0;
    for (int t = a.tile_begin + tc; t < a.tile_end; t += gx) {
      const KtcTile T = ktc_tile(a, t);
      {
        for (int kc = 0; kc < T.nkc + nch2; ++kc, ++g) {
          const KtcChunk ch = ktc_chunk(a, T, gb, ga0, kc);
          const bool colok = 128 * ch.cb + r < a.k_pad;
          const int rr = g % kRaw;
          mbar_wait(&raw_full[rr], (g / kRaw) & 1);
          const float *src = reinterpret_cast<const float *>(raw + rr * kRawBytes) + r;
          float v[kKC];
#pragma unroll
          for (int j = 0; j < kKC; ++j) v[j] = (j < ch.n && colok) ? src[128 * j] * sx : 0.f;
          arrive(&raw_empty[rr]);
          const int s = g % kStages;
          mbar_wait(&empty[s], ((g / kStages) & 1) ^ 1);
          unsigned char *st = smem + s * kStageBytes;
#pragma unroll
          for (int q = 0; q < kKC / 8; ++q) put8(st, st + kAPart, r, 8 * q, v + 8 * q);
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          arrive(&full[s]);
        }
      }
    }
  } else if (warp >= 8) {
    // ---------------- epilogue ----------------
    const int q = warp & 3;
    const int r = 32 * q + lane;  // TMEM lane = row of the 128-column block
    const float sy = ldexpf(1.f, ey - ex - a.eq);
    uint32_t unit = 0;
    for (int t = a.tile_begin + tc; t < a.tile_end; t += gx, ++unit) {
      {
        mbar_wait(&d1_full, unit & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        float y[64];
        {
          float v[32];
          tmem_ld32(tmem + ((uint32_t)(32 * q) << 16), v);
#pragma unroll
          for (int i = 0; i < 32; ++i) y[i] = v[i] * sy;
          tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + 32, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) y[32 + i] = v[i] * sy;
        }
        if (unit > 0) mbar_wait(&b2_free, (unit - 1) & 1);
#pragma unroll
        for (int kc2 = 0; kc2 < kOwn / kKC; ++kc2) {
          unsigned char *part = b2 + kc2 * 2 * kAPart;
#pragma unroll
          for (int qq = 0; qq < kKC / 8; ++qq) put8(part, part + kAPart, r, 8 * qq, y + kc2 * kKC + 8 * qq);
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        arrive(&b2_full);
      }
    }
    mbar_wait(&z_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    for (int i = 0; i < gna; ++i) {
      const int blk = blk_index(ga0 + i, gb, nb);
      float4 *dst = reinterpret_cast<float4 *>(
          a.zpart + (((int64_t)tc * nblk + blk) * 128 + r) * 128);
      const bool any = a.tile_begin + tc < a.tile_end;  // a tile-CTA with no tiles writes zeros
#pragma unroll 1
      for (int h = 0; h < 4; ++h) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + 128 + 128 * i + 32 * h, v);
        if (!any)
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = 0.f;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          dst[8 * h + i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

// Z (fp64, upper 128-blocks) = sum over CTAs of the partial blocks, in CTA
// order, scaled by 2^-(ex+ey): coalesced over the partial array.
__global__ void __launch_bounds__(256)
k_ktc_zsum(const float *__restrict__ zpart, int ncta, int nblk, const int *__restrict__ exps,
           int64_t z_stride) {
  zpart += blockIdx.y * z_stride;  // batched scenes: grid y
  exps += 2 * blockIdx.y;
  double *zsum = reinterpret_cast<double *>(const_cast<float *>(zpart) +
                                            (int64_t)ncta * nblk * 128 * 128);
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

// Partial (this rank's tiles [tile_begin, tile_end)) fp64 Z blocks into zsum.
sf_status launch_ktilde_tc_partial(const KtcArgs &a, int grid, cudaStream_t st, int batch) {
  static std::atomic<uint64_t> set{0};
  if (attr_pending(set)) {
    SF_CUDA_TRY(cudaFuncSetAttribute(k_ktilde_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)ktc::kSmem));
    attr_done(set);
  }
  // grid = tile-CTAs; each runs once per group of Z blocks
  k_ktilde_tc<<<dim3(grid * a.ngroups, batch), ktc::kThreads, ktc::kSmem, st>>>(a);
  SF_LAUNCH_CHECK();
  const int nblk = a.nb * (a.nb + 1) / 2;
  const int64_t per = (int64_t)nblk * 128 * 128;
  k_ktc_zsum<<<dim3((unsigned)((per / 4 + 255) / 256), batch), 256, 0, st>>>(a.zpart, grid, nblk,
                                                                             a.exps, a.z_stride);
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

// Static operand of GEMM 1: per tile, the dense Q_{O,U} (64 own pixels x the
// tile's union, zero-padded to 32) scaled by 2^eq and split into fp16 hi/lo
// canonical chunks [chunk][hi 64x32 | lo 64x32].
sf_status build_ktc_panels(const QTileHost &qt, std::vector<__half> &panels,
                           std::vector<int32_t> &chunk_off, int *eq_out, float *qrow_max) {
  double qmax = 0.0, rmax = 0.0;
  for (int t = 0; t < qt.tiles; ++t)
    for (int o = qt.pix_off[t]; o < qt.pix_off[t + 1]; ++o) {
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
  chunk_off.assign(qt.tiles + 1, 0);
  for (int t = 0; t < qt.tiles; ++t) {
    const int nu = qt.union_off[t + 1] - qt.union_off[t];
    chunk_off[t + 1] = chunk_off[t] + (nu + ktc::kKC - 1) / ktc::kKC;
  }
  const size_t part = (size_t)ktc::kOwn * ktc::kKC;  // halves per part
  panels.assign((size_t)chunk_off[qt.tiles] * 2 * part, __float2half(0.f));
  for (int t = 0; t < qt.tiles; ++t) {
    const int p0 = qt.pix_off[t], np = qt.pix_off[t + 1] - p0;
    if (np > ktc::kOwn) return fail(SF_EUNSUPPORTED, "K~ tiles: more than 64 pixels");
    for (int o = 0; o < np; ++o)
      for (int k = qt.ent_off[p0 + o]; k < qt.ent_off[p0 + o + 1]; ++k) {
        const int u = qt.ent_u[k];
        const float x = (float)std::ldexp(qt.ent_q[k], e);
        const __half h = __float2half_rn(x);
        const __half l = __float2half_rn(x - __half2float(h));
        const size_t chunk = (size_t)chunk_off[t] + u / ktc::kKC;
        const int kk = u % ktc::kKC;
        const size_t off = (size_t)(o >> 3) * (ktc::kSBO / 2) + (size_t)(kk >> 3) * (ktc::kLBO / 2) +
                           (size_t)(o & 7) * 8 + (size_t)(kk & 7);  // in halves
        panels[chunk * 2 * part + off] = h;
        panels[chunk * 2 * part + part + off] = l;
      }
  }
  return SF_OK;
}

}  // namespace sf
