// sf_gram.cu -- sufficient-statistics update of the packed symmetric Re(A).
//
// Reference: solver.py:178-183 (dA = G^H R^-1 G) and solver.py:191-193
// (A <- sym(A + dA)).  Only Re(A) feeds the solver (solver.py:214-222), and
//   Re(G^H G)/sigma^2 = P^T P,   P = [Re G~ ; Im G~]  (2 N_r x M, G~ = G/sigma),
// a real symmetric rank-2N_r update.  The engine stores Re(A) as the upper
// triangle of 128x128 fp32 tiles (I <= J); tile (I,J) += P[:,I]^T P[:,J].
//
// Two arithmetic paths (chosen by measured accuracy):
//   k_gram_tc<NPROD>: tcgen05 kind::tf32, 128x128 accumulator in TMEM.
//       NPROD = 3: error-compensated split x = hi + lo (hi = rna_tf32(x),
//       lo = rna_tf32(x - hi)), D += hi*hi + hi*lo + lo*hi.  NPROD = 1: hi*hi.
//       Operand panels are produced by the CTA's threads straight into shared
//       memory in the UMMA canonical K-major (no-swizzle) layout; one elected
//       thread issues the MMAs; completion is tracked with tcgen05.commit on
//       mbarriers; the epilogue is TMEM -> registers -> read-modify-write of the
//       HBM tile (coalesced 512 B per warp instruction).
//   k_gram_simt: fp32 FFMA, 4x16 register block per thread.
#include <cuda_fp16.h>

#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {

// ---------------------------------------------------------------------------
// SIMT fp32 path
__global__ void __launch_bounds__(256)
k_gram_simt(const float *__restrict__ Gp, int k_pad, const int2 *__restrict__ tiles, int nt,
            const float *Ain, float *A) {
  __shared__ float sa[kKChunk][kTile];
  __shared__ float sb[kKChunk][kTile];
  const int t = blockIdx.x;
  const int2 ij = tiles[t];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float *PA = Gp + (int64_t)ij.x * kTile * k_pad;
  const float *PB = Gp + (int64_t)ij.y * kTile * k_pad;
  float acc[4][16];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < 16; ++c) acc[i][c] = 0.f;
  for (int k0 = 0; k0 < k_pad; k0 += kKChunk) {
    for (int e = threadIdx.x; e < kTile * (kKChunk / 4); e += 256) {
      const int r = e / (kKChunk / 4), q = e % (kKChunk / 4);
      const float4 va = *reinterpret_cast<const float4 *>(PA + (int64_t)r * k_pad + k0 + 4 * q);
      const float4 vb = *reinterpret_cast<const float4 *>(PB + (int64_t)r * k_pad + k0 + 4 * q);
      sa[4 * q + 0][r] = va.x; sa[4 * q + 1][r] = va.y;
      sa[4 * q + 2][r] = va.z; sa[4 * q + 3][r] = va.w;
      sb[4 * q + 0][r] = vb.x; sb[4 * q + 1][r] = vb.y;
      sb[4 * q + 2][r] = vb.z; sb[4 * q + 3][r] = vb.w;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kKChunk; ++k) {
      float ar[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) ar[i] = sa[k][lane + 32 * i];
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        const float4 bv = *reinterpret_cast<const float4 *>(&sb[k][4 * (warp + 8 * s4)]);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          acc[i][4 * s4 + 0] += ar[i] * bv.x;
          acc[i][4 * s4 + 1] += ar[i] * bv.y;
          acc[i][4 * s4 + 2] += ar[i] * bv.z;
          acc[i][4 * s4 + 3] += ar[i] * bv.w;
        }
      }
    }
    __syncthreads();
  }
  float4 *T = reinterpret_cast<float4 *>(A + tri_index(ij.x, ij.y, nt) * kTileElems);
  const float4 *Ti = reinterpret_cast<const float4 *>(Ain + tri_index(ij.x, ij.y, nt) * kTileElems);
#pragma unroll
  for (int s4 = 0; s4 < 4; ++s4) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = lane + 32 * i;
      float4 *p = T + (int64_t)(warp + 8 * s4) * kTile + r;
      float4 v = Ti[(int64_t)(warp + 8 * s4) * kTile + r];
      v.x += acc[i][4 * s4 + 0];
      v.y += acc[i][4 * s4 + 1];
      v.z += acc[i][4 * s4 + 2];
      v.w += acc[i][4 * s4 + 3];
      *p = v;
    }
  }
}

// ---------------------------------------------------------------------------
// tcgen05 path
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory matrix descriptor, K-major, SWIZZLE_NONE:
// core matrix = 8 rows x 16 B (contiguous 128 B); LBO = byte distance between
// K-adjacent core matrices, SBO = between M/N-adjacent 8-row groups.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

// Instruction descriptor, kind::tf32: D f32, A/B tf32, both K-major, M=128, N=128.
constexpr uint32_t kIdescTf32 = (1u << 4)           // c_format = F32
                              | (2u << 7)           // a_format = TF32
                              | (2u << 10)          // b_format = TF32
                              | ((128u >> 3) << 17) // n_dim
                              | ((128u >> 4) << 24);// m_dim

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(kIdescTf32), "r"(accumulate));
}

__device__ __forceinline__ void commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint32_t rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return r;
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

// One K-chunk (16 tf32 = 4 core matrices along K) of a 128-row panel in the
// canonical layout: byte offset of (row r, core q) = (r/8)*512 + q*128 + (r%8)*16.
constexpr int kTfChunk = 16;  // tf32 elements per stage of k_gram_tc
constexpr uint32_t kLBO = 128, kSBO = 512;
constexpr uint32_t kPanelBytes = kTile * kTfChunk * 4;  // 8 KiB

}  // namespace tc

template <int NPROD>
__global__ void __launch_bounds__(128)
k_gram_tc(const float *__restrict__ Gp, int k_pad, const int2 *__restrict__ tiles, int nt,
          const float *Ain, float *A) {
  using namespace tc;
  // stage layout: [A_hi | A_lo | B_hi | B_lo] (lo panels only for NPROD == 3)
  constexpr int kPanels = (NPROD == 3) ? 4 : 2;
  constexpr uint32_t kStageBytes = kPanels * kPanelBytes;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t mbar[2];
  __shared__ uint32_t tmem_base_slot;

  const int tid = threadIdx.x, warp = tid >> 5;
  const int t = blockIdx.x;
  const int2 ij = tiles[t];
  const bool diag = (ij.x == ij.y);
  const float *PA = Gp + (int64_t)ij.x * kTile * k_pad;
  const float *PB = Gp + (int64_t)ij.y * kTile * k_pad;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tmem_base_slot)),
                 "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_base_slot;

  const int nchunks = k_pad / kTfChunk;
  const uint32_t sbase = smem_u32(smem);
  // Producer mapping: thread tid owns row tid of each panel; 4 x 16 B per row.
  const uint32_t row_off = (uint32_t)(tid >> 3) * kSBO + (uint32_t)(tid & 7) * 16;
  for (int c = 0; c < nchunks; ++c) {
    const int s = c & 1;
    if (c >= 2) mbar_wait(&mbar[s], (uint32_t)(((c >> 1) - 1) & 1));
    unsigned char *st = smem + s * kStageBytes;
    const int k0 = c * kTfChunk;
#pragma unroll
    for (int side = 0; side < 2; ++side) {
      if (side == 1 && diag) break;
      const float *src = (side == 0 ? PA : PB) + (int64_t)tid * k_pad + k0;
      unsigned char *hi = st + (side == 0 ? 0 : (kPanels / 2)) * kPanelBytes;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 v = __ldg(reinterpret_cast<const float4 *>(src + 4 * q));
        uint4 h;
        h.x = rna_tf32(v.x);
        h.y = rna_tf32(v.y);
        h.z = rna_tf32(v.z);
        h.w = rna_tf32(v.w);
        *reinterpret_cast<uint4 *>(hi + row_off + q * kLBO) = h;
        if (NPROD == 3) {
          uint4 l;
          l.x = rna_tf32(v.x - __uint_as_float(h.x));
          l.y = rna_tf32(v.y - __uint_as_float(h.y));
          l.z = rna_tf32(v.z - __uint_as_float(h.z));
          l.w = rna_tf32(v.w - __uint_as_float(h.w));
          *reinterpret_cast<uint4 *>(hi + kPanelBytes + row_off + q * kLBO) = l;
        }
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t a_hi = sbase + s * kStageBytes;
      const uint32_t a_lo = a_hi + kPanelBytes;
      const uint32_t b_hi = diag ? a_hi : a_hi + (kPanels / 2) * kPanelBytes;
      const uint32_t b_lo = b_hi + kPanelBytes;
#pragma unroll
      for (int kk = 0; kk < kTfChunk / 8; ++kk) {
        const uint32_t off = kk * 2 * kLBO;  // K = 8 tf32 = 2 core matrices
        const uint32_t acc = (c > 0 || kk > 0) ? 1u : 0u;
        mma_tf32(tmem, make_desc(a_hi + off, kLBO, kSBO), make_desc(b_hi + off, kLBO, kSBO), acc);
        if (NPROD == 3) {
          mma_tf32(tmem, make_desc(a_hi + off, kLBO, kSBO), make_desc(b_lo + off, kLBO, kSBO), 1u);
          mma_tf32(tmem, make_desc(a_lo + off, kLBO, kSBO), make_desc(b_hi + off, kLBO, kSBO), 1u);
        }
      }
      commit(&mbar[s]);
    }
  }
  {
    const int cl = nchunks - 1;
    mbar_wait(&mbar[cl & 1], (uint32_t)((cl >> 1) & 1));
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");

  // Epilogue: warp w owns TMEM lanes 32w..32w+31 = tile rows; 4 x 32 columns.
  const int r = tid;  // row = 32*warp + lane
  float4 *T = reinterpret_cast<float4 *>(A + tri_index(ij.x, ij.y, nt) * kTileElems);
  const float4 *Ti = reinterpret_cast<const float4 *>(Ain + tri_index(ij.x, ij.y, nt) * kTileElems);
#pragma unroll 1
  for (int cc = 0; cc < 4; ++cc) {
    float4 old[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) old[q] = Ti[(int64_t)(cc * 8 + q) * kTile + r];
    float v[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(cc * 32), v);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      float4 o = old[q];
      o.x += v[4 * q + 0];
      o.y += v[4 * q + 1];
      o.z += v[4 * q + 2];
      o.w += v[4 * q + 3];
      T[(int64_t)(cc * 8 + q) * kTile + r] = o;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(128));
}

// Tile (I,I) sits at index I*nt - I*(I-1)/2 of the row-major upper-triangle list.
__global__ void k_symmetrize_diag(float *__restrict__ A, int nt) {
  const int I = blockIdx.x;
  float *T = A + ((int64_t)I * nt - (int64_t)I * (I - 1) / 2) * kTileElems;
  for (int e = threadIdx.x; e < kTileElems; e += blockDim.x) {
    const int r = e / kTile, c = e % kTile;
    if (c <= r) continue;
    const int64_t a = tile_offset(r, c), b = tile_offset(c, r);
    const float s = 0.5f * (T[a] + T[b]);
    T[a] = s;
    T[b] = s;
  }
}

sf_status launch_symmetrize_diag(float *A, int nt, cudaStream_t st) {
  if (nt == 0) return SF_OK;
  k_symmetrize_diag<<<nt, 256, 0, st>>>(A, nt);
  SF_LAUNCH_CHECK();
  return SF_OK;
}


// ---------------------------------------------------------------------------
// f16x3 path (default).  Operands are pre-split by k_split_panels into scaled
// fp16 hi/lo parts (x * 2^e = hi + lo, |lo| <= 2^-11 |hi|) stored in the UMMA
// canonical K-major layout, one contiguous 8 KiB block per (128-row block,
// 32-wide K chunk, part).  D += hi*hi + hi*lo + lo*hi carries ~22 significant
// bits like TF32x3, at the kind::f16 rate; the 2^-2e factor is folded into the
// epilogue.
//
// Persistent, warp-specialised, one CTA per SM:
//   warp 0      TMA producer: cp.async.bulk of the panel chunks into a 3-stage ring
//   warp 1      TMEM owner + single-thread tcgen05.mma issuer
//   warps 4-11  epilogue: tcgen05.ld -> scale -> read-modify-write of the HBM
//               tiles (16 x 16 B loads in flight per thread)
// Work item = 2x2 super-tile (tile rows 2SI, 2SI+1 x tile cols 2SJ, 2SJ+1,
// SI <= SJ): 4 accumulators of 128x128 fp32 = all 512 TMEM columns, 4 panel
// chunks per stage for 4 tiles (each panel read once per 2 tiles).
namespace f16 {
constexpr int kKC = kKChunk;                       // fp16 per chunk
constexpr uint32_t kPart = kTile * kKC * 2;        // 8 KiB
constexpr uint32_t kLBO = 128;                     // K-adjacent core matrices
constexpr uint32_t kSBO = (kKC / 8) * 128;         // 8-row groups
constexpr int kStages = 3;
constexpr uint32_t kStageBytes = 8 * kPart;        // A0,A1,B0,B1 x hi,lo
constexpr uint32_t kIdesc = (1u << 4)              // D f32
                          | (0u << 7) | (0u << 10) // A, B f16
                          | ((128u >> 3) << 17) | ((128u >> 4) << 24);
constexpr int kThreads = 384;

__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(acc));
}

__device__ __forceinline__ void arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(tc::smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(tc::smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          tc::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(tc::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ int64_t tile_index(int I, int J, int nt) {
  return (int64_t)I * nt - (int64_t)I * (I - 1) / 2 + (J - I);
}
}  // namespace f16

// (x * 2^e) -> fp16 hi/lo canonical panels; e chosen from max|x| so the
// largest entry lands in [2^13, 2^14).
__global__ void k_split_panels(const float *__restrict__ Gp, int64_t m_pad, int k_pad,
                               const unsigned *__restrict__ maxbits, int *__restrict__ exp_out,
                               __half *__restrict__ Gh) {
  {  // batched scenes: grid y
    const int64_t sc = blockIdx.y;
    Gp += sc * m_pad * k_pad;
    maxbits += sc;
    exp_out += sc;
    Gh += sc * m_pad * k_pad * 2;
  }
  const float mx = __uint_as_float(*maxbits);
  int e = 0;
  if (mx > 0.f) {
    int ex;
    frexpf(mx, &ex);  // mx in [2^(ex-1), 2^ex)
    e = 14 - ex;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *exp_out = e;
  const float s = ldexpf(1.f, e);
  const int groups = k_pad / 8;
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= m_pad * groups) return;
  const int64_t j = idx / groups;
  const int kg = (int)(idx - j * groups);
  const float4 *src = reinterpret_cast<const float4 *>(Gp + j * k_pad + kg * 8);
  const float4 v0 = src[0], v1 = src[1];
  const float x[8] = {v0.x * s, v0.y * s, v0.z * s, v0.w * s, v1.x * s, v1.y * s, v1.z * s, v1.w * s};
  __align__(16) __half hi[8], lo[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    hi[i] = __float2half_rn(x[i]);
    lo[i] = __float2half_rn(x[i] - __half2float(hi[i]));
  }
  const int64_t rb = j / kTile;
  const int r = (int)(j % kTile);
  const int k = kg * 8;
  const int kc = k / f16::kKC, kk = k % f16::kKC;
  const int nkc = k_pad / f16::kKC;
  const int64_t chunk = (rb * nkc + kc) * 2;  // part 0 = hi, 1 = lo
  const uint32_t off = (uint32_t)(r >> 3) * f16::kSBO + (uint32_t)(kk >> 3) * f16::kLBO +
                       (uint32_t)(r & 7) * 16;
  char *base = reinterpret_cast<char *>(Gh);
  *reinterpret_cast<uint4 *>(base + chunk * f16::kPart + off) = *reinterpret_cast<uint4 *>(hi);
  *reinterpret_cast<uint4 *>(base + (chunk + 1) * f16::kPart + off) = *reinterpret_cast<uint4 *>(lo);
}

__global__ void __launch_bounds__(f16::kThreads, 1)
k_gram_f16x3(const __half *__restrict__ Gh, int k_pad, int nt, const int2 *__restrict__ items,
             int n_items, const int *__restrict__ exp_in, const float *Ain, float *A, int batch,
             int64_t gh_stride, int64_t a_stride) {
  using namespace f16;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t full[kStages], empty[kStages], tmem_full, tmem_empty;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nkc = k_pad / kKC;

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     tc::smem_u32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&tmem_full, 1);
    tc::mbar_init(&tmem_empty, 256);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      uint32_t g = 0;
      for (int it = blockIdx.x; it < n_items * batch; it += gridDim.x) {
        const int sc = it / n_items;  // batched scenes share the item list
        const char *gbase = reinterpret_cast<const char *>(Gh + sc * gh_stride);
        const int2 st = items[it - sc * n_items];
        const int I0 = 2 * st.x, J0 = 2 * st.y;
        const bool diag = st.x == st.y;
        const bool a1 = I0 + 1 < nt, b1 = J0 + 1 < nt;
        for (int kc = 0; kc < nkc; ++kc, ++g) {
          const int s = g % kStages;
          tc::mbar_wait(&empty[s], ((g / kStages) & 1) ^ 1);
          unsigned char *dst = smem + s * kStageBytes;
          const uint32_t nparts = 2u * ((a1 ? 2 : 1) + (diag ? 0 : (b1 ? 2 : 1)));
          arrive_expect_tx(&full[s], nparts * kPart);
          const int rows[4] = {I0, I0 + 1, J0, J0 + 1};
          const bool ok[4] = {true, a1, !diag, !diag && b1};
#pragma unroll
          for (int o = 0; o < 4; ++o) {
            if (!ok[o]) continue;
            const char *src = gbase + ((int64_t)rows[o] * nkc + kc) * 2 * kPart;
            bulk_g2s(dst + (2 * o) * kPart, src, 2 * kPart, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t sbase = tc::smem_u32(smem);
      uint32_t g = 0, n = 0;
      for (int it = blockIdx.x; it < n_items * batch; it += gridDim.x, ++n) {
        const int2 st = items[it % n_items];
        const int I0 = 2 * st.x, J0 = 2 * st.y;
        const bool diag = st.x == st.y;
        const bool a1 = I0 + 1 < nt, b1 = J0 + 1 < nt;
        if (n > 0) tc::mbar_wait(&tmem_empty, (n - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        for (int kc = 0; kc < nkc; ++kc, ++g) {
          const int s = g % kStages;
          tc::mbar_wait(&full[s], (g / kStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t st0 = sbase + s * kStageBytes;
#pragma unroll
          for (int a = 0; a < 2; ++a) {
            if (a == 1 && !a1) continue;
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              if (b == 1 && !b1) continue;
              if (diag && a == 1 && b == 0) continue;  // lower tile of a diagonal block
              const uint32_t ah = st0 + (2 * a) * kPart;
              const uint32_t bh = diag ? st0 + (2 * b) * kPart : st0 + (2 * (2 + b)) * kPart;
              const uint32_t d = tmem + (uint32_t)(2 * a + b) * 128;
#pragma unroll
              for (int ks = 0; ks < kKC / 16; ++ks) {
                const uint32_t off = ks * 2 * kLBO;  // 16 fp16 = 2 core matrices
                const uint32_t acc = (kc > 0 || ks > 0) ? 1u : 0u;
                mma(d, tc::make_desc(ah + off, kLBO, kSBO), tc::make_desc(bh + off, kLBO, kSBO), acc);
                mma(d, tc::make_desc(ah + off, kLBO, kSBO),
                    tc::make_desc(bh + kPart + off, kLBO, kSBO), 1u);
                mma(d, tc::make_desc(ah + kPart + off, kLBO, kSBO),
                    tc::make_desc(bh + off, kLBO, kSBO), 1u);
              }
            }
          }
          tc::commit(&empty[s]);
        }
        tc::commit(&tmem_full);
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int ew = warp - 4;
    const int q = warp & 3;      // TMEM lane quarter == tile row group
    const int h = ew >> 2;       // column half
    const int r = 32 * q + lane; // tile row
    uint32_t n = 0;
    for (int it = blockIdx.x; it < n_items * batch; it += gridDim.x, ++n) {
      const int sc = it / n_items;
      const float inv2 = ldexpf(1.f, -2 * exp_in[sc]);
      const float *Ain_s = Ain + sc * a_stride;
      float *A_s = A + sc * a_stride;
      const int2 st = items[it - sc * n_items];
      const int I0 = 2 * st.x, J0 = 2 * st.y;
      const bool diag = st.x == st.y;
      const bool a1 = I0 + 1 < nt, b1 = J0 + 1 < nt;
      tc::mbar_wait(&tmem_full, n & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll 1
      for (int a = 0; a < 2; ++a) {
        if (a == 1 && !a1) continue;
#pragma unroll 1
        for (int b = 0; b < 2; ++b) {
          if (b == 1 && !b1) continue;
          if (diag && a == 1 && b == 0) continue;
          float4 *T = reinterpret_cast<float4 *>(A_s + tile_index(I0 + a, J0 + b, nt) * kTileElems);
          const float4 *Ti =
              reinterpret_cast<const float4 *>(Ain_s + tile_index(I0 + a, J0 + b, nt) * kTileElems);
          float4 old[16];
#pragma unroll
          for (int s = 0; s < 16; ++s) old[s] = Ti[(int64_t)(16 * h + s) * kTile + r];
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            float v[32];
            tc::tmem_ld32(tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(2 * a + b) * 128 +
                              (uint32_t)(64 * h + 32 * half),
                          v);
#pragma unroll
            for (int s = 0; s < 8; ++s) {
              float4 o = old[8 * half + s];
              o.x = fmaf(v[4 * s + 0], inv2, o.x);
              o.y = fmaf(v[4 * s + 1], inv2, o.y);
              o.z = fmaf(v[4 * s + 2], inv2, o.z);
              o.w = fmaf(v[4 * s + 3], inv2, o.w);
              T[(int64_t)(16 * h + 8 * half + s) * kTile + r] = o;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      arrive(&tmem_empty);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

sf_status launch_split_panels(const float *Gp, int64_t m_pad, int k_pad, const unsigned *maxbits,
                              int *exp_out, __half *Gh, cudaStream_t st, int batch) {
  const int64_t tot = m_pad * (k_pad / 8);
  const int bs = 256;
  k_split_panels<<<dim3((unsigned)((tot + bs - 1) / bs), batch), bs, 0, st>>>(
      Gp, m_pad, k_pad, maxbits, exp_out, Gh);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_gram_f16x3(const __half *Gh, int k_pad, int nt, const int2 *items, int n_items,
                            const int *exp_in, const float *Ain, float *A, int grid,
                            cudaStream_t st, int batch, int64_t gh_stride, int64_t a_stride) {
  if (n_items == 0) return SF_OK;
  const size_t smem = (size_t)f16::kStages * f16::kStageBytes;
  static std::atomic<uint64_t> set{0};
  if (attr_pending(set)) {
    SF_CUDA_TRY(cudaFuncSetAttribute(k_gram_f16x3, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    attr_done(set);
  }
  const int64_t tot = (int64_t)n_items * batch;
  const int g = (int)(tot < grid ? tot : grid);
  k_gram_f16x3<<<g, f16::kThreads, smem, st>>>(Gh, k_pad, nt, items, n_items, exp_in, Ain, A,
                                               batch, gh_stride, a_stride);
  SF_LAUNCH_CHECK();
  return SF_OK;
}

sf_status launch_gram(int precision, const float *Gp, int k_pad, const int2 *tiles,
                      int64_t n_tiles, int nt, const float *Ain, float *A, cudaStream_t st) {
  if (n_tiles == 0) return SF_OK;
  if (k_pad % kKChunk != 0) return fail(SF_EINVAL, "k_pad must be a multiple of 32");
  if (n_tiles > 0x7fffffffLL) return fail(SF_EINVAL, "too many tiles");
  const unsigned grid = (unsigned)n_tiles;
  if (precision == SF_PREC_FP32) {
    k_gram_simt<<<grid, 256, 0, st>>>(Gp, k_pad, tiles, nt, Ain, A);
  } else if (precision == SF_PREC_TF32X3) {
    const size_t smem = 2 * 4 * tc::kPanelBytes;
    static std::atomic<uint64_t> set{0};
    if (attr_pending(set)) {
      SF_CUDA_TRY(cudaFuncSetAttribute(k_gram_tc<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
      attr_done(set);
    }
    k_gram_tc<3><<<grid, 128, smem, st>>>(Gp, k_pad, tiles, nt, Ain, A);
  } else if (precision == SF_PREC_TF32) {
    const size_t smem = 2 * 2 * tc::kPanelBytes;
    k_gram_tc<1><<<grid, 128, smem, st>>>(Gp, k_pad, tiles, nt, Ain, A);
  } else {
    return fail(SF_EINVAL, "unknown precision");
  }
  SF_LAUNCH_CHECK();
  return SF_OK;
}

}  // namespace sf
