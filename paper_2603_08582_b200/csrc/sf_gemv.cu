// sf_gemv.cu -- the FISTA matvec y = Re(B) x (pixel space) or Re(A) z (atom
// space) on the packed symmetric tile store (kernels.py:86, np.dot(gram_re, z)).
//
// Layout: upper triangle of 128x128 fp32 tiles, tile (I, J >= I) a contiguous
// 64 KiB block [c/4][r][c%4].  Output: partial slots
// P[I][J][0..128) (row partial of tile (I,J), i.e. T x_J) and P[J][I][..]
// (column partial, T^T x_I); k_pix_reduce / k_fista_step sum the nt slots of
// every element in a fixed order, so every path is deterministic.
//
// Two kernels, chosen per launch by the number of tiles:
//   k_gemv_cta   one 256-thread CTA per tile (2 per SM), 16 float4 per thread
//                in flight, support-blind: for stores of a few hundred tiles
//                (cfg0/cfg1, L2-resident) where one warp per tile would leave
//                SMs idle and the step is latency-bound.
//   k_gemv_sym   one warp per tile, 16 tiles in flight per SM, with a sparse
//                path that reads only the live slabs / rows: for large stores
//                (cfg2 batched, cfg3, cfg4) where the sparse iterate makes most
//                of every tile's products exact zeros.
#include <string>

#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {

__device__ __forceinline__ bool slab_live(float4 v) {
  return v.x != 0.f || v.y != 0.f || v.z != 0.f || v.w != 0.f;
}

// ---- k_gemv_cta ----------------------------------------------------------------
// One 256-thread CTA per tile, 2 CTAs per SM.  Warp w covers column slabs
// {w, w+8, w+16, w+24} (16 columns); lane l covers rows {l, l+32, l+64, l+96}:
// 16 independent 16-byte loads per thread per tile.  The row partials of the 8
// warps are summed through shared memory, the column partials by a butterfly
// reduce-scatter.  The store is read-only during a FISTA call, so a CTA issues
// its first tile's loads before griddepcontrol.wait (under PDL they overlap the
// producer of x); only x and the slots depend on the producer.  Support-blind:
// these stores are L2-resident and the step latency-bound, where issuing the
// tile loads before x is known wins over skipping them.
__device__ __forceinline__ void cta_tile_compute(const float4 (&a)[4][4], int I, int J,
                                                  const float *__restrict__ z32,
                                                  float *__restrict__ P, int nt, int sym,
                                                  float (*s_row)[kTile], float *s_col) {
  const int gt = threadIdx.x;
  const int lane = gt & 31, warp = gt >> 5;
  {
    float zr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) zr[i] = __ldcg(z32 + (int64_t)I * kTile + lane + 32 * i);
    float4 zc[4];
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4)
      zc[s4] = __ldcg(reinterpret_cast<const float4 *>(z32 + (int64_t)J * kTile) + warp + 8 * s4);

    float rp[4];
    float cp[16];
#pragma unroll
    for (int i = 0; i < 4; ++i) rp[i] = 0.f;
#pragma unroll
    for (int k = 0; k < 16; ++k) cp[k] = 0.f;
    const bool diag_sym = sym && (I == J);
    if (diag_sym) {
      // keep c >= r for the row partial, c > r for the column partial
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = lane + 32 * i, c0 = 4 * (warp + 8 * s4);
          float4 v = a[s4][i];
          v.x = (c0 + 0 >= row) ? v.x : 0.f;
          v.y = (c0 + 1 >= row) ? v.y : 0.f;
          v.z = (c0 + 2 >= row) ? v.z : 0.f;
          v.w = (c0 + 3 >= row) ? v.w : 0.f;
          rp[i] += v.x * zc[s4].x + v.y * zc[s4].y + v.z * zc[s4].z + v.w * zc[s4].w;
          cp[4 * s4 + 0] += (c0 + 0 > row) ? v.x * zr[i] : 0.f;
          cp[4 * s4 + 1] += (c0 + 1 > row) ? v.y * zr[i] : 0.f;
          cp[4 * s4 + 2] += (c0 + 2 > row) ? v.z * zr[i] : 0.f;
          cp[4 * s4 + 3] += (c0 + 3 > row) ? v.w * zr[i] : 0.f;
        }
      }
    } else {
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 v = a[s4][i];
          rp[i] += v.x * zc[s4].x + v.y * zc[s4].y + v.z * zc[s4].z + v.w * zc[s4].w;
          cp[4 * s4 + 0] += v.x * zr[i];
          cp[4 * s4 + 1] += v.y * zr[i];
          cp[4 * s4 + 2] += v.z * zr[i];
          cp[4 * s4 + 3] += v.w * zr[i];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) s_row[warp][lane + 32 * i] = rp[i];

    const bool do_col = sym;
    if (do_col) {
      // butterfly reduce-scatter of 16 column partials over the 32 lanes
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const bool hi = lane & 16;
        const float send = hi ? cp[k] : cp[k + 8];
        const float keep = hi ? cp[k + 8] : cp[k];
        cp[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool hi = lane & 8;
        const float send = hi ? cp[k] : cp[k + 4];
        const float keep = hi ? cp[k + 4] : cp[k];
        cp[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const bool hi = lane & 4;
        const float send = hi ? cp[k] : cp[k + 2];
        const float keep = hi ? cp[k + 2] : cp[k];
        cp[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
      }
      {
        const bool hi = lane & 2;
        const float send = hi ? cp[0] : cp[1];
        const float keep = hi ? cp[1] : cp[0];
        cp[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
      }
      cp[0] += __shfl_xor_sync(0xffffffffu, cp[0], 1);
      if ((lane & 1) == 0) {
        const int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 +
                        ((lane >> 1) & 1);
        const int col = 4 * (warp + 8 * (idx >> 2)) + (idx & 3);
        if (diag_sym) s_col[col] = cp[0];
        else P[((int64_t)J * nt + I) * kTile + col] = cp[0];
      }
    }
    __syncthreads();
    if (gt < kTile) {
      float s = 0.f;
#pragma unroll
      for (int w = 0; w < 8; ++w) s += s_row[w][gt];
      if (diag_sym) s += s_col[gt];
      P[((int64_t)I * nt + J) * kTile + gt] = s;
    }
    __syncthreads();
  }
}


__global__ void __launch_bounds__(256, 2)
k_gemv_cta(const float *__restrict__ A, const int2 *__restrict__ tiles, int64_t n_tiles,
           const float *__restrict__ z32, float *__restrict__ P, int nt, int batch,
           int64_t xstride, int reverse, int /*dense: always*/,
           unsigned long long *__restrict__ bytes) {
  __shared__ float s_row[8][kTile];
  __shared__ float s_col[kTile];
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  const int64_t a_stride = (int64_t)nt * (nt + 1) / 2 * kTileElems;
  const int64_t p_stride = (int64_t)nt * nt * kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t total = n_tiles * batch;
  float4 a[4][4];
  auto load = [&](int64_t t, int2 &ij) {
    if (reverse) t = total - 1 - t;
    const int64_t sc = t / n_tiles;
    ij = tiles[t - sc * n_tiles];
    const float4 *T = reinterpret_cast<const float4 *>(A + sc * a_stride +
                                                       tri_index(ij.x, ij.y, nt) * (int64_t)kTileElems);
#pragma unroll
    for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
      for (int i = 0; i < 4; ++i) a[s4][i] = __ldg(T + (int64_t)(warp + 8 * s4) * kTile + lane + 32 * i);
  };
  int64_t t = blockIdx.x;
  int2 ij = make_int2(0, 0);
  if (t < total) load(t, ij);
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  for (; t < total; t += gridDim.x) {
    if (t != blockIdx.x) load(t, ij);
    const int64_t sc = (reverse ? total - 1 - t : t) / n_tiles;
    cta_tile_compute(a, ij.x, ij.y, z32 + sc * xstride, P + sc * p_stride, nt, 1, s_row, s_col);
    if (bytes && threadIdx.x == 0) atomicAdd(bytes, (unsigned long long)kTileElems * 4);
  }
}

// ---- k_gemv_sym (one warp per tile) -------------------------------------------
// y = S x on the packed symmetric tile store, one WARP per tile (I, J), I <= J:
// the row partial (T x_J, 128 rows) goes to slot P[I][J], the column partial
// (T^T x_I, 128 columns) to slot P[J][I]; k_pix_reduce sums the nt slots of
// every element in a fixed order.  A diagonal tile contributes through its
// upper triangle only (element (r,c), c > r, acts as both (r,c) and (c,r)), so
// the operator is exactly symmetric whatever rounding the Gram update left in
// the tile's lower half; this replaces the reference's A <- (A + A^H)/2
// (solver.py:193).
//
// Support-aware: the iterate is sparse (the l1 solution; cfg3 ~40% of atoms
// nonzero in the first pulses, < 1% after 150 pulses), and element (r, c)
// enters y only through T[r][c] x_J[c] and T[r][c] x_I[r].  Each warp reads x_I
// and x_J first, ballots the live column slabs (4 columns, one 16-byte float4
// of every row) and live rows, and picks per tile:
//   * sparse: the row partial from the live slabs only (coalesced 2 KB slab
//     reads), the column partial from the live rows only (lane = slab: one
//     512-byte row read per live row); each round loads 2 slabs and 4 rows;
//   * dense: the whole tile in 16 batches of 2 slabs, each landed by cp.async
//     in a two-stage per-warp ring in shared memory (the next batch in flight
//     while this one is multiplied), the column partial by a butterfly
//     reduce-scatter per batch.
// The row partial sums the slabs in increasing order on both paths (a skipped
// slab adds exact zeros), so it is path-independent; the column partial's
// order depends on the path, which depends only on x: results are
// deterministic.  One warp per tile (no block barriers) keeps 16 independent
// tiles in flight per SM, so a sparse step costs a few dependent round trips
// per tile instead of a full 64 KiB stream.
// sparse path when live slabs + live rows / 2 <= this; measured at cfg3 (full
// arc, pulses/s): 8 -> 651, 16 -> 694, 24 -> 706, 28 -> 706, 32 -> 704, 40 -> 695,
// 48 -> 683 (the sparse matvec alone at the late pulses: 48.7 / 35.7 / 32.1 us ...)
constexpr int kSparseCut = 24;
// per sparse round: live slabs and live rows loaded together; slabs per dense
// batch.  Measured at cfg3 (full arc, pulses/s): <2,4,2> 686.9 (no spills),
// <2,4,4> 683 (spills), <3,4,2> 686.6, <4,4,2> 662.6 (spills); 3 or 4 CTAs per
// SM with narrower batches spill and lose (607 / 470).
constexpr int kSparseSlabs = 2, kSparseRows = 4, kDenseSlabs = 2;

__device__ __forceinline__ float4 shfl4(float4 v, int src) {
  return make_float4(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src),
                     __shfl_sync(0xffffffffu, v.z, src), __shfl_sync(0xffffffffu, v.w, src));
}
// keep columns c0..c0+3 of row `row` with c > row (strict) or c >= row
__device__ __forceinline__ float4 tri_mask(float4 v, int c0, int row, bool strict) {
  const int lo = strict ? row + 1 : row;
  v.x = (c0 + 0 >= lo) ? v.x : 0.f;
  v.y = (c0 + 1 >= lo) ? v.y : 0.f;
  v.z = (c0 + 2 >= lo) ? v.z : 0.f;
  v.w = (c0 + 3 >= lo) ? v.w : 0.f;
  return v;
}
// tile load with an L2 eviction-priority hint (createpolicy value)
__device__ __forceinline__ float4 ldg_pol(const float4 *p, uint64_t pol) {
  float4 v;
  asm("ld.global.nc.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;\n"
      : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
      : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float dot4(float acc, float4 a, float4 z) {
  return acc + a.x * z.x + a.y * z.y + a.z * z.z + a.w * z.w;
}

// A warp's work item: tile (I, J) of scene sc.  Its x (rows of I, this lane's
// slab of J) is staged into the warp's shared-memory slot with cp.async while
// the previous tile is processed, so it costs no registers in flight.
struct WarpTile {
  int I, J;
  int64_t sc;
};
__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16_pol(void *dst, const void *src, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void warp_tile_fetch(WarpTile &w, int64_t t, int64_t total,
                                                int64_t n_tiles, int reverse,
                                                const int2 *__restrict__ tiles,
                                                const float *__restrict__ z32, int64_t xstride,
                                                int lane, float *xr_buf, float4 *xs_buf) {
  const int64_t tt = reverse ? total - 1 - t : t;
  w.sc = tt / n_tiles;
  const int2 ij = tiles[tt - w.sc * n_tiles];
  w.I = ij.x;
  w.J = ij.y;
  const float *x = z32 + w.sc * xstride;
#pragma unroll
  for (int i = 0; i < 4; ++i) cp_async4(xr_buf + lane + 32 * i, x + (int64_t)w.I * kTile + lane + 32 * i);
  cp_async16(xs_buf + lane, reinterpret_cast<const float4 *>(x + (int64_t)w.J * kTile) + lane);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

template <int NS, int NR, int NQ, int MINB, int RING>
__global__ void __launch_bounds__(256, MINB)
k_gemv_sym(const float *__restrict__ A, const int2 *__restrict__ tiles, int64_t n_tiles,
           const float *__restrict__ z32, float *__restrict__ P, int nt, int batch,
           int64_t xstride, int reverse, int dense_only, unsigned long long *__restrict__ bytes,
           int64_t keep_from) {
  __shared__ float s_col[8][kTile];  // per-warp column partial of a diagonal tile
  __shared__ float s_xr[8][kTile];   // per-warp staged x_I of the next tile
  __shared__ float4 s_xs[8][32];     // per-warp staged x_J slabs of the next tile
  // RING > 0: the dense path lands its batches in a per-warp ring of RING
  // stages (cp.async, lane-private slots: a lane reads back only what it
  // copied, so no barrier), RING - 1 batches in flight per warp instead of one
  extern __shared__ __align__(16) unsigned char s_ring_raw[];
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  // batched scenes share the tile list: work item t covers scene t / n_tiles
  const int64_t a_stride = (int64_t)nt * (nt + 1) / 2 * kTileElems;
  const int64_t p_stride = (int64_t)nt * nt * kTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t total = n_tiles * batch;
  const int64_t nw = (int64_t)gridDim.x * 8;
  float *colbuf = s_col[warp];
  float *xr_buf = s_xr[warp];
  float4 *xs_buf = s_xs[warp];
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  int64_t t = (int64_t)blockIdx.x * 8 + warp;
  unsigned long long nbytes = 0;  // tile bytes this warp requested (profiling only)
  const uint64_t pol_first = bulk::policy_evict_first(), pol_last = bulk::policy_evict_last(),
                 pol_norm = bulk::policy_evict_normal();
  WarpTile cur, nxt;
  if (t < total) warp_tile_fetch(cur, t, total, n_tiles, reverse, tiles, z32, xstride, lane, xr_buf, xs_buf);
  // the next tile's index and x are fetched while this tile's loads are in
  // flight, so a tile never starts with a dependent round trip
  auto fetch_next = [&] {
    if (t + nw < total)
      warp_tile_fetch(nxt, t + nw, total, n_tiles, reverse, tiles, z32, xstride, lane, xr_buf, xs_buf);
  };
  for (; t < total; t += nw) {
    const int I = cur.I, J = cur.J;
    const bool diag = I == J;
    const float4 *T = reinterpret_cast<const float4 *>(A + cur.sc * a_stride +
                                                       tri_index(I, J, nt) * (int64_t)kTileElems);
    // dense tiles of a store larger than L2 are streamed evict_first (they do
    // not displace x, the slots and the other streams' data), except the last
    // keep MiB of the traversal, which the next (reversed) step reads first
    const uint64_t pol = keep_from < 0 ? pol_norm : (t >= keep_from ? pol_last : pol_first);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    const float4 zs = xs_buf[lane];
    float zr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) zr[i] = xr_buf[lane + 32 * i];
    const unsigned smask = __ballot_sync(0xffffffffu, slab_live(zs));
    unsigned rm[4];
    int nr = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      rm[i] = __ballot_sync(0xffffffffu, zr[i] != 0.f);
      nr += __popc(rm[i]);
    }
    float *Prow = P + cur.sc * p_stride + ((int64_t)I * nt + J) * kTile;
    float *Pcol = P + cur.sc * p_stride + ((int64_t)J * nt + I) * kTile;
    float rp[4] = {0.f, 0.f, 0.f, 0.f};
    if (!dense_only && __popc(smask) + (nr >> 1) <= kSparseCut) {
      nbytes += (unsigned long long)__popc(smask) * kTile * 16 + (unsigned long long)nr * 32 * 16;
      // ---- sparse: each round loads up to NS live slabs (row partial) and up
      // to NR live rows (column partial, lane = slab) together, so a tile
      // costs max(slab rounds, row rounds) dependent trips; slabs and rows are
      // consumed in increasing order ----
      unsigned m = smask, r0 = rm[0], r1 = rm[1], r2 = rm[2], r3 = rm[3];
      auto pop_row = [&]() -> int {
        int b = -1;
        if (r0) { b = __ffs(r0) - 1; r0 &= r0 - 1; }
        else if (r1) { b = 32 + __ffs(r1) - 1; r1 &= r1 - 1; }
        else if (r2) { b = 64 + __ffs(r2) - 1; r2 &= r2 - 1; }
        else if (r3) { b = 96 + __ffs(r3) - 1; r3 &= r3 - 1; }
        return b;
      };
      float4 cp = make_float4(0.f, 0.f, 0.f, 0.f);
      bool first = true;
      do {
        int sl[NS], rw[NR];
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          sl[q] = m ? __ffs(m) - 1 : -1;
          m &= m - 1;
        }
#pragma unroll
        for (int k = 0; k < NR; ++k) rw[k] = pop_row();
        float4 v[NS][4], w[NR];
#pragma unroll
        for (int q = 0; q < NS; ++q)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            v[q][i] = sl[q] >= 0 ? __ldg(T + (int64_t)sl[q] * kTile + lane + 32 * i)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int k = 0; k < NR; ++k)
          w[k] = rw[k] >= 0 ? __ldg(T + (int64_t)lane * kTile + rw[k]) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (first) fetch_next();
        first = false;
#pragma unroll
        for (int q = 0; q < NS; ++q) {
          if (sl[q] < 0) break;
          const float4 z = shfl4(zs, sl[q]);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float4 a4 = diag ? tri_mask(v[q][i], 4 * sl[q], lane + 32 * i, false) : v[q][i];
            rp[i] = dot4(rp[i], a4, z);
          }
        }
#pragma unroll
        for (int k = 0; k < NR; ++k) {
          if (rw[k] < 0) break;
          const int h = rw[k] >> 5;
          const float zsel = h == 0 ? zr[0] : h == 1 ? zr[1] : h == 2 ? zr[2] : zr[3];
          const float xr = __shfl_sync(0xffffffffu, zsel, rw[k] & 31);
          const float4 a4 = diag ? tri_mask(w[k], 4 * lane, rw[k], true) : w[k];
          cp.x += a4.x * xr;
          cp.y += a4.y * xr;
          cp.z += a4.z * xr;
          cp.w += a4.w * xr;
        }
      } while (m | r0 | r1 | r2 | r3);
      if (diag) reinterpret_cast<float4 *>(colbuf)[lane] = cp;
      else reinterpret_cast<float4 *>(Pcol)[lane] = cp;
    } else {
      nbytes += (unsigned long long)kTileElems * 4;
      // ---- dense: 32 / NQ batches of NQ slabs; batch b+1 is loaded as soon
      // as batch b's products are formed, so its trip overlaps b's column
      // reduction ----
      constexpr int NB = 32 / NQ, NV = 4 * NQ;  // batches; column partials per batch
      float4 v[NQ][4];
      float4 *ring = reinterpret_cast<float4 *>(s_ring_raw) +
                     (size_t)warp * (RING > 0 ? RING : 1) * NV * 32;
      auto ring_issue = [&](int b) {  // batch b -> stage b % RING (one group, empty past the end)
        if (b < NB) {
          float4 *dst = ring + (size_t)(b % (RING > 0 ? RING : 1)) * NV * 32;
#pragma unroll
          for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int i = 0; i < 4; ++i)
              cp_async16_pol(dst + (q * 4 + i) * 32 + lane,
                             T + (int64_t)(NQ * b + q) * kTile + lane + 32 * i, pol);
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
      };
      if (RING > 0) {
        fetch_next();  // (its group is older than every batch group of this tile)
#pragma unroll
        for (int b = 0; b < RING - 1; ++b) ring_issue(b);
      } else {
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
          for (int i = 0; i < 4; ++i) v[q][i] = ldg_pol(T + (int64_t)q * kTile + lane + 32 * i, pol);
        fetch_next();
      }
#pragma unroll 1
      for (int b = 0; b < NB; ++b) {
        if (RING > 0) {
          ring_issue(b + RING - 1);
          asm volatile("cp.async.wait_group %0;\n" ::"n"(RING > 0 ? RING - 1 : 0) : "memory");
          const float4 *src = ring + (size_t)(b % (RING > 0 ? RING : 1)) * NV * 32;
#pragma unroll
          for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int i = 0; i < 4; ++i) v[q][i] = src[(q * 4 + i) * 32 + lane];
        }
        float cp[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) cp[k] = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float4 z = shfl4(zs, NQ * b + q);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int row = lane + 32 * i, c0 = 4 * (NQ * b + q);
            const float4 ar = diag ? tri_mask(v[q][i], c0, row, false) : v[q][i];
            const float4 ac = diag ? tri_mask(v[q][i], c0, row, true) : v[q][i];
            rp[i] = dot4(rp[i], ar, z);
            cp[4 * q + 0] += ac.x * zr[i];
            cp[4 * q + 1] += ac.y * zr[i];
            cp[4 * q + 2] += ac.z * zr[i];
            cp[4 * q + 3] += ac.w * zr[i];
          }
        }
        if (RING == 0 && b < NB - 1) {
#pragma unroll
          for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int i = 0; i < 4; ++i)
              v[q][i] = ldg_pol(T + (int64_t)(NQ * (b + 1) + q) * kTile + lane + 32 * i, pol);
        }
        // butterfly reduce-scatter of the NV column partials over the 32 lanes:
        // halve the live values per lane at lane offsets 16, 8, ..., then sum
        // the remaining lane groups; lane bits above the final offset give the
        // column index
        constexpr int kLevels = NV == 16 ? 4 : NV == 8 ? 3 : NV == 4 ? 2 : 1;
        constexpr int kOff = 16 >> kLevels;  // lane offset after the halving levels
#pragma unroll
        for (int l = 0; l < kLevels; ++l) {
          const int off = 16 >> l, half = NV >> (l + 1);
          const bool hi = lane & off;
#pragma unroll
          for (int k = 0; k < half; ++k) {
            const float send = hi ? cp[k] : cp[k + half];
            const float keep = hi ? cp[k + half] : cp[k];
            cp[k] = keep + __shfl_xor_sync(0xffffffffu, send, off);
          }
        }
#pragma unroll
        for (int o = kOff; o > 0; o >>= 1) cp[0] += __shfl_xor_sync(0xffffffffu, cp[0], o);
        if ((lane & (2 * kOff - 1)) == 0) {
          const int idx = (lane >> (kLevels == 4 ? 1 : kLevels == 3 ? 2 : 3)) &
                          ((1 << kLevels) - 1);
          const int col = NV * b + idx;  // lane bit 16 is the index's top bit
          if (diag) colbuf[col] = cp[0];
          else Pcol[col] = cp[0];
        }
      }
    }
    if (diag) {
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 4; ++i) rp[i] += colbuf[lane + 32 * i];
      __syncwarp();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) Prow[lane + 32 * i] = rp[i];
    cur = nxt;
  }
  if (bytes && lane == 0 && nbytes) atomicAdd(bytes, nbytes);
}

// Tile count from which one warp per tile keeps every SM busy (16 warps per SM).
constexpr int64_t kWarpTileMin = 148 * 16;
// 64 KiB tiles: a store above kL2Tiles does not fit L2; kKeepTiles = 48 MiB
constexpr int64_t kL2Tiles = 126 * 16, kKeepTiles = 48 * 16;

sf_status launch_gemv(const float *A, const int2 *tiles, int64_t n_tiles, const float *z32,
                      float *P, int nt, int sym, int grid, cudaStream_t st, int batch,
                      int64_t xstride, int reverse, int dense, unsigned long long *bytes) {
  if (n_tiles == 0) return SF_OK;
  if (!sym) return fail(SF_EUNSUPPORTED, "matvec: symmetric stores only");
  const int64_t tot = n_tiles * batch;
  cudaError_t ce;
  if (tot >= kWarpTileMin) {
    // equal tile counts per warp: R rounds over at most grid*8 warps, then the
    // fewest warps that still finish in R rounds (no half-empty last round)
    // dense batches land in a two-stage per-warp ring in shared memory
    // (cp.async): measured at cfg3 against the register double buffer, dense
    // prefix / full arc 729 / 848 vs 723 / 835 pulses/s; a three-stage ring
    // (two batches in flight) needs the maximum shared-memory carve-out, and
    // the sparse path's row reads then lose their L1 (53 vs 33 us per launch)
    constexpr int kRing = 2;
    const char *rg = getenv("SF_GEMV_RING");
    const bool ring = !(rg && rg[0] == '0');
    auto kern = ring ? k_gemv_sym<kSparseSlabs, kSparseRows, kDenseSlabs, 2, kRing>
                     : k_gemv_sym<kSparseSlabs, kSparseRows, kDenseSlabs, 2, 0>;
    const size_t dsm = ring ? (size_t)8 * kRing * 4 * kDenseSlabs * 32 * 16 : 0;
    if (ring) {
      static std::atomic<uint64_t> set{0};
      if (attr_pending(set)) {
        SF_CUDA_TRY(cudaFuncSetAttribute(k_gemv_sym<kSparseSlabs, kSparseRows, kDenseSlabs, 2, kRing>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm));
        attr_done(set);
      }
    }
    const int64_t maxw = (int64_t)grid * 8;  // grid = 2 CTAs per SM
    const int64_t rounds = (tot + maxw - 1) / maxw;
    const int64_t warps = (tot + rounds - 1) / rounds;
    const int64_t g = (warps + 7) / 8;
    // L2 hints for stores that do not fit L2 (126 MB): measured at cfg3 (541 MB
    // store, pulses/s over the dense first pulses / the full arc): no hints
    // 675 / 806, evict_first with the last 16 / 48 / 64 / 96 / 128 MiB of the
    // traversal evict_last 700 / 830, 705 / 833, 702 / 830, 705 / 830, 697 / 831;
    // evict_last alone (the rest evict_normal) 684 / 811
    const int64_t keep_from = tot > kL2Tiles ? tot - kKeepTiles : -1;
    ce = launch_pdl(kern, dim3((unsigned)g), dim3(256), dsm, st, A, tiles, n_tiles, z32, P, nt,
                    batch, xstride, reverse, dense, bytes, keep_from);
  } else {
    const int64_t g = tot < grid ? tot : grid;
    ce = launch_pdl(k_gemv_cta, dim3((unsigned)g), dim3(256), 0, st, A, tiles, n_tiles, z32, P, nt,
                    batch, xstride, reverse, dense, bytes);
  }
  if (ce != cudaSuccess) return fail(SF_ECUDA, std::string("matvec: ") + cudaGetErrorString(ce));
  SF_LAUNCH_CHECK();
  return SF_OK;
}

}  // namespace sf
