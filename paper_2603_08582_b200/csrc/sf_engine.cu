// sf_engine.cu -- handle-based engine behind the C ABI of include/sarfista_b200.h.
//
// Device state per engine (all resident in HBM for the engine's lifetime):
//   A      packed upper-triangle tiles of Re(A), fp32, 64 KiB per 128x128 tile
//   b      running b, complex fp64 [M]        L, pulse/fallback counters (device)
//   Gp     packed per-pulse operator [m_pad][k_pad] fp32 (G/sigma, Re | Im)
//   P      FISTA partial slots [nt][nt][128] fp32
// Host side keeps only sizes, the tile list and pinned staging for pulse inputs.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cstdio>
#include <string>
#include <vector>

#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {

static thread_local std::string t_last_error;
std::atomic<int64_t> g_launches{0};
static thread_local bool t_capturing = false;
void set_capturing(bool on) { t_capturing = on; }
static bool capturing() { return t_capturing; }
bool debug_sync() {
  static const bool v = getenv("SF_DEBUG_SYNC") != nullptr;
  return v && !t_capturing;
}

void set_error(const std::string &msg) { t_last_error = msg; }
sf_status fail(sf_status st, const std::string &msg) {
  set_error(msg);
  return st;
}

template <class T>
static sf_status dalloc(T **p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void **)p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? SF_ENOMEM : SF_ECUDA,
                std::string("cudaMalloc(") + std::to_string(count * sizeof(T)) +
                    " bytes): " + cudaGetErrorString(e));
  }
  return SF_OK;
}

static int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

// RAII device scratch for the engine-less seam functions.
struct DevBuf {
  void *p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};
template <class T>
static sf_status dscratch(DevBuf &b, T **out, size_t count) {
  sf_status s = dalloc(out, count);
  b.p = *out;
  return s;
}

// Devices already checked (bit per ordinal): the check runs on every engine
// creation and seam call, so it must stay cheap after the first time.
static std::atomic<uint64_t> g_checked{0};

static sf_status check_device(int device) {
  if (device >= 0 && device < 64 && (g_checked.load(std::memory_order_acquire) >> device & 1)) {
    SF_CUDA_TRY(cudaSetDevice(device));
    return SF_OK;
  }
  int n = 0;
  SF_CUDA_TRY(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(SF_EINVAL, "invalid CUDA device ordinal");
  int major = 0;
  SF_CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major != 10) {
    cudaDeviceProp prop;
    SF_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    return fail(SF_EUNSUPPORTED, std::string("sm_100 (B200) device required, found ") +
                                     prop.name);
  }
  SF_CUDA_TRY(cudaSetDevice(device));
  if (device < 64) g_checked.fetch_or(1ull << device, std::memory_order_release);
  return SF_OK;
}

}  // namespace sf

using namespace sf;

struct sf_engine {
  int device = 0;
  cudaStream_t own_stream = nullptr, stream = nullptr;
  int64_t m = 0, m_pad = 0, n_tiles = 0, n_pix = 0;
  int nt = 0, n_r = 0, k_pad_max = 0, ell_width = 0, precision = 0;
  int sm_count = 148, compose_grid = 0, gemv_grid = 0;
  int mode = SF_MODE_ATOM;
  // keep_complex (atom mode): the complex A in fp64, the tiles derived from it
  bool keep_complex = false;
  double2 *A64 = nullptr;
  // batched scenes (sf_desc.batch > 1, pixel mode): every per-scene buffer is
  // `batch` consecutive copies; scene s of a buffer of per-scene size S starts
  // at s * S.  Pulse inputs per scene in PulseSet::in: omega | d | gamma | sig
  // at in_off_* (even offsets, so d is 16-byte aligned for any n_r).
  int batch = 1;
  int64_t in_off_d = 0, in_off_g = 0, in_off_s = 0, in_stride = 0, zstride = 0;
  int64_t dpad = 0;  // padded dimension of the stored symmetric matrix (M or N)
  // pixel-space state (SF_MODE_PIXEL)
  double2 *beta = nullptr, *hv0 = nullptr, *bp = nullptr;  // bp: sum_k F_k^H d_k
  double *ypix = nullptr;
  // Pipelined per-pulse scratch (pixel mode): the operator phase of pulse n+1
  // (F, K~, power iteration, operand split) runs on the side stream while the
  // main stream runs pulse n's Gram update and FISTA.  Two sets, reused
  // alternately; `consumed` guards reuse, `ready` hands a set to the main stream.
  struct PulseSet {
    double *in = nullptr;  // per scene: omega | d | gamma | 1/sigma, sigma^2 (in_off_*)
    double *raw = nullptr;  // batched inputs before the per-scene scatter
    double *tau = nullptr, *pdiag = nullptr;
    double2 *Ft = nullptr, *W = nullptr, *Kpart = nullptr, *K = nullptr, *u0part = nullptr,
            *u0 = nullptr, *dbeta = nullptr;
    float2 *Kf = nullptr;
    float *Gp = nullptr;
    __half *Gh = nullptr;
    unsigned *maxbits = nullptr;
    int *gexp = nullptr;
    float *zpart = nullptr;  // tensor-core K~: per-CTA Z blocks
    int *kexp = nullptr;
    __half *kxs = nullptr;   // tensor-core K~: X / Y slabs
    DirPix *dtab = nullptr;  // closed-form Gram: per-pixel table of this pulse
    // prep: the Gram update's per-pixel inputs are ready (recorded inside the
    // operator graph); ready: the whole operator phase (incl. the power
    // iteration) is done; consumed: the state update has read this set
    cudaEvent_t prep = nullptr, ready = nullptr, consumed = nullptr;
    // replayed chains: operator phase; state update per buffer parity (2: in place)
    cudaGraphExec_t op_exec = nullptr, st_exec[3] = {nullptr, nullptr, nullptr},
                    fd_exec[3] = {nullptr, nullptr, nullptr};
    int64_t op_kernels = 0, st_kernels = 0, fd_kernels = 0;
  } ps[6];
  int ps_next = 0;
  // Double-buffered solver state (pixel mode, when two tile stores fit): pulse
  // n+1's state update (Gram, fold, b = H^T beta) runs on `stats` writing the
  // alternate buffers while the main stream's FISTA for pulse n reads the
  // current ones; then the host swaps the pointers.  A, b, bmax and the FISTA
  // copy of L are the buffers FISTA reads; beta, bp, counters stay single
  // (written only on `stats`, read by host-synchronous getters).
  bool dbuf = false;
  cudaStream_t stats = nullptr;
  float *A_alt = nullptr;
  double2 *b_alt = nullptr;
  unsigned long long *bmax_alt = nullptr;
  double *Lsnap = nullptr, *Lsnap_alt = nullptr;
  cudaEvent_t ev_stats = nullptr, ev_readers = nullptr;
  int prio_hi = 0;                      // the device's greatest stream priority
  // CUDA graphs of the pixel FISTA chain, one per (state buffers, steps); the
  // per-call scalars (lambda rule, t0) are patched into the setup node
  struct FGraph {
    const void *A = nullptr, *b = nullptr, *bmax = nullptr, *L = nullptr;
    int steps = 0;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t setup = nullptr;
    bool prologue = false;  // the setup node is k_fista_prologue (setup + init + H z)
    // the last atom step (writes c_out): with the prologue, c0 and c_out are
    // patched per call instead of copied through e->cin / e->cout
    cudaGraphNode_t last_step = nullptr;
    AtomStepNodeArgs last_args{};
    dim3 last_grid, last_block;
    int64_t kernels = 0;
  };
  std::vector<FGraph> fgraphs;
  cudaStream_t cap_stream = nullptr;
  double *wbuf = nullptr;  // momentum weights of the current FISTA call (device)
  int wbuf_cap = 0;
  // operator phases of consecutive pulses are independent: rotate over
  // kSide pipeline streams so several single-SM power iterations run at once
  cudaStream_t side2 = nullptr, side3 = nullptr, side4 = nullptr, side5 = nullptr;
  int side_next = 0, n_side = 4;
  double l_floor = 1e-12;
  double power_rel_tol = 1e-6;
  int power_max_iter = 500;
  int64_t pulse_count = 0;  // host mirror (each accumulate adds exactly one)
  double bbox_lo[3] = {0, 0, 0}, bbox_hi[3] = {0, 0, 0};
  std::vector<double> h_xyz;
  std::vector<int2> h_tiles;
  // device state
  float *A = nullptr;
  int2 *tiles = nullptr;
  double2 *b = nullptr;
  double *L = nullptr;
  long long *counters = nullptr;  // [0] pulse_count, [1] fallbacks
  double *diag = nullptr;         // power-iteration diagnostics
  double *scal = nullptr;         // tau, thresh, lambda
  double2 *v0 = nullptr;
  float *Gp = nullptr;
  double2 *Ft = nullptr;
  double *tau = nullptr, *omega = nullptr, *xyz = nullptr, *gamma = nullptr;
  int *zero_flag = nullptr;
  int32_t *ell_idx = nullptr;
  double *ell_w = nullptr;
  int64_t *csr_ptr = nullptr;
  int32_t *csr_atom = nullptr;
  // batched engines: the CSR of H transposed entry-major ([entry][pixel], -1 =
  // none) for k_hz_ell (lane = pixel, coalesced index loads)
  int32_t *hz_atomT = nullptr;
  double *hz_wT = nullptr;
  int hz_ents = 0;
  double *csr_w = nullptr;
  double2 *dt = nullptr, *u0part = nullptr, *Kpart = nullptr, *K = nullptr, *u0 = nullptr;
  float2 *Kf = nullptr;
  int kpart_splits = 0, px_splits = 0;
  // pixel-space Lipschitz operator: Q = H H^T (CSR, pixel-major), W = Q F
  // tensor-core K~ (sf_ktc.cu; default for one pixel-mode scene with 2 N_r <= 256)
  bool ktc_on = false;
  int ktc_grid = 0;
  KtcArgs ktc;
  void *ktc_mem[2] = {};
  int64_t *qptr = nullptr;
  int32_t *qcol = nullptr;
  double *qval = nullptr;
  double2 *W = nullptr;
  unsigned long long *bmax = nullptr;
  // side stream: K~ build + power iteration overlap the Gram update
  cudaStream_t side = nullptr;
  cudaEvent_t ev_c = nullptr, ev_p = nullptr;
  float *P = nullptr, *z32 = nullptr;
  double *zd = nullptr, *cprev = nullptr, *cin = nullptr, *cout = nullptr, *img = nullptr;
  double2 *Gd = nullptr;
  size_t Gd_count = 0;
  // f16x3 Gram path: canonical fp16 hi/lo panels, scale, super-tile list
  __half *Gh = nullptr;
  unsigned *maxbits = nullptr;
  int *gexp = nullptr;
  int2 *items = nullptr;
  int n_items = 0;
  // sharding of one scene over `world` GPUs (pixel mode): this rank's Gram
  // items and matvec tiles; unsharded engines alias the full lists
  int shard_rank = 0, shard_world = 1;
  void *comm = nullptr;     // NCCL: FISTA y_pix exchange
  void *comm_op = nullptr;  // NCCL: operator-phase K~ partials (own communicator)
  cudaEvent_t ev_opcoll = nullptr;  // orders the operator-phase exchanges across side streams
  LoopGroup *loop = nullptr;  // in-process loopback exchange (emulated ranks, tests)
  PeerGroup *peer = nullptr;  // peer-memory exchange (one process per GPU, no collective library)
  int2 *items_local = nullptr, *tiles_local = nullptr;
  int n_items_local = 0;
  int64_t n_tiles_local = 0;
  bool own_local = false;
  // pinned staging ring for per-pulse host inputs (omega + d~)
  static constexpr int kRing = 8;
  double *h_stage = nullptr;
  int64_t stage_slot_size = 0;  // doubles per ring slot
  cudaEvent_t stage_ev[kRing] = {};
  int stage_slot = 0;
  cudaEvent_t ev_acc0 = nullptr, ev_acc1 = nullptr, ev_f0 = nullptr, ev_f1 = nullptr;
  bool acc_timed = false, fista_timed = false;
  bool call_timing = false;  // set by the first sf_last_timings call
  int64_t device_bytes = 0;
  // per-kernel event timing (sf_profile)
  struct Prof {
    std::vector<cudaEvent_t> start, stop;
    size_t used = 0;
  } prof[8];
  bool profiling = false;
  unsigned long long *gemv_bytes = nullptr;  // matvec tile bytes requested while profiling
  double *metrics = nullptr;                 // sf_pulse_metrics scratch
  unsigned long long *gram_next = nullptr;   // closed-form Gram: work-item counter

  ~sf_engine() {
    cudaSetDevice(device);
    for (auto &p : prof) {
      for (auto ev : p.start) cudaEventDestroy(ev);
      for (auto ev : p.stop) cudaEventDestroy(ev);
    }
    for (auto &q : ps) {
      void *pb[] = {q.in, q.tau, q.pdiag, q.Ft, q.W, q.Kpart, q.K, q.u0part, q.u0, q.dbeta, q.Kf,
                    q.Gp, q.Gh, q.maxbits, q.gexp, q.raw, q.dtab, q.zpart, q.kexp, q.kxs};
      for (void *b : pb)
        if (b) cudaFree(b);
      if (q.prep) cudaEventDestroy(q.prep);
      if (q.ready) cudaEventDestroy(q.ready);
      if (q.consumed) cudaEventDestroy(q.consumed);
      if (q.op_exec) cudaGraphExecDestroy(q.op_exec);
      for (auto x : q.st_exec)
        if (x) cudaGraphExecDestroy(x);
      for (auto x : q.fd_exec)
        if (x) cudaGraphExecDestroy(x);
    }
    void *bufs[] = {A, tiles, b, L, counters, diag, scal, v0, Gp, Ft, tau, omega, xyz, gamma, gemv_bytes,
                    metrics, gram_next,
                    zero_flag,
                    ell_idx, ell_w, csr_ptr, csr_atom, csr_w, hz_atomT, hz_wT, dt, u0part, Kpart, K, u0, Kf,
                    P, z32, zd, cprev, cin, cout, img, Gd, Gh, maxbits, gexp, items, qptr,
                    qcol, qval, W, bmax, beta, hv0, ypix, bp, A_alt, b_alt, bmax_alt,
                    Lsnap, Lsnap_alt, A64};
    for (void *p : bufs)
      if (p) cudaFree(p);
    if (h_stage) cudaFreeHost(h_stage);
    for (auto &e : stage_ev)
      if (e) cudaEventDestroy(e);
    cudaEvent_t evs[] = {ev_acc0, ev_acc1, ev_f0,    ev_f1,      ev_c,
                         ev_p,    ev_stats, ev_readers};
    for (auto e : evs)
      if (e) cudaEventDestroy(e);
    if (own_stream) cudaStreamDestroy(own_stream);
    if (side) cudaStreamDestroy(side);
    if (side2) cudaStreamDestroy(side2);
    if (side3) cudaStreamDestroy(side3);
    if (side4) cudaStreamDestroy(side4);
    if (side5) cudaStreamDestroy(side5);
    if (stats) cudaStreamDestroy(stats);
    for (auto &g : fgraphs) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      if (g.graph) cudaGraphDestroy(g.graph);
    }
    if (cap_stream) cudaStreamDestroy(cap_stream);
    for (void *p : ktc_mem)
      if (p) cudaFree(p);
    if (wbuf) cudaFree(wbuf);
    if (own_local) {
      if (items_local) cudaFree(items_local);
      if (tiles_local) cudaFree(tiles_local);
    }
    nccl_comm_destroy(comm);
    nccl_comm_destroy(comm_op);
    if (ev_opcoll) cudaEventDestroy(ev_opcoll);
  }
};

namespace {

template <class T>
sf_status track_alloc(sf_engine *e, T **p, size_t count) {
  sf_status s = dalloc(p, count);
  if (s == SF_OK) e->device_bytes += (int64_t)(count * sizeof(T));
  return s;
}

sf_status to_device(sf_engine *e, void *dst, const void *src, size_t bytes, int mem) {
  SF_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes,
                              mem == SF_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                   : cudaMemcpyHostToDevice,
                              e->stream));
  return SF_OK;
}

sf_status from_device(sf_engine *e, void *dst, const void *src, size_t bytes, int mem) {
  SF_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes,
                              mem == SF_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                   : cudaMemcpyDeviceToHost,
                              e->stream));
  if (mem != SF_MEM_DEVICE) SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return SF_OK;
}

// Host-side guard of geometry.py:102-103 (platform on a scene pixel).  A
// platform outside the scene's bounding box cannot coincide with a pixel.
bool platform_hits_pixel(const sf_engine *e, const double *g) {
  bool outside = false;
  for (int k = 0; k < 3; ++k)
    if (g[k] < e->bbox_lo[k] || g[k] > e->bbox_hi[k]) outside = true;
  if (outside) return false;
  for (int64_t p = 0; p < e->n_pix; ++p) {
    const double *x = &e->h_xyz[3 * p];
    if (x[0] == g[0] && x[1] == g[1] && x[2] == g[2]) return true;
  }
  return false;
}

// Event pair around one launch (only while sf_profile is on).
sf_status prof_mark(sf_engine *e, int kind, bool begin, cudaStream_t st) {
  if (!e->profiling) return SF_OK;
  auto &p = e->prof[kind];
  if (begin) {
    if (p.used == p.start.size()) {
      cudaEvent_t a, b;
      SF_CUDA_TRY(cudaEventCreate(&a));
      SF_CUDA_TRY(cudaEventCreate(&b));
      p.start.push_back(a);
      p.stop.push_back(b);
    }
    SF_CUDA_TRY(cudaEventRecord(p.start[p.used], st));
  } else {
    SF_CUDA_TRY(cudaEventRecord(p.stop[p.used], st));
    p.used++;
  }
  return SF_OK;
}

#define SF_PROF(kind, begin)                     \
  do {                                           \
    sf_status _ps = prof_mark(e, kind, begin, e->stream); \
    if (_ps) return _ps;                         \
  } while (0)

// Shared tail of both accumulate flavours.  Geometric pulses build K~ in pixel
// space and run the power iteration on the side stream, overlapping the Gram
// update (which then leaves one SM to the single-CTA power iteration); dense
// pulses do everything in order on the main stream.
sf_status accumulate_tail(sf_engine *e, int n_r, int k_pad, bool geometric, double inv_sigma) {
  // keep_complex (dense pulses): K~ partials from the fp64 operator and the
  // exact Hermitian update of the complex A, then the tiles re-derived from it
  const bool exact = e->keep_complex && !geometric;
  sf_status s;
  SF_PROF(SF_K_OPERATOR, false);
  int gram_grid = e->sm_count;
  if (geometric) {
    SF_CUDA_TRY(cudaEventRecord(e->ev_c, e->stream));
    SF_CUDA_TRY(cudaStreamWaitEvent(e->side, e->ev_c, 0));
    if ((s = prof_mark(e, SF_K_LIPSCHITZ, true, e->side))) return s;
    s = launch_fq(e->qptr, e->qcol, e->qval, e->Ft, e->n_pix, n_r, e->W, e->side);
    if (s) return s;
    s = launch_kgram_px(e->Ft, e->W, e->n_pix, n_r, e->px_splits, e->Kpart, e->side, 1);
    if (s) return s;
    s = launch_kreduce(e->Kpart, e->px_splits, e->u0part, e->compose_grid, n_r, 1,
                       inv_sigma * inv_sigma, e->K, e->Kf, e->u0, e->side);
    if (s) return s;
    s = launch_power_iter(e->K, e->Kf, e->u0, n_r, e->power_rel_tol, e->power_max_iter, e->L,
                          e->counters, e->diag, e->side);
    if (s) return s;
    if ((s = prof_mark(e, SF_K_LIPSCHITZ, false, e->side))) return s;
    SF_CUDA_TRY(cudaEventRecord(e->ev_p, e->side));
    gram_grid = e->sm_count > 1 ? e->sm_count - 1 : 1;
  } else {
    if ((s = prof_mark(e, SF_K_LIPSCHITZ, true, e->stream))) return s;
    s = exact ? launch_kgram_c64(e->Gd, e->m, n_r, inv_sigma * inv_sigma, e->kpart_splits, e->Kpart,
                                 e->stream)
              : launch_kgram(e->Gp, e->m, n_r, k_pad, e->kpart_splits, e->Kpart, e->stream);
    if (s) return s;
    s = launch_kreduce(e->Kpart, e->kpart_splits, e->u0part, e->compose_grid, n_r, 0, 1.0, e->K,
                       e->Kf, e->u0, e->stream);
    if (s) return s;
    s = launch_power_iter(e->K, e->Kf, e->u0, n_r, e->power_rel_tol, e->power_max_iter, e->L,
                          e->counters, e->diag, e->stream);
    if (s) return s;
    if ((s = prof_mark(e, SF_K_LIPSCHITZ, false, e->stream))) return s;
  }
  SF_PROF(SF_K_GRAM, true);
  if (exact) {
    s = launch_herk_c64(e->Gd, n_r, e->m, inv_sigma * inv_sigma, e->A64, e->stream);
    if (s) return s;
    s = launch_pack_re(e->A64, e->m, e->tiles, e->n_tiles, e->A, e->stream);
  } else if (e->precision == SF_PREC_F16X3) {
    s = launch_split_panels(e->Gp, e->m_pad, k_pad, e->maxbits, e->gexp, e->Gh, e->stream);
    if (s) return s;
    s = launch_gram_f16x3(e->Gh, k_pad, e->nt, e->items, e->n_items, e->gexp, e->A, e->A, gram_grid,
                          e->stream);
  } else {
    s = launch_gram(e->precision, e->Gp, k_pad, e->tiles, e->n_tiles, e->nt, e->A, e->A, e->stream);
  }
  if (s) return s;
  SF_PROF(SF_K_GRAM, false);
  if (geometric) SF_CUDA_TRY(cudaStreamWaitEvent(e->stream, e->ev_p, 0));
  e->pulse_count += 1;
  return SF_OK;
}

// Pixel-space pulse, pipelined.  Side stream (operator phase, depends only on
// this pulse's inputs): delays -> F (fp64) + packed F~ + dbeta + u0 ->
// K~ = F Q F^H / s^2 -> power iteration record -> fp16 hi/lo operand split.
// Main stream (state, in pulse order): Re(B) += P^T P (tcgen05) -> fold
// dbeta and the L increment -> b = H^T beta.
sf_status stage_inputs(sf_engine *e, double **slot_out);

// Drop every captured graph (they bake in buffer pointers and tile lists).
void drop_graphs(sf_engine *e) {
  cudaDeviceSynchronize();
  for (auto &q : e->ps) {
    if (q.op_exec) cudaGraphExecDestroy(q.op_exec);
    q.op_exec = nullptr;
    for (auto &x : q.st_exec) {
      if (x) cudaGraphExecDestroy(x);
      x = nullptr;
    }
    for (auto &x : q.fd_exec) {
      if (x) cudaGraphExecDestroy(x);
      x = nullptr;
    }
  }
  for (auto &g : e->fgraphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    if (g.graph) cudaGraphDestroy(g.graph);
  }
  e->fgraphs.clear();
}

// Sum `n` doubles over the ranks of a sharded engine, in place on `st`:
// channel 0 = the FISTA chain's y_pix, 1 = the operator phase's K~ partials
// (its own NCCL communicator; an event chain keeps those exchanges in pulse
// order across the rotating side streams, the order every rank issues them in).
// `pushed`: the producer kernel already stored the partial into the peer slots
// (k_pix_reduce in a peer-memory group).
static sf_status exchange_sum(sf_engine *e, int ch, double *buf, size_t n, cudaStream_t st,
                              bool pushed = false) {
  void *c = ch == 0 ? e->comm : e->comm_op;
  if (!e->loop && !e->peer && !c) return SF_OK;
  if (ch == 1) SF_CUDA_TRY(cudaStreamWaitEvent(st, e->ev_opcoll, 0));
  sf_status s;
  if (e->loop) s = loop_allreduce_f64(e->loop, ch, e->shard_rank, buf, n, st);
  else if (e->peer) s = peer_allreduce_f64(e->peer, ch, buf, n, st, pushed);
  else s = nccl_allreduce_f64(buf, n, c, st);
  if (s) return s;
  if (ch == 1) SF_CUDA_TRY(cudaEventRecord(e->ev_opcoll, st));
  return SF_OK;
}

// Operator phase of one pixel-space pulse on `side` (inputs already in q.in:
// omega | d | gamma | 1/sigma | sigma^2): delays -> F (fp64) + packed F~ +
// dbeta + u0 -> K~ = F Q F^H / s^2 -> power iteration record -> fp16 split.
sf_status enqueue_operator(sf_engine *e, sf_engine::PulseSet &q, int k_pad, cudaStream_t side) {
  sf_status s;
  const int n_r = e->n_r, B = e->batch;
  const double *sig = q.in + e->in_off_s;
  if ((s = launch_pixel_delays(e->xyz, e->n_pix, q.in + e->in_off_g, q.tau, e->zero_flag, side, B,
                               e->in_stride)))
    return s;
  SF_CUDA_TRY(cudaMemsetAsync(q.maxbits, 0, sizeof(unsigned) * B, side));
  PixelForwardArgs a;
  a.omega = q.in;
  a.n_r = n_r;
  a.tau = q.tau;
  a.n = e->n_pix;
  a.n_pad = e->dpad;
  a.k_pad = k_pad;
  a.sig = sig;
  a.d = reinterpret_cast<const double2 *>(q.in + e->in_off_d);
  a.batch = B;
  a.in_stride = e->in_stride;
  a.hv0 = e->hv0;
  a.Ft = q.Ft;
  a.Gp = q.Gp;
  a.dbeta = q.dbeta;
  a.u0part = q.u0part;
  a.maxbits = q.maxbits;
  a.grid = e->compose_grid;
  // closed-form Gram + tensor-core K~: nothing else reads the fp32 panel, so
  // the forward kernel writes the K~ build's fp16 slabs itself
  const bool fuse_slabs = e->ktc_on && e->precision == SF_PREC_DIRICHLET;
  if (fuse_slabs) {
    a.Gp = nullptr;
    a.slabs.xs = q.kxs;
    a.slabs.xs_stride = e->ktc.xs_stride;
    a.slabs.slab_stride = e->ktc.slab_stride;
    a.slabs.ngrp = e->ktc.ngrp;
    a.slabs.grp_pix = e->ktc.grp_pix;
    a.slabs.exps = q.kexp;
    a.slabs.qrow_max = e->ktc.qrow_max;
    a.slabs.nb = e->ktc.nb;
  }
  if ((s = launch_forward_pix(a, side))) return s;
  // the Gram update's inputs first, so the state stream can start the Gram
  // update while this pulse's K~ and power iteration are still running
  if (e->precision == SF_PREC_F16X3 &&
      (s = launch_split_panels(q.Gp, e->dpad, k_pad, q.maxbits, q.gexp, q.Gh, side, B)))
    return s;
  if (e->precision == SF_PREC_DIRICHLET &&
      (s = launch_dirichlet_prep(q.tau, e->n_pix, e->dpad, q.in, e->in_stride, n_r, q.dtab,
                                 e->zero_flag, side, B)))
    return s;
  SF_CUDA_TRY(cudaEventRecordWithFlags(q.prep, side,
                                       capturing() ? cudaEventRecordExternal : cudaEventRecordDefault));
  if (e->ktc_on) {  // K~ on tensor cores, then K~ / its fp32 copy / u0
    KtcArgs ka = e->ktc;
    ka.X = q.Gp;
    ka.maxbits = q.maxbits;
    ka.zpart = q.zpart;
    ka.xs = q.kxs;
    ka.exps = q.kexp;
    ka.presplit = fuse_slabs ? 1 : 0;
    if ((s = prof_mark(e, SF_K_KTILDE, true, side))) return s;
    // sharded: each rank builds the Z partials of its own pixel tiles, one
    // exchange sums them, every rank then assembles the same K~
    if ((s = launch_ktilde_tc_partial(ka, e->ktc_grid, side, B))) return s;
    if (e->shard_world > 1 &&
        (s = exchange_sum(e, 1, ktc_zsum(ka, e->ktc_grid),
                          (size_t)(ka.nb * (ka.nb + 1) / 2) * 128 * 128, side)))
      return s;
    if ((s = launch_ktilde_assemble(ka, e->ktc_grid, q.u0part, e->compose_grid, n_r, q.K, q.Kf,
                                    q.u0, side, B)))
      return s;
    if ((s = prof_mark(e, SF_K_KTILDE, false, side))) return s;
  } else {
    if ((s = launch_fq(e->qptr, e->qcol, e->qval, q.Ft, e->n_pix, n_r, q.W, side, B))) return s;
    if ((s = launch_kgram_px(q.Ft, q.W, e->n_pix, n_r, e->px_splits, q.Kpart, side, B))) return s;
    if ((s = launch_kreduce(q.Kpart, e->px_splits, q.u0part, e->compose_grid, n_r, 1, 1.0, q.K,
                            q.Kf, q.u0, side, sig, B, e->in_stride)))
      return s;
  }
  if ((s = prof_mark(e, SF_K_LIPSCHITZ, true, side))) return s;
  if ((s = launch_power_iter(q.K, q.Kf, q.u0, n_r, e->power_rel_tol, e->power_max_iter, nullptr,
                             nullptr, q.pdiag, side, 0, B)))
    return s;
  return prof_mark(e, SF_K_LIPSCHITZ, false, side);
}

// State update of one pulse on `ss`, first half: Re(B) out = Re(B) in + the
// pulse's Gram increment (closed form, or tcgen05 for f16x3); needs only the
// operator phase's per-pixel table / operand panels (event q.prep).
sf_status enqueue_gram(sf_engine *e, sf_engine::PulseSet &q, int k_pad, cudaStream_t ss,
                       const float *A_in, float *A_out) {
  const int B = e->batch;
  if (e->precision == SF_PREC_F16X3)
    return launch_gram_f16x3(q.Gh, k_pad, e->nt, e->items_local, e->n_items_local, q.gexp, A_in,
                             A_out, e->sm_count, ss, B, (int64_t)e->dpad * k_pad * 2,
                             e->n_tiles * (int64_t)kTileElems);
  if (e->precision == SF_PREC_DIRICHLET)
    return launch_gram_dirichlet(q.dtab, e->dpad, e->tiles_local, e->n_tiles_local, e->nt, q.in,
                                 e->in_stride, e->in_off_s, e->n_r, A_in, A_out, e->sm_count, ss, B,
                                 e->n_tiles * (int64_t)kTileElems, e->gram_next);
  return launch_gram(e->precision, q.Gp, k_pad, e->tiles_local, e->n_tiles_local, e->nt, A_in,
                     A_out, ss);
}

// Second half (after the power iteration, event q.ready): fold dbeta / L /
// counters / BP, b = H^T beta and max|b|, FISTA's copy of L.
sf_status enqueue_fold(sf_engine *e, sf_engine::PulseSet &q, cudaStream_t ss, double2 *b_out,
                       unsigned long long *bmax_out, double *Lsnap_out) {
  sf_status s;
  const int B = e->batch;
  const double *sig = q.in + e->in_off_s;
  if ((s = launch_fold(q.dbeta, e->beta, e->n_pix, q.pdiag, e->L, e->counters, e->diag, 0.0,
                       e->bp, ss, sig, B, e->in_stride)))
    return s;
  SF_CUDA_TRY(cudaMemsetAsync(bmax_out, 0, sizeof(unsigned long long) * B, ss));
  if ((s = launch_bupdate(e->ell_idx, e->ell_w, e->ell_width, e->m, e->beta, b_out, bmax_out, ss,
                          B, e->n_pix)))
    return s;
  if (Lsnap_out)
    SF_CUDA_TRY(cudaMemcpyAsync(Lsnap_out, e->L, sizeof(double) * B, cudaMemcpyDeviceToDevice, ss));
  return SF_OK;
}

// Capture `body` (which enqueues on the given stream) as an instantiated graph.
template <class F>
static sf_status capture_graph(sf_engine *e, F &&body, cudaGraphExec_t *exec, int64_t *kernels) {
  if (!e->cap_stream) SF_CUDA_TRY(cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking));
  const int64_t l0 = g_launches.load();
  SF_CUDA_TRY(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal));
  set_capturing(true);
  sf_status s = body(e->cap_stream);
  set_capturing(false);
  cudaGraph_t g = nullptr;
  cudaError_t ce = cudaStreamEndCapture(e->cap_stream, &g);
  *kernels = g_launches.load() - l0;
  g_launches -= *kernels;
  if (s) {
    if (g) cudaGraphDestroy(g);
    return s;
  }
  if (ce != cudaSuccess) return fail(SF_ECUDA, std::string("graph capture: ") + cudaGetErrorString(ce));
  ce = cudaGraphInstantiate(exec, g, 0);
  cudaGraphDestroy(g);
  if (ce != cudaSuccess) return fail(SF_ECUDA, std::string("graph instantiate: ") + cudaGetErrorString(ce));
  return SF_OK;
}

// Pixel-space pulse, pipelined.  Side stream: the operator phase (depends only
// on this pulse's inputs).  `stats` stream (or the main stream when not
// double-buffered): the state update, in pulse order.  Both chains replay as
// CUDA graphs (captured once per scratch set / buffer parity) unless
// profiling or SF_NO_GRAPHS.
// Next scratch set + pipeline stream for a pulse; waits until the set is free.
sf_status next_pulse_set(sf_engine *e, sf_engine::PulseSet **qo, cudaStream_t *sideo) {
  const int si = e->ps_next;
  e->ps_next = (e->ps_next + 1) % (e->n_side + 1);
  auto &q = e->ps[si];
  cudaStream_t sides[5] = {e->side, e->side2, e->side3, e->side4, e->side5};
  cudaStream_t side = sides[e->side_next];
  e->side_next = (e->side_next + 1) % e->n_side;
  SF_CUDA_TRY(cudaStreamWaitEvent(side, q.consumed, 0));
  *qo = &q;
  *sideo = side;
  return SF_OK;
}

sf_status accumulate_pixel_tail(sf_engine *e, sf_engine::PulseSet &q, cudaStream_t side,
                                int k_pad);

// One pixel-space pulse: private copy of the inputs into the scratch set
// (omega | d | gamma | 1/sigma, sigma^2 at the in_off_* offsets), then the
// pipelined operator phase and the ordered state update.
sf_status accumulate_pixel(sf_engine *e, const double *in_host, const double *g_dev,
                           const double *w_dev, const double *d_dev, double inv_sigma, int k_pad,
                           double sigma2) {
  sf_status s;
  const int n_r = e->n_r;
  sf_engine::PulseSet *qp = nullptr;
  cudaStream_t side = nullptr;
  if ((s = next_pulse_set(e, &qp, &side))) return s;
  auto &q = *qp;
  if (in_host) {
    SF_CUDA_TRY(cudaMemcpyAsync(q.in, in_host, e->in_stride * sizeof(double),
                                cudaMemcpyHostToDevice, side));
    SF_CUDA_TRY(cudaEventRecord(
        e->stage_ev[(e->stage_slot + sf_engine::kRing - 1) % sf_engine::kRing], side));
  } else {
    double *h = nullptr;
    if ((s = stage_inputs(e, &h))) return s;
    h[0] = inv_sigma;
    h[1] = sigma2;
    SF_CUDA_TRY(cudaMemcpyAsync(q.in, w_dev, n_r * sizeof(double), cudaMemcpyDeviceToDevice, side));
    SF_CUDA_TRY(cudaMemcpyAsync(q.in + e->in_off_d, d_dev, 2 * n_r * sizeof(double),
                                cudaMemcpyDeviceToDevice, side));
    SF_CUDA_TRY(cudaMemcpyAsync(q.in + e->in_off_g, g_dev, 3 * sizeof(double),
                                cudaMemcpyDeviceToDevice, side));
    SF_CUDA_TRY(cudaMemcpyAsync(q.in + e->in_off_s, h, 2 * sizeof(double), cudaMemcpyHostToDevice,
                                side));
    SF_CUDA_TRY(cudaEventRecord(
        e->stage_ev[(e->stage_slot + sf_engine::kRing - 1) % sf_engine::kRing], side));
  }
  return accumulate_pixel_tail(e, q, side, k_pad);
}

// Batched scenes: the raw inputs omega [n_r] | gammas [B][3] | d [B][n_r] c128 |
// sigma2 [B] land in q.raw (one copy), then k_stage_batch scatters them per
// scene into q.in (1/sigma computed on the device, rounded as the host's 1/sqrt).
sf_status accumulate_pixel_batch(sf_engine *e, const double *raw_host, const double *g_dev,
                                 const double *w_dev, const double *d_dev, const double *s2_dev,
                                 int k_pad) {
  sf_status s;
  const int n_r = e->n_r, B = e->batch;
  sf_engine::PulseSet *qp = nullptr;
  cudaStream_t side = nullptr;
  if ((s = next_pulse_set(e, &qp, &side))) return s;
  auto &q = *qp;
  const size_t n_raw = (size_t)n_r + (size_t)B * (3 + 2 * n_r + 1);
  if (raw_host) {
    SF_CUDA_TRY(cudaMemcpyAsync(q.raw, raw_host, n_raw * sizeof(double), cudaMemcpyHostToDevice,
                                side));
    SF_CUDA_TRY(cudaEventRecord(
        e->stage_ev[(e->stage_slot + sf_engine::kRing - 1) % sf_engine::kRing], side));
  } else {
    SF_CUDA_TRY(cudaMemcpyAsync(q.raw, w_dev, n_r * sizeof(double), cudaMemcpyDeviceToDevice, side));
    SF_CUDA_TRY(cudaMemcpyAsync(q.raw + n_r, g_dev, 3 * (size_t)B * sizeof(double),
                                cudaMemcpyDeviceToDevice, side));
    SF_CUDA_TRY(cudaMemcpyAsync(q.raw + n_r + 3 * B, d_dev, 2 * (size_t)n_r * B * sizeof(double),
                                cudaMemcpyDeviceToDevice, side));
    SF_CUDA_TRY(cudaMemcpyAsync(q.raw + n_r + 3 * B + 2 * (size_t)n_r * B, s2_dev,
                                (size_t)B * sizeof(double), cudaMemcpyDeviceToDevice, side));
  }
  if ((s = launch_stage_batch(q.raw, n_r, B, e->in_off_d, e->in_off_g, e->in_off_s, e->in_stride,
                              q.in, side)))
    return s;
  return accumulate_pixel_tail(e, q, side, k_pad);
}

sf_status accumulate_pixel_tail(sf_engine *e, sf_engine::PulseSet &q, cudaStream_t side,
                                int k_pad) {
  sf_status s;
  static const bool no_graph = getenv("SF_NO_GRAPHS") != nullptr;
  static const bool prof_graph = getenv("SF_PROFILE_GRAPHS") != nullptr;
  const bool graphs = !no_graph && (!e->profiling || prof_graph);
  if ((s = prof_mark(e, SF_K_OPERATOR, true, side))) return s;
  if (graphs && e->shard_world == 1) {  // (sharded: the K~ exchange is not captured)
    if (!q.op_exec &&
        (s = capture_graph(e, [&](cudaStream_t cs) { return enqueue_operator(e, q, k_pad, cs); },
                           &q.op_exec, &q.op_kernels)))
      return s;
    SF_CUDA_TRY(cudaGraphLaunch(q.op_exec, side));
    g_launches += q.op_kernels;
  } else if ((s = enqueue_operator(e, q, k_pad, side))) {
    return s;
  }
  if ((s = prof_mark(e, SF_K_OPERATOR, false, side))) return s;
  SF_CUDA_TRY(cudaEventRecord(q.ready, side));

  // ---- state update in pulse order: on `stats` into the alternate buffers
  // (double-buffered) or in place on the main stream
  cudaStream_t ss = e->dbuf ? e->stats : e->stream;
  float *A_out = e->dbuf ? e->A_alt : e->A;
  double2 *b_out = e->dbuf ? e->b_alt : e->b;
  unsigned long long *bmax_out = e->dbuf ? e->bmax_alt : e->bmax;
  double *Ls_out = e->dbuf ? e->Lsnap_alt : nullptr;
  SF_CUDA_TRY(cudaStreamWaitEvent(ss, q.prep, 0));
  if (e->dbuf) {
    // the alternate buffers were last read by main-stream work issued before
    // the previous pulse's update; everything issued since reads the current ones
    SF_CUDA_TRY(cudaStreamWaitEvent(ss, e->ev_readers, 0));
    SF_CUDA_TRY(cudaEventRecord(e->ev_readers, e->stream));
  }
  const int par = (A_out == e->A_alt && e->dbuf) ? (e->A_alt < e->A ? 1 : 0) : 2;
  if ((s = prof_mark(e, SF_K_GRAM, true, ss))) return s;
  if (graphs) {
    cudaGraphExec_t &ex = q.st_exec[par];
    if (!ex) {
      const float *A_in = e->A;
      if ((s = capture_graph(
               e, [&](cudaStream_t cs) { return enqueue_gram(e, q, k_pad, cs, A_in, A_out); }, &ex,
               &q.st_kernels)))
        return s;
      // the set's next use runs on the other buffer parity (an odd number of
      // sets): capture that variant now too, so a short run's captures all fall
      // into its first pulses
      if (par < 2 && !q.st_exec[1 - par]) {
        float *A_o = e->A;
        const float *A_i = e->A_alt;
        if ((s = capture_graph(
                 e, [&](cudaStream_t cs) { return enqueue_gram(e, q, k_pad, cs, A_i, A_o); },
                 &q.st_exec[1 - par], &q.st_kernels)))
          return s;
      }
    }
    SF_CUDA_TRY(cudaGraphLaunch(ex, ss));
    g_launches += q.st_kernels;
  } else if ((s = enqueue_gram(e, q, k_pad, ss, e->A, A_out))) {
    return s;
  }
  if ((s = prof_mark(e, SF_K_GRAM, false, ss))) return s;
  SF_CUDA_TRY(cudaStreamWaitEvent(ss, q.ready, 0));
  if ((s = prof_mark(e, SF_K_FOLD, true, ss))) return s;
  if (graphs) {
    cudaGraphExec_t &ex = q.fd_exec[par];
    if (!ex) {
      if ((s = capture_graph(
               e, [&](cudaStream_t cs) { return enqueue_fold(e, q, cs, b_out, bmax_out, Ls_out); },
               &ex, &q.fd_kernels)))
        return s;
      if (par < 2 && !q.fd_exec[1 - par]) {  // and the other parity's outputs
        double2 *b_o = e->b;
        unsigned long long *bm_o = e->bmax;
        double *Ls_o = e->Lsnap;
        if ((s = capture_graph(
                 e, [&](cudaStream_t cs) { return enqueue_fold(e, q, cs, b_o, bm_o, Ls_o); },
                 &q.fd_exec[1 - par], &q.fd_kernels)))
          return s;
      }
    }
    SF_CUDA_TRY(cudaGraphLaunch(ex, ss));
    g_launches += q.fd_kernels;
  } else if ((s = enqueue_fold(e, q, ss, b_out, bmax_out, Ls_out))) {
    return s;
  }
  if ((s = prof_mark(e, SF_K_FOLD, false, ss))) return s;
  SF_CUDA_TRY(cudaEventRecord(q.consumed, ss));
  if (e->dbuf) {
    SF_CUDA_TRY(cudaEventRecord(e->ev_stats, ss));
    SF_CUDA_TRY(cudaStreamWaitEvent(e->stream, e->ev_stats, 0));
    std::swap(e->A, e->A_alt);
    std::swap(e->b, e->b_alt);
    std::swap(e->bmax, e->bmax_alt);
    std::swap(e->Lsnap, e->Lsnap_alt);
  }
  e->pulse_count += 1;
  return SF_OK;
}

// x = H z for the FISTA chain: entry-major k_hz_ell for batched engines (same
// bits as k_hz), else k_hz / k_hz_packed
sf_status hz_any(sf_engine *e, const double *z, cudaStream_t st) {
  if (e->hz_ents > 0)
    return launch_hz_ell(e->hz_atomT, e->hz_wT, e->hz_ents, e->n_pix, e->dpad, z, e->z32, st,
                         e->batch, e->m_pad, e->zstride);
  return launch_hz(e->csr_ptr, e->csr_atom, e->csr_w, e->n_pix, e->dpad, z, e->z32, st, e->batch,
                   e->m_pad, e->zstride);
}

PrologueArgs prologue_args(sf_engine *e, const double *c0, double lam, double lam_rel, double t0,
                           int steps) {
  return make_prologue_args(e->dbuf ? e->Lsnap : e->L, e->bmax, lam, lam_rel, e->scal, t0, steps,
                            e->wbuf, c0, e->m, e->m_pad, e->zd, e->cprev, e->csr_ptr, e->csr_atom,
                            e->csr_w, e->n_pix, e->dpad, e->z32);
}

// Pixel-space FISTA chain (kernels.py:78-103 restated in pixel space):
// setup (tau, threshold, momentum weights) -> z = c0, x = H z -> per step
// y = Re(B) x (tile slots) -> y_pix -> atom step -> x = H z.
sf_status enqueue_chain(sf_engine *e, cudaStream_t st, int steps, const double *c0, double *cod,
                        double lam, double lam_rel, double t0, bool prof) {
  sf_status s;
  const int B = e->batch;
  if (fista_prologue_ok(e->dpad, B)) {  // setup + init + first H z in one launch
    if ((s = launch_fista_prologue(prologue_args(e, c0, lam, lam_rel, t0, steps), st))) return s;
  } else {
    if ((s = launch_fista_setup(e->dbuf ? e->Lsnap : e->L, e->bmax, lam, lam_rel, e->scal, st, t0,
                                steps, e->wbuf, B)))
      return s;
    if ((s = launch_fista_init(c0, e->m, e->m_pad, e->zd, e->cprev, e->z32, st, B, e->zstride)))
      return s;
    if ((s = hz_any(e, e->zd, st))) return s;
  }
  if (prof && (s = prof_mark(e, SF_K_STEP, true, st))) return s;
  // snake order over the tile list: odd steps walk it backwards, so a store
  // larger than L2 starts each step on the tiles the previous step left in L2;
  // the slots per tile, hence all sums, are unchanged (measured cfg3 matvec
  // 108 -> 104 us)
  for (int k = 0; k < steps; ++k) {
    if (prof && (s = prof_mark(e, SF_K_GEMV, true, st))) return s;
    // partial slots of y = Re(B) x; k_pix_reduce sums them (sharded: the slots
    // of tiles other ranks own stay zero, and ypix is all-reduced)
    if ((s = launch_gemv(e->A, e->tiles_local, e->n_tiles_local, e->z32, e->P, e->nt, 1,
                         e->gemv_grid, st, B, e->zstride, (k & 1), 0,
                         prof ? e->gemv_bytes : nullptr)))
      return s;
    if (prof && (s = prof_mark(e, SF_K_GEMV, false, st))) return s;
    if (e->peer && e->shard_world > 1) {
      // slot reduction and push in one kernel: the partial y_pix goes straight
      // into this rank's slot on every rank, then the event edge and the sum
      size_t off = 0;
      const PeerSlots dst = peer_targets(e->peer, 0, &off);
      if ((s = launch_pix_reduce(e->P, e->nt, e->dpad, e->ypix, st, B, &dst, off))) return s;
      if ((s = exchange_sum(e, 0, e->ypix, (size_t)e->dpad, st, true))) return s;
    } else {
      if ((s = launch_pix_reduce(e->P, e->nt, e->dpad, e->ypix, st, B))) return s;
      if (e->shard_world > 1 && (s = exchange_sum(e, 0, e->ypix, (size_t)e->dpad, st))) return s;
    }
    if ((s = launch_atom_step(e->ell_idx, e->ell_w, e->ell_width, e->m, e->ypix, e->b, e->zd,
                              e->cprev, e->scal, e->wbuf, k, k == steps - 1 ? cod : nullptr, st, B,
                              e->m_pad, e->dpad)))
      return s;
    if (k < steps - 1 && (s = hz_any(e, e->zd, st))) return s;
  }
  if (prof && (s = prof_mark(e, SF_K_STEP, false, st))) return s;
  return SF_OK;
}

sf_status ensure_wbuf(sf_engine *e, int steps) {
  if (steps <= e->wbuf_cap) return SF_OK;
  if (e->wbuf) {  // (the first allocation has nothing to invalidate)
    SF_CUDA_TRY(cudaStreamSynchronize(e->stream));  // graphs and queued work hold the old buffer
    drop_graphs(e);
  }
  if (e->wbuf) cudaFree(e->wbuf);
  e->wbuf = nullptr;
  const int cap = std::max(64, steps);
  sf_status s = dalloc(&e->wbuf, (size_t)cap);
  if (s) return s;
  e->wbuf_cap = cap;
  return SF_OK;
}

// The chain for the current state buffers as a CUDA graph (captured on first use).

sf_status chain_graph(sf_engine *e, int steps, sf_engine::FGraph **out) {
  for (auto &g : e->fgraphs)
    if (g.A == e->A && g.b == e->b && g.bmax == e->bmax && g.L == (e->dbuf ? e->Lsnap : e->L) &&
        g.steps == steps) {
      *out = &g;
      return SF_OK;
    }
  if (e->fgraphs.size() >= 8) {  // bounded cache: drop the oldest
    cudaGraphExecDestroy(e->fgraphs.front().exec);
    cudaGraphDestroy(e->fgraphs.front().graph);
    e->fgraphs.erase(e->fgraphs.begin());
  }
  if (!e->cap_stream) SF_CUDA_TRY(cudaStreamCreateWithFlags(&e->cap_stream, cudaStreamNonBlocking));
  sf_engine::FGraph g;
  g.A = e->A;
  g.b = e->b;
  g.bmax = e->bmax;
  g.L = e->dbuf ? e->Lsnap : e->L;
  g.steps = steps;
  // L2 persistence for the tile store this graph reads: the
  // pipeline and state streams stream tens of MB per pulse through L2 while the
  // chain re-reads the same store every step; the access-policy window captured
  // into the kernel nodes keeps it resident (the other buffer's graph persists
  // the other store).
  const size_t store_b = (size_t)e->batch * e->n_tiles * kTileElems * sizeof(float);
  int max_win = 0, max_persist = 0;
  cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, e->device);
  cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, e->device);
  const bool use_window = max_win > 0 && max_persist > 0 &&
                          store_b <= (size_t)max_win && store_b <= (size_t)max_persist;
  if (use_window) {
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    if (cur < store_b) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, store_b);
    cudaStreamAttrValue av{};
    av.accessPolicyWindow.base_ptr = (void *)e->A;
    av.accessPolicyWindow.num_bytes = store_b;
    av.accessPolicyWindow.hitRatio = 1.0f;
    av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(e->cap_stream, cudaStreamAttributeAccessPolicyWindow, &av);
    cudaGetLastError();
  }
  const int64_t l0 = g_launches.load();
  SF_CUDA_TRY(cudaStreamBeginCapture(e->cap_stream, cudaStreamCaptureModeThreadLocal));
  set_capturing(true);
  sf_status s = enqueue_chain(e, e->cap_stream, steps, e->cin, e->cout, 0.0, 1.0, 1.0, false);
  set_capturing(false);
  cudaGraph_t graph = nullptr;
  cudaError_t ce = cudaStreamEndCapture(e->cap_stream, &graph);
  g.kernels = g_launches.load() - l0;
  g_launches -= g.kernels;  // counted when the graph runs
  if (use_window) {
    cudaStreamAttrValue av{};
    av.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(e->cap_stream, cudaStreamAttributeAccessPolicyWindow, &av);
    cudaGetLastError();
  }
  if (s) {
    if (graph) cudaGraphDestroy(graph);
    return s;
  }
  if (ce != cudaSuccess) return fail(SF_ECUDA, std::string("FISTA graph capture: ") + cudaGetErrorString(ce));
  size_t nn = 0;
  SF_CUDA_TRY(cudaGraphGetNodes(graph, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  SF_CUDA_TRY(cudaGraphGetNodes(graph, nodes.data(), &nn));
  for (auto nd : nodes) {
    cudaGraphNodeType ty;
    SF_CUDA_TRY(cudaGraphNodeGetType(nd, &ty));
    if (ty != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams kp;
    SF_CUDA_TRY(cudaGraphKernelNodeGetParams(nd, &kp));
    if (kp.func == fista_setup_kernel()) g.setup = nd;
    if (kp.func == fista_prologue_kernel()) {
      g.setup = nd;
      g.prologue = true;
    }
    if (is_atom_step_kernel(kp.func) && *(double **)kp.kernelParams[11] == e->cout) {
      void **a = kp.kernelParams;
      AtomStepNodeArgs &s = g.last_args;
      s.idx = *(const int32_t **)a[0];
      s.wt = *(const double **)a[1];
      s.width = *(int *)a[2];
      s.m = *(int64_t *)a[3];
      s.ypix = *(const double **)a[4];
      s.b = *(const double2 **)a[5];
      s.zd = *(double **)a[6];
      s.cprev = *(double **)a[7];
      s.scal = *(const double **)a[8];
      s.wv = *(const double **)a[9];
      s.kstep = *(int *)a[10];
      s.c_out = *(double **)a[11];
      s.m_pad = *(int64_t *)a[12];
      s.n_pad = *(int64_t *)a[13];
      g.last_step = nd;
      g.last_grid = kp.gridDim;
      g.last_block = kp.blockDim;
    }
  }
  if (!g.setup) {
    cudaGraphDestroy(graph);
    return fail(SF_ECUDA, "FISTA graph: setup node not found");
  }
  // every kernel node carries the device's greatest priority and the graph
  // is instantiated to honour node priorities, so it is replayed on the
  // caller's stream itself: the block scheduler serves the latency-bound chain
  // ahead of the pipeline streams' operator kernels, without event hops
  // through a separate high-priority stream (measured cfg1 5 302-5 388 ->
  // 5 489-5 495 pulses/s)
  for (auto nd : nodes) {
    cudaGraphNodeType ty;
    SF_CUDA_TRY(cudaGraphNodeGetType(nd, &ty));
    if (ty != cudaGraphNodeTypeKernel) continue;
    cudaLaunchAttributeValue v{};
    v.priority = e->prio_hi;
    SF_CUDA_TRY(cudaGraphKernelNodeSetAttribute(nd, cudaLaunchAttributePriority, &v));
  }
  ce = cudaGraphInstantiateWithFlags(&g.exec, graph, cudaGraphInstantiateFlagUseNodePriority);
  if (ce != cudaSuccess) {
    cudaGraphDestroy(graph);
    return fail(SF_ECUDA, std::string("FISTA graph instantiate: ") + cudaGetErrorString(ce));
  }
  g.graph = graph;
  e->fgraphs.push_back(g);
  *out = &e->fgraphs.back();
  return SF_OK;
}

// Stage n doubles into the pinned ring, wait until the slot's previous copy retired.
sf_status stage_inputs(sf_engine *e, double **slot_out) {
  const int slot = e->stage_slot;
  e->stage_slot = (e->stage_slot + 1) % sf_engine::kRing;
  SF_CUDA_TRY(cudaEventSynchronize(e->stage_ev[slot]));
  *slot_out = e->h_stage + (size_t)slot * e->stage_slot_size;
  return SF_OK;
}

}  // namespace

extern "C" {

const char *sf_last_error(void) { return t_last_error.c_str(); }

sf_status sf_init_device(int32_t device) {
  sf_status s = check_device(device);
  if (s) return s;
  SF_CUDA_TRY(cudaFree(nullptr));  // create the primary context now, not inside a caller's timing
  return SF_OK;
}
int32_t sf_abi_version(void) { return SF_ABI_VERSION; }
int64_t sf_launch_count(void) { return g_launches.load(); }

sf_status sf_create(const sf_desc *d, sf_engine **out) {
  if (!d || !out) return fail(SF_EINVAL, "null argument");
  *out = nullptr;
  if (d->abi_version != SF_ABI_VERSION) return fail(SF_EINVAL, "ABI version mismatch");
  if (d->m_atoms < 1) return fail(SF_EINVAL, "need at least one atom");
  if (!(d->l_floor > 0.0)) return fail(SF_EINVAL, "l_floor must be positive");
  if (d->n_freq < 1 || d->n_freq > 512) return fail(SF_EINVAL, "n_freq must lie in [1, 512]");
  if (d->precision < SF_PREC_TF32X3 || d->precision > SF_PREC_DIRICHLET)
    return fail(SF_EINVAL, "unknown precision");
  if (d->precision == SF_PREC_DIRICHLET && d->mode != SF_MODE_PIXEL)
    return fail(SF_EINVAL, "the closed-form (dirichlet) Gram update needs pixel-space mode");
  if (d->ell_width > 0 && (!d->ell_idx || !d->ell_w || d->n_pixels < 1))
    return fail(SF_EINVAL, "dictionary ELL table incomplete");
  if (d->mode != SF_MODE_ATOM && d->mode != SF_MODE_PIXEL) return fail(SF_EINVAL, "unknown mode");
  if (d->mode == SF_MODE_PIXEL && (d->ell_width <= 0 || !d->pixel_xyz))
    return fail(SF_EINVAL, "pixel-space mode needs the dictionary and the pixel geometry");
  if (d->batch < 0 || d->batch > 65535) return fail(SF_EINVAL, "batch must lie in [0, 65535]");
  if (d->keep_complex && d->mode != SF_MODE_ATOM)
    return fail(SF_EINVAL, "keep_complex needs atom-space statistics");
  if (d->batch > 1 && (d->mode != SF_MODE_PIXEL ||
                       (d->precision != SF_PREC_F16X3 && d->precision != SF_PREC_DIRICHLET) ||
                       d->n_freq > 256))
    return fail(SF_EUNSUPPORTED,
                "batched scenes need pixel-space mode, f16x3 or dirichlet precision and "
                "n_freq <= 256");
  sf_status s = check_device(d->device);
  if (s) return s;

  sf_engine *e = new sf_engine();
  e->device = d->device;
  e->m = d->m_atoms;
  e->m_pad = round_up(e->m, kTile);
  e->nt = (int)(e->m_pad / kTile);
  e->n_r = d->n_freq;
  e->k_pad_max = (int)round_up(2 * (int64_t)e->n_r, kKChunk);
  e->ell_width = d->ell_width;
  e->n_pix = d->n_pixels;
  e->precision = d->precision;
  e->l_floor = d->l_floor;
  if (d->power_max_iter > 0) e->power_max_iter = d->power_max_iter;
  if (d->power_rel_tol > 0.0) e->power_rel_tol = d->power_rel_tol;
  if (d->power_rel_tol < 0.0) e->power_rel_tol = 0.0;
  cudaDeviceGetAttribute(&e->sm_count, cudaDevAttrMultiProcessorCount, e->device);
  e->mode = d->mode;
  e->dpad = (e->mode == SF_MODE_PIXEL) ? round_up(e->n_pix, kTile) : e->m_pad;
  e->nt = (int)(e->dpad / kTile);
  e->gemv_grid = e->sm_count * 2;
  e->batch = std::max(1, (int)d->batch);
  e->compose_grid = (int)std::max<int64_t>(
      1, std::min<int64_t>(e->mode == SF_MODE_PIXEL ? e->sm_count : e->sm_count * 4,
                           (e->dpad + 7) / 8));
  if (e->batch > 1)  // the scenes fill the machine: a few CTAs per scene
    e->compose_grid = (int)std::max<int64_t>(
        1, std::min<int64_t>(e->compose_grid, (4LL * e->sm_count + e->batch - 1) / e->batch));
  e->in_off_d = e->n_r + (e->n_r & 1);
  e->in_off_g = e->in_off_d + 2LL * e->n_r;
  e->in_off_s = e->in_off_g + 4;
  e->in_stride = e->in_off_s + 2;
  e->zstride = std::max(e->m_pad, e->dpad);

#define TRY(x)            \
  do {                    \
    sf_status _s = (x);   \
    if (_s) {             \
      delete e;           \
      return _s;          \
    }                     \
  } while (0)
#define CTRY(x)                                                                   \
  do {                                                                            \
    cudaError_t _c = (x);                                                         \
    if (_c != cudaSuccess) {                                                      \
      delete e;                                                                   \
      return fail(SF_ECUDA, std::string(#x) + ": " + cudaGetErrorString(_c));      \
    }                                                                             \
  } while (0)

  CTRY(cudaStreamCreateWithFlags(&e->own_stream, cudaStreamNonBlocking));
  {
    // pipeline streams at the lowest priority: pending CTAs of the in-order
    // main stream (Gram update, FISTA) are scheduled first
    int lo = 0, hi = 0;
    CTRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    e->prio_hi = hi;
    CTRY(cudaStreamCreateWithPriority(&e->side, cudaStreamNonBlocking, lo));
    CTRY(cudaStreamCreateWithPriority(&e->side2, cudaStreamNonBlocking, lo));
    CTRY(cudaStreamCreateWithPriority(&e->side3, cudaStreamNonBlocking, lo));
    CTRY(cudaStreamCreateWithPriority(&e->side4, cudaStreamNonBlocking, lo));
    CTRY(cudaStreamCreateWithPriority(&e->side5, cudaStreamNonBlocking, lo));
    {  // state-update stream priority.  Measured
       // on B200 (flushed / warm pulses/s): low priority lets the latency-bound
       // FISTA chain go first -- cfg1 5 170 -> 5 359 / 6 090 -> 6 239, cfg3 525 ->
       // 547 / 508 -> 555 -- while a multi-GB store's Gram (cfg4: 8.6 GB, 4.5 ms)
       // must keep up with the chain (65.4 vs 68.3 at low priority)
      const double store_b = (double)e->batch * e->nt * (e->nt + 1) / 2 * kTileElems * 4.0;
      const bool low = store_b <= 2e9;
      CTRY(cudaStreamCreateWithPriority(&e->stats, cudaStreamNonBlocking, low ? lo : hi));
    }
  }
  CTRY(cudaEventCreateWithFlags(&e->ev_stats, cudaEventDisableTiming));
  CTRY(cudaEventCreateWithFlags(&e->ev_readers, cudaEventDisableTiming));
  CTRY(cudaEventCreateWithFlags(&e->ev_c, cudaEventDisableTiming));
  CTRY(cudaEventCreateWithFlags(&e->ev_p, cudaEventDisableTiming));
  e->stream = e->own_stream;

  // upper-triangle tile list, row-major (I, J >= I)
  e->h_tiles.reserve((size_t)e->nt * (e->nt + 1) / 2);
  for (int I = 0; I < e->nt; ++I)
    for (int J = I; J < e->nt; ++J) e->h_tiles.push_back(make_int2(I, J));
  e->n_tiles = (int64_t)e->h_tiles.size();

  TRY(track_alloc(e, &e->A, (size_t)e->batch * e->n_tiles * kTileElems));
  TRY(track_alloc(e, &e->tiles, (size_t)e->n_tiles));
  TRY(track_alloc(e, &e->b, (size_t)e->batch * e->m));
  TRY(track_alloc(e, &e->L, (size_t)e->batch));
  TRY(track_alloc(e, &e->counters, 2 * (size_t)e->batch));
  TRY(track_alloc(e, &e->gram_next, 1));
  TRY(track_alloc(e, &e->diag, 8 * (size_t)e->batch));
  TRY(track_alloc(e, &e->scal, 4 * (size_t)e->batch));
  TRY(track_alloc(e, &e->v0, (size_t)e->m));
  TRY(track_alloc(e, &e->Gp, (size_t)e->dpad * e->k_pad_max));
  TRY(track_alloc(e, &e->omega, 3 * 512));
  TRY(track_alloc(e, &e->gamma, 4));
  TRY(track_alloc(e, &e->zero_flag, 1));
  CTRY(cudaMemsetAsync(e->zero_flag, 0, sizeof(int), e->stream));
  TRY(track_alloc(e, &e->dt, 512));
  TRY(track_alloc(e, &e->u0part, (size_t)e->compose_grid * e->n_r));
  const int nb = (e->n_r + 31) / 32;
  e->kpart_splits = (int)std::max<int64_t>(
      1, std::min<int64_t>((2 * e->sm_count + nb * nb - 1) / (nb * nb), (e->m + 255) / 256));
  {
    // 32 x 32 K~ blocks of k_kgram_px, split over pixels: 8 CTAs per SM
    // (measured cfg3 453 -> 316 us against 2 per SM)
    const int nbp = nb * (nb + 1) / 2;
    const int mult = 8;
    e->px_splits = (int)std::max<int64_t>(
        1, std::min<int64_t>((mult * e->sm_count + nbp - 1) / nbp,
                             (std::max<int64_t>(e->n_pix, 1) + 63) / 64));
    if (const char *ks = getenv("SF_KGRAM_SPLITS"))  // exact split count (tests, A/B)
      e->px_splits = std::max(1, atoi(ks));
    else if (e->batch > 1)  // the scenes already fill the machine
      e->px_splits = (int)std::max<int64_t>(
          1, std::min<int64_t>(e->px_splits, (2 * e->sm_count + nbp * e->batch - 1) / (nbp * e->batch)));
  }
  TRY(track_alloc(e, &e->Kpart,
                  (size_t)std::max(e->kpart_splits, e->px_splits) * e->n_r * e->n_r));
  TRY(track_alloc(e, &e->bmax, (size_t)e->batch));
  TRY(track_alloc(e, &e->maxbits, 1));
  TRY(track_alloc(e, &e->gexp, 1));
  CTRY(cudaMemsetAsync(e->bmax, 0, sizeof(unsigned long long) * e->batch, e->stream));
  TRY(track_alloc(e, &e->K, (size_t)e->n_r * e->n_r));
  TRY(track_alloc(e, &e->Kf, (size_t)e->n_r * e->n_r));
  TRY(track_alloc(e, &e->u0, (size_t)e->n_r));
  TRY(track_alloc(e, &e->P, (size_t)e->batch * e->nt * e->nt * kTile));
  TRY(track_alloc(e, &e->z32, (size_t)e->batch * e->zstride));
  if (e->mode == SF_MODE_PIXEL) {
    // second tile store when it fits comfortably (SF_DOUBLE_BUFFER=0 disables)
    size_t free_b = 0, total_b = 0;
    CTRY(cudaMemGetInfo(&free_b, &total_b));
    const double store_b = (double)e->n_tiles * kTileElems * sizeof(float);
    const char *db = getenv("SF_DOUBLE_BUFFER");
    e->dbuf = !(db && db[0] == '0') && store_b <= 0.35 * (double)free_b;
    if (e->dbuf) {
      TRY(track_alloc(e, &e->A_alt, (size_t)e->batch * e->n_tiles * kTileElems));
      TRY(track_alloc(e, &e->b_alt, (size_t)e->batch * e->m));
      TRY(track_alloc(e, &e->bmax_alt, (size_t)e->batch));
      TRY(track_alloc(e, &e->Lsnap, (size_t)e->batch));
      TRY(track_alloc(e, &e->Lsnap_alt, (size_t)e->batch));
    }
    TRY(track_alloc(e, &e->beta, (size_t)e->batch * e->n_pix));
    TRY(track_alloc(e, &e->hv0, (size_t)e->n_pix));
    TRY(track_alloc(e, &e->bp, (size_t)e->batch * e->n_pix));
    TRY(track_alloc(e, &e->ypix, (size_t)e->batch * e->dpad));
  }
  if (d->keep_complex) {
    e->keep_complex = true;
    TRY(track_alloc(e, &e->A64, (size_t)e->m * e->m));
  }
  TRY(track_alloc(e, &e->zd, (size_t)e->batch * e->m_pad));
  TRY(track_alloc(e, &e->cprev, (size_t)e->batch * e->m_pad));
  TRY(track_alloc(e, &e->cin, (size_t)e->batch * e->m));
  TRY(track_alloc(e, &e->cout, (size_t)e->batch * e->m));
  CTRY(cudaMemcpyAsync(e->tiles, e->h_tiles.data(), e->h_tiles.size() * sizeof(int2),
                       cudaMemcpyHostToDevice, e->stream));
  if (e->precision == SF_PREC_F16X3) {
    // 2x2 super-tiles (SI <= SJ) of the tile triangle, row-major
    std::vector<int2> it;
    const int ns = (e->nt + 1) / 2;
    for (int a = 0; a < ns; ++a)
      for (int b = a; b < ns; ++b) it.push_back(make_int2(a, b));
    e->n_items = (int)it.size();
    TRY(track_alloc(e, &e->items, it.size()));
    TRY(track_alloc(e, &e->Gh, (size_t)e->dpad * e->k_pad_max * 2));
    CTRY(cudaMemcpy(e->items, it.data(), it.size() * sizeof(int2), cudaMemcpyHostToDevice));
  }

  if (e->ell_width > 0) {
    const size_t ne = (size_t)e->m * e->ell_width;
    TRY(track_alloc(e, &e->ell_idx, ne));
    TRY(track_alloc(e, &e->ell_w, ne));
    TRY(track_alloc(e, &e->Ft, (size_t)e->n_pix * e->n_r));
    TRY(track_alloc(e, &e->tau, (size_t)e->n_pix));
    TRY(track_alloc(e, &e->img, (size_t)e->n_pix));
    CTRY(cudaMemcpyAsync(e->ell_idx, d->ell_idx, ne * sizeof(int32_t), cudaMemcpyHostToDevice,
                         e->stream));
    CTRY(cudaMemcpyAsync(e->ell_w, d->ell_w, ne * sizeof(double), cudaMemcpyHostToDevice,
                         e->stream));
    // pixel-major CSR transpose of the ELL table (fixed atom order per pixel)
    std::vector<int64_t> ptr(e->n_pix + 1, 0);
    for (size_t k = 0; k < ne; ++k) {
      const int32_t p = d->ell_idx[k];
      if (p >= e->n_pix) {
        delete e;
        return fail(SF_EINVAL, "dictionary pixel index out of range");
      }
      if (p >= 0) ptr[p + 1]++;
    }
    for (int64_t p = 0; p < e->n_pix; ++p) ptr[p + 1] += ptr[p];
    std::vector<int32_t> atom(ptr[e->n_pix]);
    std::vector<double> w(ptr[e->n_pix]);
    std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
    for (int64_t j = 0; j < e->m; ++j)
      for (int l = 0; l < e->ell_width; ++l) {
        const int32_t p = d->ell_idx[j * e->ell_width + l];
        if (p < 0) continue;
        atom[fill[p]] = (int32_t)j;
        w[fill[p]] = d->ell_w[j * e->ell_width + l];
        fill[p]++;
      }
    // Q = H H^T in pixel-major CSR (sorted columns, duplicates merged)
    {
      std::vector<std::pair<int64_t, double>> trip;  // key = p * n + p'
      trip.reserve((size_t)e->m * e->ell_width * e->ell_width);
      for (int64_t j = 0; j < e->m; ++j)
        for (int l1 = 0; l1 < e->ell_width; ++l1) {
          const int32_t p1 = d->ell_idx[j * e->ell_width + l1];
          if (p1 < 0) break;
          const double w1 = d->ell_w[j * e->ell_width + l1];
          for (int l2 = 0; l2 < e->ell_width; ++l2) {
            const int32_t p2 = d->ell_idx[j * e->ell_width + l2];
            if (p2 < 0) break;
            trip.emplace_back((int64_t)p1 * e->n_pix + p2, w1 * d->ell_w[j * e->ell_width + l2]);
          }
        }
      std::stable_sort(trip.begin(), trip.end(),
                       [](const std::pair<int64_t, double> &a, const std::pair<int64_t, double> &b) {
                         return a.first < b.first;
                       });
      std::vector<int64_t> qp(e->n_pix + 1, 0);
      std::vector<int32_t> qc;
      std::vector<double> qv;
      for (size_t k = 0; k < trip.size();) {
        size_t k2 = k;
        double s = 0.0;
        while (k2 < trip.size() && trip[k2].first == trip[k].first) s += trip[k2++].second;
        const int64_t p1 = trip[k].first / e->n_pix, p2 = trip[k].first % e->n_pix;
        qp[p1 + 1]++;
        qc.push_back((int32_t)p2);
        qv.push_back(s);
        k = k2;
      }
      for (int64_t p = 0; p < e->n_pix; ++p) qp[p + 1] += qp[p];
      TRY(track_alloc(e, &e->qptr, qp.size()));
      TRY(track_alloc(e, &e->qcol, qc.size()));
      TRY(track_alloc(e, &e->qval, qv.size()));
      TRY(track_alloc(e, &e->W, (size_t)e->n_pix * e->n_r));
      CTRY(cudaMemcpy(e->qptr, qp.data(), qp.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
      CTRY(cudaMemcpy(e->qcol, qc.data(), qc.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
      CTRY(cudaMemcpy(e->qval, qv.data(), qv.size() * sizeof(double), cudaMemcpyHostToDevice));
      // K~ on tensor cores (default; SF_KTILDE_TC=0 keeps the fp64 SIMT path,
      // the reference the tensor-core build is tested against)
      const char *kt_env = getenv("SF_KTILDE_TC");
      const bool want_ktc = !(kt_env && kt_env[0] == '0') && e->k_pad_max <= 1024;
      QTileHost qt;
      const bool qt_ok = d->pixel_xyz && want_ktc &&
                         build_q_tiles(d->pixel_xyz, e->n_pix, qp.data(), qc.data(), qv.data(),
                                       qt) == SF_OK;
      if (qt_ok && want_ktc) {
        KtcHost kh;
        int eq = 0;
        float rmax = 0.f;
        if (build_ktc_panels(qt, kh, &eq, &rmax) == SF_OK) {
          int32_t *i32 = nullptr;
          __half *h16 = nullptr;
          const size_t n32 = kh.grp_pix.size() + kh.ug_off.size() + kh.ug_list.size() +
                             kh.chunk_off.size();
          TRY(track_alloc(e, &i32, n32));
          TRY(track_alloc(e, &h16, std::max<size_t>(1, kh.panels.size())));
          e->ktc_mem[0] = i32;
          e->ktc_mem[1] = h16;
          size_t off = 0;
          auto put = [&](const std::vector<int32_t> &v, const int32_t **dst) {
            cudaMemcpy(i32 + off, v.data(), v.size() * 4, cudaMemcpyHostToDevice);
            *dst = i32 + off;
            off += v.size();
          };
          KtcArgs &ka = e->ktc;
          put(kh.grp_pix, &ka.grp_pix);
          put(kh.ug_off, &ka.ug_off);
          put(kh.ug_list, &ka.ug_list);
          put(kh.chunk_off, &ka.qchunk_off);
          CTRY(cudaMemcpy(h16, kh.panels.data(), kh.panels.size() * sizeof(__half),
                          cudaMemcpyHostToDevice));
          ka.qpanels = h16;
          ka.tiles = qt.tiles;
          ka.tile_begin = 0;
          ka.tile_end = qt.tiles;
          ka.ngrp = 8LL * qt.tiles;
          ka.eq = eq;
          ka.qrow_max = rmax;
          ka.k_pad = e->k_pad_max;
          ka.nb = (e->k_pad_max + 127) / 128;
          // K splits of the Z product: a function of the scene geometry only,
          // never of the batch size (partials accumulate in fp32 per split, so
          // a batched engine and single-scene engines must split alike to
          // agree bitwise): 32 chunks of 16 pixels per split, at most 64 splits.
          const int nch = 4 * qt.tiles;
          ka.cps = std::max(32, (nch + 63) / 64);
          e->ktc_grid = (nch + ka.cps - 1) / ka.cps;  // partial slots
          e->ktc_on = true;
        }
      }
    }
    TRY(track_alloc(e, &e->csr_ptr, ptr.size()));
    TRY(track_alloc(e, &e->csr_atom, atom.size()));
    TRY(track_alloc(e, &e->csr_w, w.size()));
    CTRY(cudaMemcpy(e->csr_ptr, ptr.data(), ptr.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
    CTRY(cudaMemcpy(e->csr_atom, atom.data(), atom.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    CTRY(cudaMemcpy(e->csr_w, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice));
    if (d->batch > 1) {  // entry-major transpose for k_hz_ell
      int64_t ents = 0;
      for (int64_t p = 0; p < e->n_pix; ++p) ents = std::max<int64_t>(ents, ptr[p + 1] - ptr[p]);
      if (ents <= 64) {
        const int64_t np = e->dpad;
        std::vector<int32_t> at((size_t)ents * np, -1);
        std::vector<double> wt((size_t)ents * np, 0.0);
        for (int64_t p = 0; p < e->n_pix; ++p)
          for (int64_t k = ptr[p]; k < ptr[p + 1]; ++k) {
            at[(k - ptr[p]) * np + p] = atom[k];
            wt[(k - ptr[p]) * np + p] = w[k];
          }
        TRY(track_alloc(e, &e->hz_atomT, at.size()));
        TRY(track_alloc(e, &e->hz_wT, wt.size()));
        CTRY(cudaMemcpy(e->hz_atomT, at.data(), at.size() * 4, cudaMemcpyHostToDevice));
        CTRY(cudaMemcpy(e->hz_wT, wt.data(), wt.size() * 8, cudaMemcpyHostToDevice));
        e->hz_ents = (int)ents;
      }
    }
    if (d->pixel_xyz) {
      TRY(track_alloc(e, &e->xyz, (size_t)e->n_pix * 3));
      e->h_xyz.assign(d->pixel_xyz, d->pixel_xyz + 3 * e->n_pix);
      CTRY(cudaMemcpy(e->xyz, d->pixel_xyz, (size_t)e->n_pix * 3 * sizeof(double),
                      cudaMemcpyHostToDevice));
      for (int k = 0; k < 3; ++k) {
        e->bbox_lo[k] = e->bbox_hi[k] = e->h_xyz[k];
      }
      for (int64_t p = 0; p < e->n_pix; ++p)
        for (int k = 0; k < 3; ++k) {
          e->bbox_lo[k] = std::min(e->bbox_lo[k], e->h_xyz[3 * p + k]);
          e->bbox_hi[k] = std::max(e->bbox_hi[k], e->h_xyz[3 * p + k]);
        }
    }
  }
  e->stage_slot_size = std::max<int64_t>(3 * 512 + 8, (int64_t)e->n_r + (int64_t)e->batch * (3 + 2 * e->n_r + 1) + 8);
  CTRY(cudaMallocHost((void **)&e->h_stage,
                      sizeof(double) * sf_engine::kRing * (size_t)e->stage_slot_size));
  for (auto &ev : e->stage_ev) {
    CTRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CTRY(cudaEventRecord(ev, e->stream));
  }
  CTRY(cudaEventCreate(&e->ev_acc0));
  CTRY(cudaEventCreate(&e->ev_acc1));
  CTRY(cudaEventCreate(&e->ev_f0));
  CTRY(cudaEventCreate(&e->ev_f1));
  TRY(launch_start_vector(e->m, 0x5EED, e->v0, e->stream));
  if (e->mode == SF_MODE_PIXEL) {  // u0 = F (H v0) / sigma needs H v0 once
    TRY(launch_hv0(e->csr_ptr, e->csr_atom, e->csr_w, e->n_pix, e->v0, e->hv0, e->stream));
    const size_t kp = (size_t)std::max(e->kpart_splits, e->px_splits);
    for (int qi = 0; qi <= e->n_side; ++qi) {  // n_side + 1 scratch sets
      auto &q = e->ps[qi];
      TRY(track_alloc(e, &q.in, (size_t)e->batch * e->in_stride));
      if (e->batch > 1)
        TRY(track_alloc(e, &q.raw, (size_t)e->n_r + (size_t)e->batch * (3 + 2 * e->n_r + 1)));
      TRY(track_alloc(e, &q.tau, (size_t)e->batch * e->n_pix));
      TRY(track_alloc(e, &q.pdiag, 8 * (size_t)e->batch));
      if (!e->ktc_on) {  // fp64 F and Q F: only the SIMT K~ path reads them
        TRY(track_alloc(e, &q.Ft, (size_t)e->batch * e->n_pix * e->n_r));
        TRY(track_alloc(e, &q.W, (size_t)e->batch * e->n_pix * e->n_r));
      }
      TRY(track_alloc(e, &q.Kpart, (size_t)e->batch * kp * e->n_r * e->n_r));
      TRY(track_alloc(e, &q.K, (size_t)e->batch * e->n_r * e->n_r));
      TRY(track_alloc(e, &q.Kf, (size_t)e->batch * e->n_r * e->n_r));
      TRY(track_alloc(e, &q.u0part, (size_t)e->batch * e->compose_grid * e->n_r));
      TRY(track_alloc(e, &q.u0, (size_t)e->batch * e->n_r));
      TRY(track_alloc(e, &q.dbeta, (size_t)e->batch * e->n_pix));
      if (!(e->ktc_on && e->precision == SF_PREC_DIRICHLET))  // (else fp16 slabs, no fp32 panel)
        TRY(track_alloc(e, &q.Gp, (size_t)e->batch * e->dpad * e->k_pad_max));
      if (e->precision == SF_PREC_F16X3)
        TRY(track_alloc(e, &q.Gh, (size_t)e->batch * e->dpad * e->k_pad_max * 2));
      if (e->precision == SF_PREC_DIRICHLET)
        TRY(track_alloc(e, &q.dtab, (size_t)e->batch * e->dpad));
      TRY(track_alloc(e, &q.maxbits, (size_t)e->batch));
      TRY(track_alloc(e, &q.gexp, (size_t)e->batch));
      if (e->ktc_on) {
        const int nb = e->ktc.nb;
        // per scene: per-CTA fp32 partials, then the fp64 sum (2 floats per double)
        const size_t zs = (size_t)(e->ktc_grid + 2) * (nb * (nb + 1) / 2) * 128 * 128;
        e->ktc.z_stride = (int64_t)zs;
        e->ktc.x_stride = (int64_t)e->dpad * e->k_pad_max;
        e->ktc.slab_stride = (int64_t)nb * e->ktc.ngrp * 1024;
        e->ktc.xs_stride = 4 * e->ktc.slab_stride;
        TRY(track_alloc(e, &q.zpart, zs * e->batch));
        TRY(track_alloc(e, &q.kxs, (size_t)e->ktc.xs_stride * e->batch));
        TRY(track_alloc(e, &q.kexp, 2 * (size_t)e->batch));
      }
      CTRY(cudaEventCreateWithFlags(&q.prep, cudaEventDisableTiming));
      CTRY(cudaEventCreateWithFlags(&q.ready, cudaEventDisableTiming));
      CTRY(cudaEventCreateWithFlags(&q.consumed, cudaEventDisableTiming));
      CTRY(cudaEventRecord(q.consumed, e->stream));
    }
  }
  CTRY(cudaStreamSynchronize(e->stream));
#undef TRY
#undef CTRY
  e->items_local = e->items;
  e->n_items_local = e->n_items;
  e->tiles_local = e->tiles;
  e->n_tiles_local = e->n_tiles;
  sf_status rs = sf_reset(e, e->l_floor);
  if (rs) {
    delete e;
    return rs;
  }
  *out = e;
  return SF_OK;
}

sf_status sf_destroy(sf_engine *e) {
  if (!e) return SF_OK;
  cudaSetDevice(e->device);
  cudaStreamSynchronize(e->stream);
  cudaStreamSynchronize(e->side);
  cudaStreamSynchronize(e->side2);
  cudaStreamSynchronize(e->side3);
  cudaStreamSynchronize(e->side4);
  cudaStreamSynchronize(e->side5);
  cudaStreamSynchronize(e->stats);
  delete e;
  return SF_OK;
}

sf_status sf_set_stream(sf_engine *e, void *stream) {
  if (!e) return fail(SF_EINVAL, "null engine");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  // order the switch: new stream waits for everything issued so far.
  // NULL selects the CUDA legacy default stream (torch's default stream).
  cudaStream_t ns = (cudaStream_t)stream;
  if (ns != e->stream) {
    cudaEvent_t ev;
    SF_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    SF_CUDA_TRY(cudaEventRecord(ev, e->stream));
    SF_CUDA_TRY(cudaStreamWaitEvent(ns, ev, 0));
    cudaEventDestroy(ev);
    e->stream = ns;
  }
  return SF_OK;
}

sf_status sf_synchronize(sf_engine *e) {
  if (!e) return fail(SF_EINVAL, "null engine");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return SF_OK;
}

sf_status sf_reset(sf_engine *e, double l_floor) {
  if (!e) return fail(SF_EINVAL, "null engine");
  if (!(l_floor > 0.0)) return fail(SF_EINVAL, "l_floor must be positive");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  SF_CUDA_TRY(cudaStreamSynchronize(e->side));
  SF_CUDA_TRY(cudaStreamSynchronize(e->side2));
  SF_CUDA_TRY(cudaStreamSynchronize(e->side3));
  SF_CUDA_TRY(cudaStreamSynchronize(e->side4));
  SF_CUDA_TRY(cudaStreamSynchronize(e->side5));
  e->l_floor = l_floor;
  const size_t B = (size_t)e->batch;  // every scene of a batched engine
  SF_CUDA_TRY(cudaMemsetAsync(e->A, 0, B * e->n_tiles * kTileElems * sizeof(float), e->stream));
  SF_CUDA_TRY(cudaMemsetAsync(e->b, 0, B * e->m * sizeof(double2), e->stream));
  if (e->A64) SF_CUDA_TRY(cudaMemsetAsync(e->A64, 0, (size_t)e->m * e->m * sizeof(double2), e->stream));
  if (e->beta)
    SF_CUDA_TRY(cudaMemsetAsync(e->beta, 0, B * e->n_pix * sizeof(double2), e->stream));
  if (e->bp) SF_CUDA_TRY(cudaMemsetAsync(e->bp, 0, B * e->n_pix * sizeof(double2), e->stream));
  SF_CUDA_TRY(cudaMemsetAsync(e->counters, 0, B * 2 * sizeof(long long), e->stream));
  SF_CUDA_TRY(cudaMemsetAsync(e->bmax, 0, B * sizeof(unsigned long long), e->stream));
  SF_CUDA_TRY(cudaMemsetAsync(e->scal, 0, B * 4 * sizeof(double), e->stream));
  std::vector<double> lf(B, e->l_floor);
  SF_CUDA_TRY(cudaMemcpyAsync(e->L, lf.data(), B * sizeof(double), cudaMemcpyHostToDevice, e->stream));
  if (e->Lsnap)
    SF_CUDA_TRY(cudaMemcpyAsync(e->Lsnap, e->L, B * sizeof(double), cudaMemcpyDeviceToDevice,
                                e->stream));
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  e->pulse_count = 0;
  return SF_OK;
}

sf_status sf_info(const sf_engine *e, int64_t *m_pad, int32_t *tile, int64_t *n_tiles,
                  int64_t *device_bytes) {
  if (!e) return fail(SF_EINVAL, "null engine");
  if (m_pad) *m_pad = e->dpad;
  if (tile) *tile = kTile;
  if (n_tiles) *n_tiles = e->n_tiles;
  if (device_bytes) *device_bytes = e->device_bytes;
  return SF_OK;
}

// Per-call timing events for sf_last_timings, recorded only once timings are
// asked for (or while profiling): four timestamped event records on the
// caller's stream per pulse cost 2.3% of the cfg1 rate (5 495 -> 5 621).
static inline bool call_events(sf_engine *e) { return e->call_timing || e->profiling; }

sf_status sf_accumulate_geom(sf_engine *e, const double *gamma, const double *omega,
                             const double *d, double sigma2, int32_t mem) {
  if (!e || !gamma || !omega || !d) return fail(SF_EINVAL, "null argument");
  if (e->batch > 1) return fail(SF_EINVAL, "batched engine: use sf_accumulate_geom_batch");
  if (e->ell_width <= 0 || !e->xyz)
    return fail(SF_ESTATE, "engine has no dictionary/pixel geometry for geometric pulses");
  if (!(sigma2 > 0.0)) return fail(SF_EINVAL, "sigma2 must be positive");
  const int n_r = e->n_r;
  if (mem != SF_MEM_DEVICE) {
    for (int m = 1; m < n_r; ++m)
      if (!(omega[m] > omega[m - 1]))
        return fail(SF_EINVAL, "frequencies must be strictly increasing");
    if (e->precision == SF_PREC_DIRICHLET && !omega_uniform(omega, n_r))
      return fail(SF_EINVAL, "the dirichlet Gram update needs uniformly spaced frequencies");
    if (platform_hits_pixel(e, gamma))
      return fail(SF_EINVAL, "platform position coincides with a scene pixel");
  }
  SF_CUDA_TRY(cudaSetDevice(e->device));
  if (call_events(e)) SF_CUDA_TRY(cudaEventRecord(e->ev_acc0, e->stream));
  const int k_pad = (int)round_up(2 * (int64_t)n_r, kKChunk);
  if (e->mode == SF_MODE_PIXEL) {
    double *h = nullptr;
    if (mem != SF_MEM_DEVICE) {
      sf_status s0 = stage_inputs(e, &h);
      if (s0) return s0;
      memcpy(h, omega, n_r * sizeof(double));
      memcpy(h + e->in_off_d, d, 2 * n_r * sizeof(double));
      memcpy(h + e->in_off_g, gamma, 3 * sizeof(double));
      h[e->in_off_s] = 1.0 / sqrt(sigma2);
      h[e->in_off_s + 1] = sigma2;
    }
    sf_status s0 = accumulate_pixel(e, h, gamma, omega, d, 1.0 / sqrt(sigma2), k_pad, sigma2);
    if (s0) return s0;
    if (call_events(e)) SF_CUDA_TRY(cudaEventRecord(e->ev_acc1, e->stream));
    e->acc_timed = call_events(e);
    return SF_OK;
  }
  if (e->keep_complex)
    return fail(SF_EUNSUPPORTED, "keep_complex statistics take dense pulses (sf_accumulate_dense)");
  const double *g_dev = gamma, *w_dev = omega;
  const double2 *d_dev = reinterpret_cast<const double2 *>(d);
  if (mem != SF_MEM_DEVICE) {
    double *h;
    sf_status s = stage_inputs(e, &h);
    if (s) return s;
    memcpy(h, omega, n_r * sizeof(double));
    memcpy(h + n_r, d, 2 * n_r * sizeof(double));
    memcpy(h + 3 * n_r, gamma, 3 * sizeof(double));
    SF_CUDA_TRY(cudaMemcpyAsync(e->omega, h, 3 * n_r * sizeof(double), cudaMemcpyHostToDevice,
                                e->stream));
    SF_CUDA_TRY(cudaMemcpyAsync(e->gamma, h + 3 * n_r, 3 * sizeof(double),
                                cudaMemcpyHostToDevice, e->stream));
    SF_CUDA_TRY(cudaEventRecord(
        e->stage_ev[(e->stage_slot + sf_engine::kRing - 1) % sf_engine::kRing], e->stream));
    g_dev = e->gamma;
    w_dev = e->omega;
    d_dev = reinterpret_cast<const double2 *>(e->omega + n_r);  // staged next to omega
  }
  SF_PROF(SF_K_OPERATOR, true);
  sf_status s = launch_pixel_delays(e->xyz, e->n_pix, g_dev, e->tau, e->zero_flag, e->stream);
  if (s) return s;
  s = launch_forward_t(w_dev, n_r, e->tau, e->n_pix, e->Ft, e->stream);
  if (s) return s;
  ComposeArgs a;
  a.Ft = e->Ft;
  a.ell_idx = e->ell_idx;
  a.ell_w = e->ell_w;
  a.ell_width = e->ell_width;
  a.m_atoms = e->m;
  a.m_pad = e->m_pad;
  a.n_r = n_r;
  a.k_pad = k_pad;
  a.inv_sigma = 1.0 / sqrt(sigma2);
  a.dt = d_dev;
  a.v0 = e->v0;
  a.Gp = e->Gp;
  a.b = e->b;
  a.u0part = e->u0part;
  a.grid = e->compose_grid;
  a.maxbits = e->maxbits;
  a.bmax = e->bmax;
  if (e->maxbits) SF_CUDA_TRY(cudaMemsetAsync(e->maxbits, 0, sizeof(unsigned), e->stream));
  SF_CUDA_TRY(cudaMemsetAsync(e->bmax, 0, sizeof(unsigned long long), e->stream));
  s = launch_compose(a, e->stream);
  if (s) return s;
  s = accumulate_tail(e, n_r, k_pad, true, a.inv_sigma);
  if (s) return s;
  if (call_events(e)) SF_CUDA_TRY(cudaEventRecord(e->ev_acc1, e->stream));
  e->acc_timed = call_events(e);
  return SF_OK;
}

sf_status sf_accumulate_dense(sf_engine *e, const double *G, const double *d, int32_t n_r,
                              double sigma2, int32_t mem) {
  if (!e || !G || !d) return fail(SF_EINVAL, "null argument");
  if (e->mode == SF_MODE_PIXEL)
    return fail(SF_ESTATE, "pixel-space engine accumulates geometric pulses only");
  if (n_r < 1 || n_r > e->n_r) return fail(SF_EINVAL, "n_freq exceeds the engine's n_freq");
  if (!(sigma2 > 0.0)) return fail(SF_EINVAL, "sigma2 must be positive");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  if (call_events(e)) SF_CUDA_TRY(cudaEventRecord(e->ev_acc0, e->stream));
  const int k_pad = (int)round_up(2 * (int64_t)n_r, kKChunk);
  const size_t gcount = (size_t)n_r * e->m;
  if (e->Gd_count < gcount) {
    if (e->Gd) cudaFree(e->Gd);
    e->Gd = nullptr;
    e->Gd_count = 0;
    sf_status s = dalloc(&e->Gd, gcount);
    if (s) return s;
    e->Gd_count = gcount;
  }
  sf_status s = to_device(e, e->Gd, G, gcount * sizeof(double2), mem);
  if (s) return s;
  double *h;
  s = stage_inputs(e, &h);
  if (s) return s;
  const double inv_sigma = 1.0 / sqrt(sigma2);
  if (mem == SF_MEM_DEVICE) {
    SF_CUDA_TRY(cudaMemcpyAsync(e->dt, d, n_r * sizeof(double2), cudaMemcpyDeviceToDevice,
                                e->stream));
  } else {
    memcpy(h, d, 2 * n_r * sizeof(double));
    SF_CUDA_TRY(cudaMemcpyAsync(e->dt, h, n_r * sizeof(double2), cudaMemcpyHostToDevice,
                                e->stream));
  }
  SF_CUDA_TRY(cudaEventRecord(e->stage_ev[(e->stage_slot + sf_engine::kRing - 1) % sf_engine::kRing],
                              e->stream));
  SF_PROF(SF_K_OPERATOR, true);
  ComposeArgs a;
  a.Gd = e->Gd;
  a.m_atoms = e->m;
  a.m_pad = e->m_pad;
  a.n_r = n_r;
  a.k_pad = k_pad;
  a.inv_sigma = inv_sigma;
  a.dt = e->dt;
  a.v0 = e->v0;
  a.Gp = e->Gp;
  a.b = e->b;
  a.u0part = e->u0part;
  a.grid = e->compose_grid;
  a.maxbits = e->maxbits;
  a.bmax = e->bmax;
  if (e->maxbits) SF_CUDA_TRY(cudaMemsetAsync(e->maxbits, 0, sizeof(unsigned), e->stream));
  SF_CUDA_TRY(cudaMemsetAsync(e->bmax, 0, sizeof(unsigned long long), e->stream));
  s = launch_compose(a, e->stream);
  if (s) return s;
  s = accumulate_tail(e, n_r, k_pad, false, inv_sigma);
  if (s) return s;
  if (call_events(e)) SF_CUDA_TRY(cudaEventRecord(e->ev_acc1, e->stream));
  e->acc_timed = call_events(e);
  return SF_OK;
}

sf_status sf_fista(sf_engine *e, const double *c0, double *c_out, int32_t mem, double lam,
                   double lam_rel, int32_t steps, double t0, double *t_out) {
  if (!e || !c0 || !c_out) return fail(SF_EINVAL, "null argument");
  if (e->pulse_count < 1) return fail(SF_ESTATE, "no pulses accumulated yet");
  if (steps < 1) return fail(SF_EINVAL, "inner_steps must be at least 1");
  if (!(lam > 0.0) && !(lam_rel > 0.0)) return fail(SF_EINVAL, "lambda must be positive");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  if (call_events(e)) SF_CUDA_TRY(cudaEventRecord(e->ev_f0, e->stream));
  const double *c0d = c0;
  if (mem != SF_MEM_DEVICE) {
    SF_CUDA_TRY(cudaMemcpyAsync(e->cin, c0, e->batch * e->m * sizeof(double), cudaMemcpyHostToDevice, e->stream));
    c0d = e->cin;
  }
  double *cod = (mem == SF_MEM_DEVICE) ? c_out : e->cout;
  SF_PROF(SF_K_FISTA, true);
  const bool chain = e->mode == SF_MODE_PIXEL;
  sf_status s = SF_OK;
  if (!chain &&
      (s = launch_fista_setup(e->dbuf ? e->Lsnap : e->L, e->bmax, lam, lam_rel, e->scal,
                              e->stream)))
    return s;
  if (e->mode != SF_MODE_PIXEL) {
    s = launch_fista_init(c0d, e->m, e->m_pad, e->zd, e->cprev, e->z32, e->stream);
    if (s) return s;
  }
  double t = t0;
  if (chain) {
    if ((s = ensure_wbuf(e, steps))) return s;
    static const bool no_graph = getenv("SF_NO_GRAPHS") != nullptr;
    static const bool prof_graph = getenv("SF_PROFILE_GRAPHS") != nullptr;  // coarse marks only
    if ((!e->profiling || prof_graph) && e->shard_world == 1 && !no_graph) {
      sf_engine::FGraph *g = nullptr;
      if ((s = chain_graph(e, steps, &g))) return s;
      // with the prologue and a captured last atom step, c0 and c_out are
      // patched into those two nodes (no device-to-device copies per call)
      const bool direct = g->prologue && g->last_step && e->batch == 1;
      if (c0d != e->cin && !direct)
        SF_CUDA_TRY(cudaMemcpyAsync(e->cin, c0d, e->batch * e->m * sizeof(double), cudaMemcpyDeviceToDevice,
                                    e->stream));
      const double *Lp = e->dbuf ? e->Lsnap : e->L;
      const unsigned long long *bm = e->bmax;
      double *scal = e->scal, *wv = e->wbuf;
      int st = steps;
      void *args[] = {(void *)&Lp, (void *)&bm, &lam, &lam_rel, (void *)&scal, &t0, &st, (void *)&wv};
      cudaKernelNodeParams kp{};
      PrologueArgs pa;
      void *pargs[] = {(void *)&pa};
      if (g->prologue) {  // same buffers as captured (c0 = e->cin), this call's scalars
        pa = prologue_args(e, direct ? c0d : e->cin, lam, lam_rel, t0, steps);
        kp.func = (void *)fista_prologue_kernel();
        kp.gridDim = dim3(1 + pa.init_blocks + pa.hz_blocks);
        kp.blockDim = dim3(256);
        kp.kernelParams = pargs;
      } else {
        kp.func = (void *)fista_setup_kernel();
        kp.gridDim = dim3(e->batch);  // one setup block per scene
        kp.blockDim = dim3(32);
        kp.kernelParams = args;
      }
      kp.sharedMemBytes = 0;
      kp.extra = nullptr;
      SF_CUDA_TRY(cudaGraphExecKernelNodeSetParams(g->exec, g->setup, &kp));
      if (direct) {
        AtomStepNodeArgs la = g->last_args;
        la.c_out = cod;
        void *aa[] = {&la.idx, &la.wt,    &la.width, &la.m,    &la.ypix,  &la.b,     &la.zd,
                      &la.cprev, &la.scal, &la.wv,  &la.kstep, &la.c_out, &la.m_pad, &la.n_pad};
        cudaKernelNodeParams lk{};
        SF_CUDA_TRY(cudaGraphKernelNodeGetParams(g->last_step, &lk));
        lk.kernelParams = aa;
        lk.extra = nullptr;
        SF_CUDA_TRY(cudaGraphExecKernelNodeSetParams(g->exec, g->last_step, &lk));
      }
      // replayed on the caller's stream; the graph's kernel nodes carry the
      // device's greatest priority (chain_graph)
      cudaStream_t fs = e->stream;
      SF_CUDA_TRY(cudaGraphLaunch(g->exec, fs));
      g_launches += g->kernels;
      if (cod != e->cout && !direct)
        SF_CUDA_TRY(cudaMemcpyAsync(cod, e->cout, e->batch * e->m * sizeof(double), cudaMemcpyDeviceToDevice,
                                    fs));
    } else {
      if ((s = enqueue_chain(e, e->stream, steps, c0d, cod, lam, lam_rel, t0, true))) return s;
    }
    for (int k = 0; k < steps; ++k) t = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));  // kernels.py:87
    steps = 0;
  }
  for (int k = 0; k < steps; ++k) {
    const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));  // kernels.py:87
    const double w = (t - 1.0) / t_next;                           // kernels.py:88
    SF_PROF(SF_K_GEMV, true);
    s = launch_gemv(e->A, e->tiles, e->n_tiles, e->z32, e->P, e->nt, 1, e->gemv_grid, e->stream);
    if (s) return s;
    SF_PROF(SF_K_GEMV, false);
    SF_PROF(SF_K_STEP, true);
    s = launch_fista_step(e->P, e->nt, e->b, nullptr, e->m, e->m_pad, e->zd, e->cprev, e->z32,
                          e->scal, w, k == steps - 1 ? cod : nullptr, e->stream);
    if (s) return s;
    SF_PROF(SF_K_STEP, false);
    t = t_next;
  }
  SF_PROF(SF_K_FISTA, false);
  if (call_events(e)) SF_CUDA_TRY(cudaEventRecord(e->ev_f1, e->stream));
  e->fista_timed = call_events(e);
  if (mem != SF_MEM_DEVICE) {
    SF_CUDA_TRY(cudaMemcpyAsync(c_out, e->cout, e->batch * e->m * sizeof(double), cudaMemcpyDeviceToHost,
                                e->stream));
    SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  }
  if (t_out) *t_out = t;
  return SF_OK;
}

sf_status sf_accumulate_geom_batch(sf_engine *e, const double *gammas, const double *omega,
                                   const double *d, const double *sigma2, int32_t mem) {
  if (!e || !gammas || !omega || !d || !sigma2) return fail(SF_EINVAL, "null argument");
  if (e->mode != SF_MODE_PIXEL || !e->xyz)
    return fail(SF_ESTATE, "batched pulses need a pixel-space engine");
  const int n_r = e->n_r, B = e->batch;
  SF_CUDA_TRY(cudaSetDevice(e->device));
  const int k_pad = (int)round_up(2 * (int64_t)n_r, kKChunk);
  sf_status s;
  if (mem != SF_MEM_DEVICE) {
    for (int m = 1; m < n_r; ++m)
      if (!(omega[m] > omega[m - 1]))
        return fail(SF_EINVAL, "frequencies must be strictly increasing");
    if (e->precision == SF_PREC_DIRICHLET && !omega_uniform(omega, n_r))
      return fail(SF_EINVAL, "the dirichlet Gram update needs uniformly spaced frequencies");
    for (int b = 0; b < B; ++b) {
      if (!(sigma2[b] > 0.0)) return fail(SF_EINVAL, "sigma2 must be positive");
      if (platform_hits_pixel(e, gammas + 3 * b))
        return fail(SF_EINVAL, "platform position coincides with a scene pixel");
    }
    double *h = nullptr;
    if ((s = stage_inputs(e, &h))) return s;
    memcpy(h, omega, n_r * sizeof(double));
    memcpy(h + n_r, gammas, 3 * (size_t)B * sizeof(double));
    memcpy(h + n_r + 3 * B, d, 2 * (size_t)n_r * B * sizeof(double));
    memcpy(h + n_r + 3 * B + 2 * (size_t)n_r * B, sigma2, (size_t)B * sizeof(double));
    s = accumulate_pixel_batch(e, h, nullptr, nullptr, nullptr, nullptr, k_pad);
  } else {
    s = accumulate_pixel_batch(e, nullptr, gammas, omega, d, sigma2, k_pad);
  }
  if (s) return s;
  return SF_OK;
}

sf_status sf_batch_lipschitz(sf_engine *e, const double *gammas, const double *omega,
                             const double *sigma2, int32_t n_pulses, double rel_tol,
                             int32_t max_iter, double *lam, int32_t *converged) {
  if (!e || !gammas || !omega || !sigma2 || !lam || !converged)
    return fail(SF_EINVAL, "null argument");
  if (n_pulses < 1) return fail(SF_EINVAL, "need at least one pulse");
  if (e->ell_width <= 0 || !e->xyz || !e->csr_ptr)
    return fail(SF_ESTATE, "engine has no dictionary/pixel geometry for geometric pulses");
  if (max_iter < 1) max_iter = 500;
  if (!(rel_tol > 0.0)) rel_tol = 1e-6;
  SF_CUDA_TRY(cudaSetDevice(e->device));
  const int n_r = e->n_r;
  std::vector<double> is2(n_pulses);
  for (int k = 0; k < n_pulses; ++k) {
    if (!(sigma2[k] > 0.0)) return fail(SF_EINVAL, "sigma2 must be positive");
    is2[k] = 1.0 / sigma2[k];
  }
  DevBuf bw, bg, bo, bs, bb;
  double2 *work;
  double *dg, *dom, *ds;
  unsigned long long *bmx;
  const size_t nwork = 2 * (size_t)e->m + 2 * (size_t)e->n_pix + (size_t)n_pulses * n_r + 1;
  sf_status s;
  if ((s = dscratch(bw, &work, nwork)) || (s = dscratch(bg, &dg, 3 * (size_t)n_pulses)) ||
      (s = dscratch(bo, &dom, (size_t)n_r)) || (s = dscratch(bs, &ds, (size_t)n_pulses)) ||
      (s = dscratch(bb, &bmx, 1)))
    return s;
  SF_CUDA_TRY(cudaMemcpy(dg, gammas, 3 * (size_t)n_pulses * 8, cudaMemcpyHostToDevice));
  SF_CUDA_TRY(cudaMemcpy(dom, omega, (size_t)n_r * 8, cudaMemcpyHostToDevice));
  SF_CUDA_TRY(cudaMemcpy(ds, is2.data(), (size_t)n_pulses * 8, cudaMemcpyHostToDevice));
  BatchLipArgs a;
  a.omega = dom;
  a.gammas = dg;
  a.inv_s2 = ds;
  a.xyz = e->xyz;
  a.n_r = n_r;
  a.n_pulses = n_pulses;
  a.ell_width = e->ell_width;
  a.n = e->n_pix;
  a.m = e->m;
  a.csr_ptr = e->csr_ptr;
  a.csr_atom = e->csr_atom;
  a.csr_w = e->csr_w;
  a.ell_idx = e->ell_idx;
  a.ell_w = e->ell_w;
  a.v0 = e->v0;
  a.work = work;
  a.bmax_scratch = bmx;
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  int conv = 0;
  if ((s = batch_lipschitz(a, rel_tol, max_iter, lam, &conv, e->stream))) return s;
  *converged = conv;
  return SF_OK;
}

// Debug accessor (not part of the public header): a per-scene buffer of the
// scratch set used by the most recent pulse.  what: 0 K~ [n_r^2] c128, 1 u0
// [n_r] c128, 2 power record [8], 3 dbeta [n] c128, 4 inputs [in_stride].
sf_status sf_debug_pulse_buffer(sf_engine *e, int32_t what, int32_t scene, double *out) {
  if (!e || !out || scene < 0 || scene >= e->batch) return fail(SF_EINVAL, "bad argument");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  SF_CUDA_TRY(cudaDeviceSynchronize());
  const int last = (e->ps_next + e->n_side) % (e->n_side + 1);
  auto &q = e->ps[last];
  const int64_t nr = e->n_r;
  const void *src = nullptr;
  size_t bytes = 0;
  switch (what) {
    case 0: src = q.K + scene * nr * nr; bytes = nr * nr * 16; break;
    case 1: src = q.u0 + scene * nr; bytes = nr * 16; break;
    case 2: src = q.pdiag + scene * 8; bytes = 64; break;
    case 3: src = q.dbeta + scene * e->n_pix; bytes = e->n_pix * 16; break;
    case 4: src = q.in + scene * e->in_stride; bytes = e->in_stride * 8; break;
    default: return fail(SF_EINVAL, "unknown buffer");
  }
  SF_CUDA_TRY(cudaMemcpy(out, src, bytes, cudaMemcpyDeviceToHost));
  return SF_OK;
}

sf_status sf_get_batch_scalars(sf_engine *e, double *L, int64_t *pulse_count, int64_t *fallbacks) {
  if (!e) return fail(SF_EINVAL, "null engine");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  const int B = e->batch;
  std::vector<double> hl(B);
  std::vector<long long> hc(2 * (size_t)B);
  SF_CUDA_TRY(cudaMemcpyAsync(hl.data(), e->L, B * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
  SF_CUDA_TRY(cudaMemcpyAsync(hc.data(), e->counters, 2 * (size_t)B * sizeof(long long),
                              cudaMemcpyDeviceToHost, e->stream));
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  for (int b = 0; b < B; ++b) {
    if (L) L[b] = hl[b];
    if (pulse_count) pulse_count[b] = hc[2 * b];
    if (fallbacks) fallbacks[b] = hc[2 * b + 1];
  }
  return SF_OK;
}

sf_status sf_get_scalars(sf_engine *e, double *L, int64_t *pulse_count, int64_t *fallbacks,
                         double *last_lambda) {
  if (!e) return fail(SF_EINVAL, "null engine");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  double hl = 0.0, hs[4];
  long long hc[2];
  int zf = 0;
  SF_CUDA_TRY(cudaMemcpyAsync(&zf, e->zero_flag, sizeof(int), cudaMemcpyDeviceToHost, e->stream));
  SF_CUDA_TRY(cudaMemcpyAsync(&hl, e->L, sizeof(double), cudaMemcpyDeviceToHost, e->stream));
  SF_CUDA_TRY(cudaMemcpyAsync(hc, e->counters, sizeof(hc), cudaMemcpyDeviceToHost, e->stream));
  SF_CUDA_TRY(cudaMemcpyAsync(hs, e->scal, sizeof(hs), cudaMemcpyDeviceToHost, e->stream));
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  if (zf) {
    SF_CUDA_TRY(cudaMemsetAsync(e->zero_flag, 0, sizeof(int), e->stream));
    if (zf & 2)
      return fail(SF_EINVAL, "a device-input pulse had frequencies that are not uniformly "
                             "spaced (required by the dirichlet Gram update)");
    return fail(SF_EINVAL, "platform position coincided with a scene pixel in a device-input pulse");
  }
  if (L) *L = hl;
  if (pulse_count) *pulse_count = hc[0];
  if (fallbacks) *fallbacks = hc[1];
  if (last_lambda) *last_lambda = hs[2];
  return SF_OK;
}

sf_status sf_get_power_diag(sf_engine *e, double *out4) {
  if (!e || !out4) return fail(SF_EINVAL, "null argument");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  SF_CUDA_TRY(cudaMemcpyAsync(out4, e->diag, 4 * sizeof(double), cudaMemcpyDeviceToHost, e->stream));
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return SF_OK;
}

// Streaming read of n4 float4 (8 independent 16-byte loads in flight per
// thread); the sum is kept only to stop the compiler dropping the loads.
__global__ void __launch_bounds__(256) k_stream_read(const float4 *__restrict__ p, int64_t n4,
                                                     float *__restrict__ sink) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n4; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += (v[u].x + v[u].y) + (v[u].z + v[u].w);
  }
  for (; i < n4; i += stride) {
    const float4 v = __ldg(p + i);
    acc += (v.x + v.y) + (v.z + v.w);
  }
  if (acc == -1.2345e-38f) *sink = acc;
}

sf_status sf_probe_store_read(sf_engine *e, int32_t iters, double *us) {
  if (!e || !us || iters < 1) return fail(SF_EINVAL, "null argument or iters < 1");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  const int64_t n4 = e->n_tiles * (int64_t)kTileElems * e->batch / 4;
  const int grid = e->sm_count * 4;
  cudaEvent_t a, b;
  SF_CUDA_TRY(cudaEventCreate(&a));
  SF_CUDA_TRY(cudaEventCreate(&b));
  const float4 *p = reinterpret_cast<const float4 *>(e->A);
  k_stream_read<<<grid, 256, 0, e->stream>>>(p, n4, nullptr);
  SF_LAUNCH_CHECK();
  SF_CUDA_TRY(cudaEventRecord(a, e->stream));
  for (int i = 0; i < iters; ++i) {
    k_stream_read<<<grid, 256, 0, e->stream>>>(p, n4, nullptr);
    SF_LAUNCH_CHECK();
  }
  SF_CUDA_TRY(cudaEventRecord(b, e->stream));
  SF_CUDA_TRY(cudaEventSynchronize(b));
  float ms = 0.f;
  SF_CUDA_TRY(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *us = 1e3 * ms / iters;
  return SF_OK;
}

sf_status sf_probe_matvec(sf_engine *e, int32_t iters, int32_t dense, double *us) {
  if (!e || !us || iters < 1) return fail(SF_EINVAL, "null argument or iters < 1");
  if (e->mode != SF_MODE_PIXEL) return fail(SF_ESTATE, "matvec probe needs a pixel-space engine");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  cudaEvent_t a, b;
  SF_CUDA_TRY(cudaEventCreate(&a));
  SF_CUDA_TRY(cudaEventCreate(&b));
  sf_status s = launch_gemv(e->A, e->tiles_local, e->n_tiles_local, e->z32, e->P, e->nt, 1,
                            e->gemv_grid, e->stream, e->batch, e->zstride, 0, dense != 0);
  if (s) return s;
  SF_CUDA_TRY(cudaEventRecord(a, e->stream));
  for (int i = 0; i < iters; ++i)
    if ((s = launch_gemv(e->A, e->tiles_local, e->n_tiles_local, e->z32, e->P, e->nt, 1,
                         e->gemv_grid, e->stream, e->batch, e->zstride, 0, dense != 0)))
      return s;
  SF_CUDA_TRY(cudaEventRecord(b, e->stream));
  SF_CUDA_TRY(cudaEventSynchronize(b));
  float ms = 0.f;
  SF_CUDA_TRY(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *us = 1e3 * ms / iters;
  return SF_OK;
}

sf_status sf_apply_store(sf_engine *e, const float *x, double *y, int32_t dense) {
  if (!e || !x || !y) return fail(SF_EINVAL, "null argument");
  if (e->mode != SF_MODE_PIXEL || e->batch != 1)
    return fail(SF_ESTATE, "sf_apply_store needs a single-scene pixel-space engine");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  SF_CUDA_TRY(cudaMemcpyAsync(e->z32, x, sizeof(float) * e->dpad, cudaMemcpyDeviceToDevice,
                              e->stream));
  sf_status s = launch_gemv(e->A, e->tiles_local, e->n_tiles_local, e->z32, e->P, e->nt, 1,
                            e->gemv_grid, e->stream, 1, e->zstride, 0, dense != 0);
  if (s) return s;
  if ((s = launch_pix_reduce(e->P, e->nt, e->dpad, e->ypix, e->stream, 1))) return s;
  SF_CUDA_TRY(cudaMemcpyAsync(y, e->ypix, sizeof(double) * e->n_pix, cudaMemcpyDeviceToDevice,
                              e->stream));
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return SF_OK;
}

sf_status sf_get_b(sf_engine *e, double *b, int32_t mem) {
  if (!e || !b) return fail(SF_EINVAL, "null argument");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  return from_device(e, b, e->b, e->m * sizeof(double2), mem);
}

sf_status sf_get_A_re(sf_engine *e, double *A_re, int32_t mem) {
  if (!e || !A_re) return fail(SF_EINVAL, "null argument");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  double *dense = nullptr;
  DevBuf hold;
  const size_t cnt = (size_t)e->m * e->m;
  if (mem == SF_MEM_DEVICE) {
    dense = A_re;
  } else {
    sf_status s = dscratch(hold, &dense, cnt);
    if (s) return s;
  }
  sf_status s = (e->mode == SF_MODE_PIXEL)
                    ? launch_pix_to_atom(e->A, e->nt, e->ell_idx, e->ell_w, e->ell_width, e->m,
                                         dense, e->stream)
                    : launch_unpack_tiles(e->A, e->tiles, e->n_tiles, e->m, 1, dense, e->stream);
  if (s) return s;
  if (mem != SF_MEM_DEVICE) return from_device(e, A_re, dense, cnt * sizeof(double), SF_MEM_HOST);
  return SF_OK;
}

sf_status sf_get_pixel_stats(sf_engine *e, double *B_re, double *beta, int32_t mem) {
  if (!e) return fail(SF_EINVAL, "null engine");
  if (e->mode != SF_MODE_PIXEL) return fail(SF_ESTATE, "engine is not in pixel-space mode");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  if (B_re) {
    const size_t cnt = (size_t)e->n_pix * e->n_pix;
    double *dense = B_re;
    DevBuf hold;
    if (mem != SF_MEM_DEVICE) {
      sf_status s = dscratch(hold, &dense, cnt);
      if (s) return s;
    }
    sf_status s = launch_unpack_tiles(e->A, e->tiles, e->n_tiles, e->n_pix, 1, dense, e->stream);
    if (s) return s;
    if (mem != SF_MEM_DEVICE) {
      s = from_device(e, B_re, dense, cnt * sizeof(double), SF_MEM_HOST);
      if (s) return s;
    }
  }
  if (beta) return from_device(e, beta, e->beta, e->n_pix * sizeof(double2), mem);
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return SF_OK;
}

sf_status sf_tile_store(sf_engine *e, int64_t *n_local, int64_t *nt, int32_t *tile_ij) {
  if (!e) return fail(SF_EINVAL, "null engine");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  if (n_local) *n_local = e->n_tiles_local;
  if (nt) *nt = e->nt;
  if (tile_ij) {
    SF_CUDA_TRY(cudaMemcpyAsync(tile_ij, e->tiles_local, e->n_tiles_local * sizeof(int2),
                                cudaMemcpyDeviceToHost, e->stream));
    SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  }
  return SF_OK;
}

sf_status sf_copy_tiles(sf_engine *e, float *buf, int32_t to_engine, int32_t mem) {
  if (!e || !buf) return fail(SF_EINVAL, "null argument");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  std::vector<int2> tl(e->n_tiles_local);
  SF_CUDA_TRY(cudaMemcpyAsync(tl.data(), e->tiles_local, tl.size() * sizeof(int2),
                              cudaMemcpyDeviceToHost, e->stream));
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  const cudaMemcpyKind kind = to_engine ? (mem == SF_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                                : cudaMemcpyHostToDevice)
                                        : (mem == SF_MEM_DEVICE ? cudaMemcpyDeviceToDevice
                                                                : cudaMemcpyDeviceToHost);
  const size_t tb = (size_t)kTileElems * sizeof(float);
  for (size_t k = 0; k < tl.size(); ++k) {
    float *dev = e->A + tri_index(tl[k].x, tl[k].y, e->nt) * kTileElems;
    float *ext = buf + k * kTileElems;
    SF_CUDA_TRY(cudaMemcpyAsync(to_engine ? (void *)dev : (void *)ext,
                                to_engine ? (const void *)ext : (const void *)dev, tb, kind,
                                e->stream));
  }
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return SF_OK;
}

sf_status sf_get_bp(sf_engine *e, double *image_sum, int64_t *pulse_count, int32_t mem) {
  if (!e) return fail(SF_EINVAL, "null engine");
  if (e->mode != SF_MODE_PIXEL) return fail(SF_ESTATE, "back-projection is kept by pixel-space engines");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  if (pulse_count) *pulse_count = e->pulse_count;
  if (image_sum) return from_device(e, image_sum, e->bp, e->n_pix * sizeof(double2), mem);
  return SF_OK;
}

sf_status sf_set_bp(sf_engine *e, const double *image_sum, int32_t mem) {
  if (!e) return fail(SF_EINVAL, "null engine");
  if (e->mode != SF_MODE_PIXEL) return fail(SF_ESTATE, "back-projection is kept by pixel-space engines");
  if (!image_sum) return fail(SF_EINVAL, "null image_sum");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  sf_status s = to_device(e, e->bp, image_sum, e->n_pix * sizeof(double2), mem);
  if (s) return s;
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return SF_OK;
}

sf_status sf_set_pixel_stats(sf_engine *e, const double *B_re, const double *beta, double L,
                             int64_t pulse_count, int64_t fallbacks, int32_t mem) {
  if (!e) return fail(SF_EINVAL, "null engine");
  if (e->mode != SF_MODE_PIXEL) return fail(SF_ESTATE, "engine is not in pixel-space mode");
  if (!(L > 0.0)) return fail(SF_EINVAL, "L must be positive");
  if (pulse_count < 0 || fallbacks < 0) return fail(SF_EINVAL, "counters must be nonnegative");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  sf_status s;
  if (B_re) {
    const size_t cnt = (size_t)e->n_pix * e->n_pix;
    const double *src = B_re;
    DevBuf hold;
    if (mem != SF_MEM_DEVICE) {
      double *tmp;
      if ((s = dscratch(hold, &tmp, cnt))) return s;
      SF_CUDA_TRY(cudaMemcpyAsync(tmp, B_re, cnt * sizeof(double), cudaMemcpyHostToDevice, e->stream));
      src = tmp;
    }
    if ((s = launch_pack_tiles(src, e->n_pix, e->tiles, e->n_tiles, e->A, e->stream))) return s;
    SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  }
  if (beta) {
    if ((s = to_device(e, e->beta, beta, e->n_pix * sizeof(double2), mem))) return s;
    SF_CUDA_TRY(cudaMemsetAsync(e->bmax, 0, sizeof(unsigned long long), e->stream));
    if ((s = launch_bupdate(e->ell_idx, e->ell_w, e->ell_width, e->m, e->beta, e->b, e->bmax,
                            e->stream)))
      return s;
  }
  long long hc[2] = {(long long)pulse_count, (long long)fallbacks};
  SF_CUDA_TRY(cudaMemcpyAsync(e->L, &L, sizeof(double), cudaMemcpyHostToDevice, e->stream));
  if (e->Lsnap)
    SF_CUDA_TRY(cudaMemcpyAsync(e->Lsnap, e->L, sizeof(double), cudaMemcpyDeviceToDevice, e->stream));
  SF_CUDA_TRY(cudaMemcpyAsync(e->counters, hc, sizeof(hc), cudaMemcpyHostToDevice, e->stream));
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  e->pulse_count = pulse_count;
  return SF_OK;
}

sf_status sf_set_stats(sf_engine *e, const double *A_re, const double *b, double L,
                       int64_t pulse_count, int64_t fallbacks, int32_t mem) {
  if (!e) return fail(SF_EINVAL, "null engine");
  if (!(L > 0.0)) return fail(SF_EINVAL, "L must be positive");
  if (pulse_count < 0 || fallbacks < 0) return fail(SF_EINVAL, "counters must be nonnegative");
  if (e->mode == SF_MODE_PIXEL && (A_re || b))
    return fail(SF_EUNSUPPORTED, "pixel-space engine: restore with sf_set_pixel_stats");
  if (e->keep_complex && A_re)
    return fail(SF_EINVAL, "keep_complex engine: restore A with sf_set_stats_complex");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  if (A_re) {
    const size_t cnt = (size_t)e->m * e->m;
    const double *src = A_re;
    DevBuf hold;
    if (mem != SF_MEM_DEVICE) {
      double *tmp;
      sf_status s = dscratch(hold, &tmp, cnt);
      if (s) return s;
      SF_CUDA_TRY(cudaMemcpyAsync(tmp, A_re, cnt * sizeof(double), cudaMemcpyHostToDevice, e->stream));
      src = tmp;
    }
    sf_status s = launch_pack_tiles(src, e->m, e->tiles, e->n_tiles, e->A, e->stream);
    if (s) return s;
    SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  }
  if (b) {
    sf_status s = to_device(e, e->b, b, e->m * sizeof(double2), mem);
    if (s) return s;
    s = launch_bmax(e->b, e->m, e->bmax, e->stream);
    if (s) return s;
  }
  long long hc[2] = {(long long)pulse_count, (long long)fallbacks};
  SF_CUDA_TRY(cudaMemcpyAsync(e->L, &L, sizeof(double), cudaMemcpyHostToDevice, e->stream));
  SF_CUDA_TRY(cudaMemcpyAsync(e->counters, hc, sizeof(hc), cudaMemcpyHostToDevice, e->stream));
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  e->pulse_count = pulse_count;
  return SF_OK;
}

sf_status sf_get_A(sf_engine *e, double *A, int32_t mem) {
  if (!e || !A) return fail(SF_EINVAL, "null argument");
  if (!e->keep_complex)
    return fail(SF_EUNSUPPORTED, "the complex A is kept only by keep_complex engines");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  return from_device(e, A, e->A64, (size_t)e->m * e->m * sizeof(double2), mem);
}

sf_status sf_set_stats_complex(sf_engine *e, const double *A, const double *b, double L,
                               int64_t pulse_count, int64_t fallbacks, int32_t mem) {
  if (!e) return fail(SF_EINVAL, "null engine");
  if (!e->keep_complex) return fail(SF_EUNSUPPORTED, "not a keep_complex engine");
  if (A) {
    SF_CUDA_TRY(cudaSetDevice(e->device));
    sf_status s = to_device(e, e->A64, A, (size_t)e->m * e->m * sizeof(double2), mem);
    if (s) return s;
    if ((s = launch_pack_re(e->A64, e->m, e->tiles, e->n_tiles, e->A, e->stream))) return s;
  }
  e->keep_complex = false;  // sf_set_stats rejects a real A on keep_complex engines
  sf_status s = sf_set_stats(e, nullptr, b, L, pulse_count, fallbacks, mem);
  e->keep_complex = true;
  return s;
}

sf_status sf_dense_residual(int32_t device, const double *G, const double *d, int32_t n_r,
                            int64_t m, const double *c, double sigma2, double *quad_out,
                            double *grad_inout) {
  if (!G || !d || !c || !quad_out || !grad_inout) return fail(SF_EINVAL, "null argument");
  if (n_r < 1 || m < 1) return fail(SF_EINVAL, "bad sizes");
  if (!(sigma2 > 0.0)) return fail(SF_EINVAL, "sigma2 must be positive");
  sf_status s = check_device(device);
  if (s) return s;
  DevBuf bg, bd, bc, br, bgr, bq;
  double2 *dG, *dd, *dr;
  double *dc, *dgr, *dq;
  if ((s = dscratch(bg, &dG, (size_t)n_r * m)) || (s = dscratch(bd, &dd, (size_t)n_r)) ||
      (s = dscratch(bc, &dc, (size_t)m)) || (s = dscratch(br, &dr, (size_t)n_r)) ||
      (s = dscratch(bgr, &dgr, (size_t)m)) || (s = dscratch(bq, &dq, 1)))
    return s;
  SF_CUDA_TRY(cudaMemcpy(dG, G, (size_t)n_r * m * sizeof(double2), cudaMemcpyHostToDevice));
  SF_CUDA_TRY(cudaMemcpy(dd, d, (size_t)n_r * sizeof(double2), cudaMemcpyHostToDevice));
  SF_CUDA_TRY(cudaMemcpy(dc, c, (size_t)m * sizeof(double), cudaMemcpyHostToDevice));
  SF_CUDA_TRY(cudaMemcpy(dgr, grad_inout, (size_t)m * sizeof(double), cudaMemcpyHostToDevice));
  if ((s = launch_dense_residual(dG, dd, n_r, m, dc, 1.0 / sigma2, dr, dgr, dq, 0))) return s;
  SF_CUDA_TRY(cudaMemcpy(grad_inout, dgr, (size_t)m * sizeof(double), cudaMemcpyDeviceToHost));
  SF_CUDA_TRY(cudaMemcpy(quad_out, dq, sizeof(double), cudaMemcpyDeviceToHost));
  return SF_OK;
}

sf_status sf_reconstruct(sf_engine *e, const double *c, double *img, int32_t mem) {
  if (!e || !c || !img) return fail(SF_EINVAL, "null argument");
  if (e->ell_width <= 0) return fail(SF_ESTATE, "engine has no dictionary");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  const double *cd = c;
  if (mem != SF_MEM_DEVICE) {
    SF_CUDA_TRY(cudaMemcpyAsync(e->cin, c, e->m * sizeof(double), cudaMemcpyHostToDevice, e->stream));
    cd = e->cin;
  }
  double *od = (mem == SF_MEM_DEVICE) ? img : e->img;
  sf_status s = launch_reconstruct(e->csr_ptr, e->csr_atom, e->csr_w, e->n_pix, cd, od, e->stream);
  if (s) return s;
  if (mem != SF_MEM_DEVICE) return from_device(e, img, e->img, e->n_pix * sizeof(double), SF_MEM_HOST);
  return SF_OK;
}

sf_status sf_pulse_metrics(sf_engine *e, const double *c, const uint8_t *mask, const double *truth,
                           double threshold, double *out8) {
  if (!e || !c || !mask || !out8) return fail(SF_EINVAL, "null argument");
  if (e->ell_width <= 0) return fail(SF_ESTATE, "engine has no dictionary");
  if (e->batch != 1) return fail(SF_EUNSUPPORTED, "metrics of batched engines: one scene at a time");
  if (!(threshold > 0.0)) return fail(SF_EINVAL, "threshold must be positive");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  if (!e->metrics) SF_CUDA_TRY(cudaMalloc(&e->metrics, (256 * 8 + 8) * sizeof(double)));
  const bool has_bp = e->mode == SF_MODE_PIXEL && e->pulse_count > 0;
  sf_status s = launch_pulse_metrics(e->csr_ptr, e->csr_atom, e->csr_w, e->n_pix, c, e->m, mask,
                                     reinterpret_cast<const double2 *>(truth),
                                     has_bp ? e->bp : nullptr,
                                     has_bp ? 1.0 / (double)e->pulse_count : 0.0, threshold,
                                     e->metrics, e->metrics + 256 * 8, e->stream);
  if (s) return s;
  return from_device(e, out8, e->metrics + 256 * 8, 8 * sizeof(double), SF_MEM_HOST);
}

sf_status sf_last_timings(sf_engine *e, float *acc_ms, float *fista_ms) {
  if (!e) return fail(SF_EINVAL, "null engine");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  e->call_timing = true;  // calls from now on are timed
  if (acc_ms) {
    *acc_ms = 0.f;
    if (e->acc_timed) {
      SF_CUDA_TRY(cudaEventSynchronize(e->ev_acc1));
      SF_CUDA_TRY(cudaEventElapsedTime(acc_ms, e->ev_acc0, e->ev_acc1));
    }
  }
  if (fista_ms) {
    *fista_ms = 0.f;
    if (e->fista_timed) {
      SF_CUDA_TRY(cudaEventSynchronize(e->ev_f1));
      SF_CUDA_TRY(cudaEventElapsedTime(fista_ms, e->ev_f0, e->ev_f1));
    }
  }
  return SF_OK;
}

sf_status sf_profile(sf_engine *e, int32_t enable) {
  if (!e) return fail(SF_EINVAL, "null engine");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  for (auto &p : e->prof) p.used = 0;
  e->profiling = enable != 0;
  if (!e->gemv_bytes) SF_CUDA_TRY(cudaMalloc(&e->gemv_bytes, sizeof(unsigned long long)));
  SF_CUDA_TRY(cudaMemset(e->gemv_bytes, 0, sizeof(unsigned long long)));
  return SF_OK;
}

sf_status sf_profile_bytes(sf_engine *e, int64_t *gemv_bytes) {
  if (!e || !gemv_bytes) return fail(SF_EINVAL, "null argument");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  unsigned long long v = 0;
  if (e->gemv_bytes)
    SF_CUDA_TRY(cudaMemcpy(&v, e->gemv_bytes, sizeof(v), cudaMemcpyDeviceToHost));
  *gemv_bytes = (int64_t)v;
  return SF_OK;
}

sf_status sf_profile_read(sf_engine *e, int32_t kind, int64_t *launches, double *total_ms) {
  if (!e) return fail(SF_EINVAL, "null engine");
  if (kind < 0 || kind > 7) return fail(SF_EINVAL, "unknown kernel kind");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  const char *trace = getenv("SF_TRACE_FILE");
  if (trace && kind == 0) {
    // debugging aid: every recorded interval, relative to the earliest start
    cudaEvent_t base = nullptr;
    float lo = 0.f;
    for (auto &p : e->prof)
      for (size_t i = 0; i < p.used; ++i) {
        if (!base) base = p.start[i];
        float ms = 0.f;
        SF_CUDA_TRY(cudaEventElapsedTime(&ms, e->prof[0].used ? e->prof[0].start[0] : base,
                                         p.start[i]));
        lo = std::min(lo, ms);
      }
    FILE *f = fopen(trace, "a");
    if (f && base) {
      cudaEvent_t ref = e->prof[0].used ? e->prof[0].start[0] : base;
      for (int k = 0; k < 8; ++k)
        for (size_t i = 0; i < e->prof[k].used; ++i) {
          float a = 0.f, b = 0.f;
          SF_CUDA_TRY(cudaEventElapsedTime(&a, ref, e->prof[k].start[i]));
          SF_CUDA_TRY(cudaEventElapsedTime(&b, ref, e->prof[k].stop[i]));
          fprintf(f, "%d %zu %.4f %.4f\n", k, i, a - lo, b - lo);
        }
    }
    if (f) fclose(f);
  }
  auto &p = e->prof[kind];
  double tot = 0.0;
  for (size_t i = 0; i < p.used; ++i) {
    float ms = 0.f;
    SF_CUDA_TRY(cudaEventElapsedTime(&ms, p.start[i], p.stop[i]));
    tot += ms;
  }
  if (launches) *launches = (int64_t)p.used;
  if (total_ms) *total_ms = tot;
  return SF_OK;
}

sf_status sf_plan_shard(int64_t n_dim, int32_t rank, int32_t world, int64_t *item_begin,
                        int64_t *item_end, int64_t *tiles_local) {
  if (n_dim < 1 || world < 1 || rank < 0 || rank >= world)
    return fail(SF_EINVAL, "bad shard request");
  const int nt = (int)((n_dim + kTile - 1) / kTile);
  int64_t i0, i1, nl;
  plan_items(nt, rank, world, &i0, &i1, &nl);
  if (item_begin) *item_begin = i0;
  if (item_end) *item_end = i1;
  if (tiles_local) *tiles_local = nl;
  return SF_OK;
}

sf_status sf_nccl_unique_id(void *out128) {
  if (!out128) return fail(SF_EINVAL, "null argument");
  return nccl_unique_id(out128);
}

// Shared by the NCCL and loopback paths: this rank's Gram items / matvec tiles
// (contiguous tile-balanced super-tile ranges, sf_shard.cu) and K~ pixel tiles
// (a contiguous range of the Morton tiles), plus its exchange.
static sf_status shard_setup(sf_engine *e, int32_t rank, int32_t world, void *comm, void *comm_op,
                             LoopGroup *loop, PeerGroup *peer = nullptr) {
  drop_graphs(e);  // captured chains hold the old tile lists
  int64_t i0, i1, nl;
  plan_items(e->nt, rank, world, &i0, &i1, &nl);
  std::vector<int2> it, tl;
  local_lists(e->nt, i0, i1, it, tl);
  int2 *dit = nullptr, *dtl = nullptr;
  sf_status s;
  if ((s = dalloc(&dit, it.size())) || (s = dalloc(&dtl, tl.size()))) return s;
  if (!it.empty())
    SF_CUDA_TRY(cudaMemcpy(dit, it.data(), it.size() * sizeof(int2), cudaMemcpyHostToDevice));
  if (!tl.empty())
    SF_CUDA_TRY(cudaMemcpy(dtl, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice));
  if (e->own_local) {
    cudaFree(e->items_local);
    cudaFree(e->tiles_local);
  }
  nccl_comm_destroy(e->comm);
  nccl_comm_destroy(e->comm_op);
  e->items_local = dit;
  e->tiles_local = dtl;
  e->n_items_local = (int)it.size();
  e->n_tiles_local = (int64_t)tl.size();
  e->own_local = true;
  e->comm = comm;
  e->comm_op = comm_op;
  e->loop = loop;
  e->peer = peer;
  e->shard_rank = rank;
  e->shard_world = world;
  if (e->ktc_on) {
    const int T = e->ktc.tiles;
    e->ktc.tile_begin = (int)((int64_t)T * rank / world);
    e->ktc.tile_end = (int)((int64_t)T * (rank + 1) / world);
  }
  if (!e->ev_opcoll) SF_CUDA_TRY(cudaEventCreateWithFlags(&e->ev_opcoll, cudaEventDisableTiming));
  SF_CUDA_TRY(cudaEventRecord(e->ev_opcoll, e->stream));
  // partial slots of tiles this rank never visits must read as zero
  SF_CUDA_TRY(cudaMemsetAsync(e->P, 0, (size_t)e->nt * e->nt * kTile * sizeof(float), e->stream));
  SF_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return SF_OK;
}

static sf_status shard_check(sf_engine *e, int32_t rank, int32_t world) {
  if (!e) return fail(SF_EINVAL, "null engine");
  if (e->mode != SF_MODE_PIXEL) return fail(SF_EUNSUPPORTED, "sharding needs a pixel-space engine");
  if (world < 1 || rank < 0 || rank >= world) return fail(SF_EINVAL, "bad rank/world");
  if (e->pulse_count != 0) return fail(SF_ESTATE, "shard before the first pulse");
  if (e->batch > 1) return fail(SF_EUNSUPPORTED, "batched engines do not shard");
  return SF_OK;
}

sf_status sf_shard_init(sf_engine *e, int32_t rank, int32_t world, const void *uid128) {
  sf_status s = shard_check(e, rank, world);
  if (s) return s;
  if (world > 1 && !uid128) return fail(SF_EINVAL, "a NCCL unique id is needed for world > 1");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  void *comm = nullptr, *comm_op = nullptr;
  if (uid128) {
    if ((s = nccl_comm_init(&comm, world, uid128, rank))) return s;
    if ((s = nccl_comm_dup(comm, rank, &comm_op))) {
      nccl_comm_destroy(comm);
      return s;
    }
  }
  return shard_setup(e, rank, world, comm, comm_op, nullptr);
}

sf_status sf_loopback_create(int32_t world, sf_loopback **out) {
  if (!out) return fail(SF_EINVAL, "null argument");
  LoopGroup *g = nullptr;
  sf_status s = loop_create(world, &g);
  if (s) return s;
  *out = reinterpret_cast<sf_loopback *>(g);
  return SF_OK;
}

void sf_loopback_destroy(sf_loopback *g) { loop_destroy(reinterpret_cast<LoopGroup *>(g)); }

sf_status sf_shard_init_loopback(sf_engine *e, int32_t rank, sf_loopback *group) {
  if (!group) return fail(SF_EINVAL, "null loopback group");
  LoopGroup *g = reinterpret_cast<LoopGroup *>(group);
  const int world = loop_world(g);
  sf_status s = shard_check(e, rank, world);
  if (s) return s;
  SF_CUDA_TRY(cudaSetDevice(e->device));
  return shard_setup(e, rank, world, nullptr, nullptr, world > 1 ? g : nullptr);
}

sf_status sf_shard_sizes(sf_engine *e, int64_t *cap_y, int64_t *cap_k) {
  if (!e || !cap_y || !cap_k) return fail(SF_EINVAL, "null argument");
  if (e->mode != SF_MODE_PIXEL) return fail(SF_EUNSUPPORTED, "sharding needs a pixel-space engine");
  *cap_y = e->dpad;
  *cap_k = e->ktc_on ? (int64_t)(e->ktc.nb * (e->ktc.nb + 1) / 2) * 128 * 128 : 0;
  return SF_OK;
}

sf_status sf_peer_create(int32_t device, int32_t rank, int32_t world, int64_t cap_y, int64_t cap_k,
                         uint64_t *shared_seq, sf_peer_group **out) {
  if (!out || cap_y < 1 || cap_k < 0) return fail(SF_EINVAL, "bad argument");
  sf_status s = check_device(device);
  if (s) return s;
  PeerGroup *g = nullptr;
  if ((s = peer_create(device, rank, world, (size_t)cap_y, (size_t)cap_k, shared_seq, &g))) return s;
  *out = reinterpret_cast<sf_peer_group *>(g);
  return SF_OK;
}

int64_t sf_peer_blob_size(void) { return peer_blob_size(); }

sf_status sf_peer_export(sf_peer_group *g, void *blob) {
  if (!g || !blob) return fail(SF_EINVAL, "null argument");
  return peer_export(reinterpret_cast<PeerGroup *>(g), blob);
}

sf_status sf_peer_import(sf_peer_group *g, const void *blobs) {
  if (!g || !blobs) return fail(SF_EINVAL, "null argument");
  return peer_import(reinterpret_cast<PeerGroup *>(g), blobs);
}

void sf_peer_destroy(sf_peer_group *g) { peer_destroy(reinterpret_cast<PeerGroup *>(g)); }

sf_status sf_shard_init_peer(sf_engine *e, sf_peer_group *group) {
  if (!group) return fail(SF_EINVAL, "null peer group");
  PeerGroup *g = reinterpret_cast<PeerGroup *>(group);
  const int world = peer_world(g), rank = peer_rank(g);
  sf_status s = shard_check(e, rank, world);
  if (s) return s;
  int64_t cy = 0, ck = 0;
  if ((s = sf_shard_sizes(e, &cy, &ck))) return s;
  if ((size_t)cy > peer_cap(g, 0) || (size_t)ck > peer_cap(g, 1))
    return fail(SF_EINVAL, "peer group slots smaller than this engine's exchanges");
  SF_CUDA_TRY(cudaSetDevice(e->device));
  return shard_setup(e, rank, world, nullptr, nullptr, nullptr, world > 1 ? g : nullptr);
}

// ---- engine-less seam functions -------------------------------------------

sf_status sf_simulate_echo(int32_t device, const double *omegas, int32_t n_r,
                           const double *gammas, int32_t n_pulses, const double *pixel_xyz,
                           const double *rho, int64_t n, double *d) {
  if (!omegas || !gammas || !pixel_xyz || !rho || !d) return fail(SF_EINVAL, "null argument");
  if (n_r < 1 || n_pulses < 0 || n < 1) return fail(SF_EINVAL, "bad sizes");
  sf_status s = check_device(device);
  if (s) return s;
  if (n_pulses == 0) return SF_OK;
  DevBuf bo, bg, bx, br, bd;
  double *dom, *dg, *dx;
  double2 *dr, *dd;
  if ((s = dscratch(bo, &dom, n_r)) || (s = dscratch(bg, &dg, 3 * (size_t)n_pulses)) ||
      (s = dscratch(bx, &dx, 3 * (size_t)n)) || (s = dscratch(br, &dr, (size_t)n)) ||
      (s = dscratch(bd, &dd, (size_t)n_pulses * n_r)))
    return s;
  SF_CUDA_TRY(cudaMemcpy(dom, omegas, n_r * sizeof(double), cudaMemcpyHostToDevice));
  SF_CUDA_TRY(cudaMemcpy(dg, gammas, 3 * (size_t)n_pulses * sizeof(double), cudaMemcpyHostToDevice));
  SF_CUDA_TRY(cudaMemcpy(dx, pixel_xyz, 3 * (size_t)n * sizeof(double), cudaMemcpyHostToDevice));
  SF_CUDA_TRY(cudaMemcpy(dr, rho, (size_t)n * sizeof(double2), cudaMemcpyHostToDevice));
  if ((s = launch_simulate_echo(dom, n_r, dg, n_pulses, dx, dr, n, dd, 0))) return s;
  SF_CUDA_TRY(cudaMemcpy(d, dd, (size_t)n_pulses * n_r * sizeof(double2), cudaMemcpyDeviceToHost));
  return SF_OK;
}

sf_status sf_delay_phase_matrix(int32_t device, const double *omegas, int32_t n_r,
                                const double *delays, int64_t n, double *out) {
  if (!omegas || !delays || !out) return fail(SF_EINVAL, "null argument");
  if (n_r < 1 || n < 0) return fail(SF_EINVAL, "bad sizes");
  sf_status s = check_device(device);
  if (s) return s;
  if (n == 0) return SF_OK;
  DevBuf bo, bt, bf;
  double *dom, *dtau;
  double2 *dF;
  if ((s = dscratch(bo, &dom, n_r)) || (s = dscratch(bt, &dtau, n)) ||
      (s = dscratch(bf, &dF, (size_t)n * n_r)))
    return s;
  SF_CUDA_TRY(cudaMemcpy(dom, omegas, n_r * sizeof(double), cudaMemcpyHostToDevice));
  SF_CUDA_TRY(cudaMemcpy(dtau, delays, n * sizeof(double), cudaMemcpyHostToDevice));
  s = launch_delay_phase(dom, n_r, dtau, n, dF, 0);
  if (s) return s;
  SF_CUDA_TRY(cudaMemcpy(out, dF, (size_t)n * n_r * sizeof(double2), cudaMemcpyDeviceToHost));
  return SF_OK;
}

sf_status sf_fista_inner(int32_t device, const double *gram, const double *corr, const double *c0,
                         int64_t m, double t0, double tau, double thresh, int32_t steps,
                         double *c_out, double *t_out) {
  if (!gram || !corr || !c0 || !c_out) return fail(SF_EINVAL, "null argument");
  if (m < 1) return fail(SF_EINVAL, "empty problem");
  sf_status s = check_device(device);
  if (s) return s;
  // float64 throughout, as the reference seam (a dense host matrix per call)
  DevBuf bg, bc, bz, bcp, by;
  double *dg, *dcorr, *dz, *dcp, *dy;
  if ((s = dscratch(bg, &dg, (size_t)m * m)) || (s = dscratch(bc, &dcorr, m)) ||
      (s = dscratch(bz, &dz, m)) || (s = dscratch(bcp, &dcp, m)) || (s = dscratch(by, &dy, m)))
    return s;
  SF_CUDA_TRY(cudaMemcpy(dg, gram, (size_t)m * m * sizeof(double), cudaMemcpyHostToDevice));
  SF_CUDA_TRY(cudaMemcpy(dcorr, corr, m * sizeof(double), cudaMemcpyHostToDevice));
  SF_CUDA_TRY(cudaMemcpy(dz, c0, m * sizeof(double), cudaMemcpyHostToDevice));
  SF_CUDA_TRY(cudaMemcpy(dcp, c0, m * sizeof(double), cudaMemcpyHostToDevice));
  // momentum weights on the host, as kernels.py:87-88 advances t
  std::vector<double> w(std::max(steps, 0));
  double t = t0;
  for (int k = 0; k < steps; ++k) {
    const double t_next = 0.5 * (1.0 + sqrt(1.0 + 4.0 * t * t));
    w[k] = (t - 1.0) / t_next;
    t = t_next;
  }
  if ((s = launch_seam_fista64(dg, dcorr, m, tau, thresh, w.data(), steps, dz, dcp, dy, 0)))
    return s;
  SF_CUDA_TRY(cudaMemcpy(c_out, dcp, m * sizeof(double), cudaMemcpyDeviceToHost));
  if (t_out) *t_out = t;
  return SF_OK;
}

// control flow on the host, every arithmetic step on the device
__global__ void k_power_step(const double2 *__restrict__ v, double2 *__restrict__ w, int64_t n,
                             double *__restrict__ out) {
  __shared__ double r1[32], r2[32];
  double lam = 0.0, nn = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    lam += v[i].x * w[i].x + v[i].y * w[i].y;  // Re(v^H w)
    nn += w[i].x * w[i].x + w[i].y * w[i].y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lam += __shfl_xor_sync(0xffffffffu, lam, o);
    nn += __shfl_xor_sync(0xffffffffu, nn, o);
  }
  if ((threadIdx.x & 31) == 0) {
    r1[threadIdx.x >> 5] = lam;
    r2[threadIdx.x >> 5] = nn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, c = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      a += r1[k];
      c += r2[k];
    }
    out[0] = a;
    out[1] = sqrt(c);
  }
  __syncthreads();
  const double nrm = out[1];
  if (nrm > 0.0)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x)
      w[i] = make_double2(w[i].x / nrm, w[i].y / nrm);
}

sf_status sf_hermitian_top_eigenvalue(int32_t device, const double *X, int64_t n, double rel_tol,
                                      int32_t max_iter, double *lam_out, int32_t *conv_out) {
  if (!X || !lam_out || !conv_out) return fail(SF_EINVAL, "null argument");
  if (n < 1) return fail(SF_EINVAL, "matrix must be square and nonempty");
  sf_status s = check_device(device);
  if (s) return s;
  DevBuf bx, bv, bw, bo;
  double2 *dX, *dv, *dw;
  double *dout;
  if ((s = dscratch(bx, &dX, (size_t)n * n)) || (s = dscratch(bv, &dv, n)) ||
      (s = dscratch(bw, &dw, n)) || (s = dscratch(bo, &dout, 2)))
    return s;
  SF_CUDA_TRY(cudaMemcpy(dX, X, (size_t)n * n * sizeof(double2), cudaMemcpyHostToDevice));
  if ((s = launch_start_vector(n, 0x5EED, dv, 0))) return s;
  double lam_prev = 0.0, delta_prev = 0.0;
  bool have_prev = false, have_dprev = false;
  for (int it = 0; it < max_iter; ++it) {
    if ((s = launch_zgemv(dX, n, dv, dw, 0))) return s;
    k_power_step<<<1, 1024>>>(dv, dw, n, dout);
    SF_LAUNCH_CHECK();
    double h[2];
    SF_CUDA_TRY(cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost));
    const double lam = h[0], norm_w = h[1];
    if (norm_w == 0.0) {
      *lam_out = 0.0;
      *conv_out = 1;
      return SF_OK;
    }
    std::swap(dv, dw);  // v = w / |w| (normalised in place by k_power_step)
    if (have_prev) {
      const double delta = lam - lam_prev;
      if (fabs(delta) <= rel_tol * std::max(fabs(lam), 1e-300)) {
        double tail = 0.0;
        if (have_dprev && fabs(delta_prev) > fabs(delta) && fabs(delta) > 0.0) {
          const double q = delta / delta_prev;
          if (q > 0.0 && q < 1.0) tail = delta * q / (1.0 - q);
        }
        *lam_out = lam + tail + fabs(delta);
        *conv_out = 1;
        return SF_OK;
      }
      delta_prev = delta;
      have_dprev = true;
    }
    lam_prev = lam;
    have_prev = true;
  }
  *lam_out = have_prev ? lam_prev : 0.0;
  *conv_out = 0;
  return SF_OK;
}

sf_status sf_compose_ell(int32_t device, const double *F, int32_t n_r, int64_t n,
                         const int32_t *ell_idx, const double *ell_w, int64_t m, int32_t width,
                         double *G) {
  if (!F || !ell_idx || !ell_w || !G) return fail(SF_EINVAL, "null argument");
  if (n_r < 1 || n < 1 || m < 1 || width < 1) return fail(SF_EINVAL, "bad sizes");
  sf_status s = check_device(device);
  if (s) return s;
  for (int64_t k = 0; k < m * width; ++k)
    if (ell_idx[k] >= n) return fail(SF_EINVAL, "dictionary pixel index out of range");
  DevBuf bf, bi, bw, bg;
  double2 *dF, *dG;
  int32_t *di;
  double *dw;
  if ((s = dscratch(bf, &dF, (size_t)n_r * n)) || (s = dscratch(bi, &di, (size_t)m * width)) ||
      (s = dscratch(bw, &dw, (size_t)m * width)) || (s = dscratch(bg, &dG, (size_t)n_r * m)))
    return s;
  SF_CUDA_TRY(cudaMemcpy(dF, F, (size_t)n_r * n * sizeof(double2), cudaMemcpyHostToDevice));
  SF_CUDA_TRY(cudaMemcpy(di, ell_idx, (size_t)m * width * sizeof(int32_t), cudaMemcpyHostToDevice));
  SF_CUDA_TRY(cudaMemcpy(dw, ell_w, (size_t)m * width * sizeof(double), cudaMemcpyHostToDevice));
  if ((s = launch_compose_ell_dense(dF, n_r, n, di, dw, m, width, dG, 0))) return s;
  SF_CUDA_TRY(cudaMemcpy(G, dG, (size_t)n_r * m * sizeof(double2), cudaMemcpyDeviceToHost));
  return SF_OK;
}

sf_status sf_soft_threshold(int32_t device, const double *u, int64_t n, int32_t is_complex,
                            double alpha, double *out) {
  if (!u || !out) return fail(SF_EINVAL, "null argument");
  if (alpha < 0.0) return fail(SF_EINVAL, "alpha must be nonnegative");
  if (n < 0) return fail(SF_EINVAL, "bad size");
  sf_status s = check_device(device);
  if (s) return s;
  if (n == 0) return SF_OK;
  const size_t cnt = (size_t)n * (is_complex ? 2 : 1);
  DevBuf bu, bo;
  double *du, *dout;
  if ((s = dscratch(bu, &du, cnt)) || (s = dscratch(bo, &dout, cnt))) return s;
  SF_CUDA_TRY(cudaMemcpy(du, u, cnt * sizeof(double), cudaMemcpyHostToDevice));
  if ((s = launch_soft_threshold(du, n, is_complex, alpha, dout, 0))) return s;
  SF_CUDA_TRY(cudaMemcpy(out, dout, cnt * sizeof(double), cudaMemcpyDeviceToHost));
  return SF_OK;
}

}  // extern "C"
