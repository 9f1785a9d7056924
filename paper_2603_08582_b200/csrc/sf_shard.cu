// sf_shard.cu -- one scene's pixel-space statistics sharded over several GPUs.
//
// Work partition: the 2x2 super-tiles of the stored triangle (the Gram
// kernel's work items, row-major) are split into contiguous ranges with equal
// tile counts; a rank owns the tiles inside its items, runs the Gram update and
// the FISTA matvec on those only, and the per-step partial y_pix (N fp64 values)
// is summed across ranks with one NCCL all-reduce.  Everything else per pulse
// (F, K~, power iteration, beta/b, the element-wise FISTA step, H z) is small
// and computed redundantly and identically on every rank -- no other exchange.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, the copy torch already
// loaded when present), so the library has no link-time NCCL dependency.
#include <dlfcn.h>
#include <string.h>

#include <chrono>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "sf_common.cuh"
#include "sf_kernels.cuh"

namespace sf {

// ---- the planner (host only; also exported for CPU tests) --------------------
static void super_items(int nt, std::vector<int2> &items) {
  const int ns = (nt + 1) / 2;
  for (int a = 0; a < ns; ++a)
    for (int b = a; b < ns; ++b) items.push_back(make_int2(a, b));
}

// tiles (I,J) of a super-tile item with the Gram kernel's validity rules
static int item_tiles(int2 it, int nt, int2 *out) {
  int n = 0;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) {
      const int I = 2 * it.x + a, J = 2 * it.y + b;
      if (I >= nt || J >= nt) continue;
      if (it.x == it.y && a == 1 && b == 0) continue;
      out[n++] = make_int2(I, J);
    }
  return n;
}

void plan_items(int nt, int rank, int world, int64_t *i0, int64_t *i1, int64_t *ntiles) {
  std::vector<int2> items;
  super_items(nt, items);
  int64_t total = 0;
  std::vector<int64_t> cum(items.size() + 1, 0);
  int2 tmp[4];
  for (size_t k = 0; k < items.size(); ++k) cum[k + 1] = cum[k] + item_tiles(items[k], nt, tmp);
  total = cum.back();
  // rank r takes the items whose first tile lies in [r T / W, (r+1) T / W)
  auto bound = [&](int r) {
    const int64_t target = (total * r + world - 1) / world;
    size_t k = 0;
    while (k < items.size() && cum[k] < target) ++k;
    return (int64_t)k;
  };
  *i0 = bound(rank);
  *i1 = bound(rank + 1);
  *ntiles = cum[*i1] - cum[*i0];
}

void local_lists(int nt, int64_t i0, int64_t i1, std::vector<int2> &items_out,
                 std::vector<int2> &tiles_out) {
  std::vector<int2> items;
  super_items(nt, items);
  int2 tmp[4];
  for (int64_t k = i0; k < i1; ++k) {
    items_out.push_back(items[k]);
    const int n = item_tiles(items[k], nt, tmp);
    for (int q = 0; q < n; ++q) tiles_out.push_back(tmp[q]);
  }
}

// ---- NCCL through dlopen --------------------------------------------------------
struct NcclApi {
  void *h = nullptr;
  int (*get_unique_id)(void *) = nullptr;
  int (*all_reduce)(const void *, void *, size_t, int, int, void *, cudaStream_t) = nullptr;
  int (*comm_destroy)(void *) = nullptr;
  int (*comm_split)(void *, int, int, void **, void *) = nullptr;
  const char *(*error_string)(int) = nullptr;
};

struct UniqueId {
  char internal[128];
};
typedef int (*comm_init_rank_fn)(void **, int, UniqueId, int);

static NcclApi g_nccl;
static comm_init_rank_fn g_comm_init = nullptr;

sf_status nccl_load() {
  if (g_nccl.h) return SF_OK;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return fail(SF_ENCCL, std::string("libnccl.so.2 not found: ") + dlerror());
  g_nccl.get_unique_id = (int (*)(void *))dlsym(h, "ncclGetUniqueId");
  g_comm_init = (comm_init_rank_fn)dlsym(h, "ncclCommInitRank");
  g_nccl.all_reduce = (int (*)(const void *, void *, size_t, int, int, void *, cudaStream_t))dlsym(
      h, "ncclAllReduce");
  g_nccl.comm_destroy = (int (*)(void *))dlsym(h, "ncclCommDestroy");
  g_nccl.error_string = (const char *(*)(int))dlsym(h, "ncclGetErrorString");
  g_nccl.comm_split = (int (*)(void *, int, int, void **, void *))dlsym(h, "ncclCommSplit");
  if (!g_nccl.get_unique_id || !g_comm_init || !g_nccl.all_reduce || !g_nccl.comm_destroy)
    return fail(SF_ENCCL, "libnccl.so.2 lacks the expected symbols");
  g_nccl.h = h;
  return SF_OK;
}

static sf_status nccl_check(int r, const char *what) {
  if (r == 0) return SF_OK;
  const char *msg = g_nccl.error_string ? g_nccl.error_string(r) : "";
  return fail(SF_ENCCL, std::string(what) + ": " + msg);
}

sf_status nccl_unique_id(void *out128) {
  sf_status s = nccl_load();
  if (s) return s;
  return nccl_check(g_nccl.get_unique_id(out128), "ncclGetUniqueId");
}

sf_status nccl_comm_init(void **comm, int world, const void *uid128, int rank) {
  sf_status s = nccl_load();
  if (s) return s;
  UniqueId id;
  memcpy(id.internal, uid128, 128);
  return nccl_check(g_comm_init(comm, world, id, rank), "ncclCommInitRank");
}

sf_status nccl_allreduce_f64(double *buf, size_t count, void *comm, cudaStream_t st) {
  // ncclFloat64 = 8, ncclSum = 0 (nccl.h)
  return nccl_check(g_nccl.all_reduce(buf, buf, count, 8, 0, comm, st), "ncclAllReduce");
}

void nccl_comm_destroy(void *comm) {
  if (comm && g_nccl.comm_destroy) g_nccl.comm_destroy(comm);
}

// A second communicator over the same ranks (the operator phase's K~ partials
// travel on their own communicator, never interleaved with the FISTA chain's).
sf_status nccl_comm_dup(void *comm, int rank, void **out) {
  sf_status s = nccl_load();
  if (s) return s;
  if (!g_nccl.comm_split) return fail(SF_ENCCL, "libnccl.so.2 lacks ncclCommSplit");
  return nccl_check(g_nccl.comm_split(comm, 0, rank, out, nullptr), "ncclCommSplit");
}

// ---- in-process loopback group: emulated ranks on one device ---------------------
// The ranks are engines of one process (each driven by its own host thread, in
// lockstep).  An exchange copies the rank's buffer into its slot, records an
// event, meets the other ranks at a host barrier (so every slot's event is
// recorded before anyone waits on it), makes its stream wait on all ranks'
// events and sums the slots in rank order.  No kernel ever waits on another:
// the dependencies are stream-event edges on work already enqueued.  Slots and
// events alternate between two parities, and a second barrier keeps a rank from
// re-recording a parity before every rank has enqueued its waits on it.
constexpr int kLoopMaxRanks = 16;
struct LoopGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived[kLoopChannels] = {};
  uint64_t gen[kLoopChannels] = {};
  double *slots[kLoopChannels][2] = {};
  size_t cap[kLoopChannels] = {};
  cudaEvent_t ev[kLoopChannels][2][kLoopMaxRanks] = {};
  uint64_t step[kLoopChannels][kLoopMaxRanks] = {};
};

sf_status loop_create(int world, LoopGroup **out) {
  if (world < 1 || world > kLoopMaxRanks) return fail(SF_EINVAL, "loopback world out of range");
  LoopGroup *g = new LoopGroup;
  g->world = world;
  for (int c = 0; c < kLoopChannels; ++c)
    for (int p = 0; p < 2; ++p)
      for (int r = 0; r < world; ++r)
        if (cudaEventCreateWithFlags(&g->ev[c][p][r], cudaEventDisableTiming) != cudaSuccess) {
          loop_destroy(g);
          return fail(SF_ECUDA, "loopback: event creation failed");
        }
  *out = g;
  return SF_OK;
}

void loop_destroy(LoopGroup *g) {
  if (!g) return;
  for (int c = 0; c < kLoopChannels; ++c) {
    for (int p = 0; p < 2; ++p) {
      if (g->slots[c][p]) cudaFree(g->slots[c][p]);
      for (int r = 0; r < kLoopMaxRanks; ++r)
        if (g->ev[c][p][r]) cudaEventDestroy(g->ev[c][p][r]);
    }
  }
  delete g;
}

int loop_world(const LoopGroup *g) { return g ? g->world : 1; }

static sf_status loop_barrier(LoopGroup *g, int ch) {
  std::unique_lock<std::mutex> lk(g->mu);
  const uint64_t my = g->gen[ch];
  if (++g->arrived[ch] == g->world) {
    g->arrived[ch] = 0;
    ++g->gen[ch];
    g->cv.notify_all();
    return SF_OK;
  }
  if (!g->cv.wait_for(lk, std::chrono::seconds(120), [&] { return g->gen[ch] != my; }))
    return fail(SF_ESTATE, "loopback: a rank did not reach the exchange (ranks must run in lockstep)");
  return SF_OK;
}

__global__ void k_sum_slots(const double *__restrict__ slots, int world, size_t stride, size_t n,
                            double *__restrict__ out) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int r = 0; r < world; ++r) s += slots[r * stride + i];
  out[i] = s;
}

sf_status loop_allreduce_f64(LoopGroup *g, int ch, int rank, double *buf, size_t n,
                             cudaStream_t st) {
  {
    std::lock_guard<std::mutex> lk(g->mu);
    if (!g->slots[ch][0]) {
      for (int p = 0; p < 2; ++p)
        SF_CUDA_TRY(cudaMalloc(&g->slots[ch][p], (size_t)g->world * n * sizeof(double)));
      g->cap[ch] = n;
    } else if (n > g->cap[ch]) {
      return fail(SF_EINVAL, "loopback: exchange larger than the channel's first one");
    }
  }
  const int par = (int)(g->step[ch][rank]++ & 1);
  double *slots = g->slots[ch][par];
  SF_CUDA_TRY(cudaMemcpyAsync(slots + (size_t)rank * g->cap[ch], buf, n * sizeof(double),
                              cudaMemcpyDeviceToDevice, st));
  SF_CUDA_TRY(cudaEventRecord(g->ev[ch][par][rank], st));
  sf_status s = loop_barrier(g, ch);
  if (s) return s;
  for (int r = 0; r < g->world; ++r) SF_CUDA_TRY(cudaStreamWaitEvent(st, g->ev[ch][par][r], 0));
  k_sum_slots<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(slots, g->world, g->cap[ch], n, buf);
  SF_LAUNCH_CHECK();
  return loop_barrier(g, ch);
}

// ---- peer-memory group: ranks = processes of one node, one GPU each -----------
// The exchange of the multi-GPU engine without a collective library: every rank
// owns, per channel and parity, a slot array of `world` buffers in its device
// memory and maps every other rank's array (CUDA IPC; NVLink peer access
// between GPUs).  An all-reduce is
//   push   the rank's partial stored straight into slot [rank] of EVERY rank's
//          array (one kernel, the stores cross NVLink; for the FISTA chain the
//          slot reduction k_pix_reduce is the pushing kernel, see
//          launch_pix_reduce),
//   edge   an interprocess event recorded behind the push; the ranks' host
//          threads meet at a sequence counter in shared host memory (so a wait
//          is enqueued only after the matching record), then every stream
//          waits on every rank's event,
//   sum    the slots added in rank order (k_sum_slots): every rank forms the
//          same bits.
// No kernel spins on another rank's progress: the dependencies are event edges
// on enqueued work, as in the loopback group, so two ranks may even share one
// device (how the path is tested on a one-GPU box).  Parities alternate per
// exchange; a rank re-records a parity only after every rank published the
// next sequence number, i.e. after their waits on the old record are enqueued,
// and re-pushes into a slot only behind its own previous sum, which waited on
// the owner's later record -- itself behind the owner's sum of that slot.
struct PeerBlob {
  cudaIpcMemHandle_t mem[kLoopChannels][2];
  cudaIpcEventHandle_t ev[kLoopChannels][2];
};
struct PeerGroup {
  int world = 1, rank = 0, device = 0;
  volatile uint64_t *seq = nullptr;  // shared host memory [kLoopChannels][kPeerMaxRanks]
  size_t cap[kLoopChannels] = {};
  double *local[kLoopChannels][2] = {};
  PeerSlots peer[kLoopChannels][2];
  cudaEvent_t ev[kLoopChannels][2][kPeerMaxRanks] = {};
  uint64_t step[kLoopChannels] = {};
  bool imported = false;
};

int64_t peer_blob_size() { return (int64_t)sizeof(PeerBlob); }
int peer_world(const PeerGroup *g) { return g ? g->world : 1; }
int peer_rank(const PeerGroup *g) { return g ? g->rank : 0; }
size_t peer_cap(const PeerGroup *g, int ch) { return g->cap[ch]; }

void peer_destroy(PeerGroup *g) {
  if (!g) return;
  cudaSetDevice(g->device);
  for (int c = 0; c < kLoopChannels; ++c)
    for (int p = 0; p < 2; ++p) {
      for (int r = 0; r < g->world; ++r) {
        if (r != g->rank && g->peer[c][p].p[r]) cudaIpcCloseMemHandle(g->peer[c][p].p[r]);
        if (g->ev[c][p][r]) cudaEventDestroy(g->ev[c][p][r]);
      }
      if (g->local[c][p]) cudaFree(g->local[c][p]);
    }
  delete g;
}

sf_status peer_create(int device, int rank, int world, size_t cap_y, size_t cap_k,
                      uint64_t *shared_seq, PeerGroup **out) {
  if (world < 1 || world > kPeerMaxRanks || rank < 0 || rank >= world)
    return fail(SF_EINVAL, "peer group: bad rank/world");
  if (!shared_seq) return fail(SF_EINVAL, "peer group: null shared sequence array");
  SF_CUDA_TRY(cudaSetDevice(device));
  PeerGroup *g = new PeerGroup;
  g->world = world;
  g->rank = rank;
  g->device = device;
  g->seq = shared_seq;
  g->cap[0] = cap_y;
  g->cap[1] = cap_k > 0 ? cap_k : 1;
  for (int c = 0; c < kLoopChannels; ++c)
    for (int p = 0; p < 2; ++p) {
      const size_t bytes = (size_t)world * g->cap[c] * sizeof(double);
      if (cudaMalloc(&g->local[c][p], bytes) != cudaSuccess ||
          cudaMemset(g->local[c][p], 0, bytes) != cudaSuccess ||
          cudaEventCreateWithFlags(&g->ev[c][p][rank],
                                   cudaEventDisableTiming | cudaEventInterprocess) != cudaSuccess) {
        peer_destroy(g);
        return fail(SF_ECUDA, "peer group: slot / event creation failed");
      }
      g->peer[c][p].p[rank] = g->local[c][p];
      g->peer[c][p].world = world;
    }
  SF_CUDA_TRY(cudaDeviceSynchronize());
  *out = g;
  return SF_OK;
}

sf_status peer_export(PeerGroup *g, void *blob) {
  PeerBlob b;
  memset(&b, 0, sizeof(b));
  SF_CUDA_TRY(cudaSetDevice(g->device));
  for (int c = 0; c < kLoopChannels; ++c)
    for (int p = 0; p < 2; ++p) {
      SF_CUDA_TRY(cudaIpcGetMemHandle(&b.mem[c][p], g->local[c][p]));
      SF_CUDA_TRY(cudaIpcGetEventHandle(&b.ev[c][p], g->ev[c][p][g->rank]));
    }
  memcpy(blob, &b, sizeof(b));
  return SF_OK;
}

sf_status peer_import(PeerGroup *g, const void *blobs) {
  if (g->imported) return fail(SF_ESTATE, "peer group: handles already imported");
  SF_CUDA_TRY(cudaSetDevice(g->device));
  const PeerBlob *b = static_cast<const PeerBlob *>(blobs);
  for (int r = 0; r < g->world; ++r) {
    if (r == g->rank) continue;
    for (int c = 0; c < kLoopChannels; ++c)
      for (int p = 0; p < 2; ++p) {
        void *ptr = nullptr;
        SF_CUDA_TRY(cudaIpcOpenMemHandle(&ptr, b[r].mem[c][p], cudaIpcMemLazyEnablePeerAccess));
        g->peer[c][p].p[r] = static_cast<double *>(ptr);
        SF_CUDA_TRY(cudaIpcOpenEventHandle(&g->ev[c][p][r], b[r].ev[c][p]));
      }
  }
  g->imported = true;
  return SF_OK;
}

__global__ void k_push_slots(const double *__restrict__ src, PeerSlots dst, size_t off, size_t n) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double v = src[i];
  for (int r = 0; r < dst.world; ++r) dst.p[r][off + i] = v;
}

// the slot arrays this rank pushes exchange `step` of channel ch into
PeerSlots peer_targets(PeerGroup *g, int ch, size_t *offset) {
  *offset = (size_t)g->rank * g->cap[ch];
  return g->peer[ch][(int)(g->step[ch] & 1)];
}

// Everything of an exchange behind the push: event edge, host rendezvous, sum
// into `out` (n values).  `pushed`: the caller's kernel already stored the
// partial into the slots of peer_targets(); else `buf` is pushed here.
sf_status peer_allreduce_f64(PeerGroup *g, int ch, double *buf, size_t n, cudaStream_t st,
                             bool pushed) {
  if (!g->imported && g->world > 1) return fail(SF_ESTATE, "peer group: handles not imported");
  if (n > g->cap[ch]) return fail(SF_EINVAL, "peer group: exchange larger than the channel");
  const uint64_t step = g->step[ch];
  const int par = (int)(step & 1);
  if (!pushed) {
    k_push_slots<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(buf, g->peer[ch][par],
                                                             (size_t)g->rank * g->cap[ch], n);
    SF_LAUNCH_CHECK();
  }
  SF_CUDA_TRY(cudaEventRecord(g->ev[ch][par][g->rank], st));
  volatile uint64_t *seq = g->seq + (size_t)ch * kPeerMaxRanks;
  __atomic_store_n(const_cast<uint64_t *>(&seq[g->rank]), step + 1, __ATOMIC_RELEASE);
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < g->world; ++r) {
    unsigned spins = 0;
    while (__atomic_load_n(const_cast<uint64_t *>(&seq[r]), __ATOMIC_ACQUIRE) < step + 1) {
      if ((++spins & 0xfff) == 0 &&
          std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120))
        return fail(SF_ESTATE, "peer group: a rank did not reach the exchange (ranks must run in lockstep)");
    }
  }
  for (int r = 0; r < g->world; ++r) SF_CUDA_TRY(cudaStreamWaitEvent(st, g->ev[ch][par][r], 0));
  k_sum_slots<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g->local[ch][par], g->world, g->cap[ch],
                                                          n, buf);
  SF_LAUNCH_CHECK();
  g->step[ch] = step + 1;
  return SF_OK;
}

}  // namespace sf
