// sf_kernels.cuh -- launcher declarations shared by the engine translation units.
#pragma once

#include <cuda_fp16.h>

#include <vector>

#include "sf_common.cuh"

namespace sf {

struct ComposeArgs {
  const double2 *Ft = nullptr;      // [N][N_r] forward operator (transposed)
  const int32_t *ell_idx = nullptr; // [M][ell_width] (nullptr: dense mode)
  const double *ell_w = nullptr;
  int ell_width = 0;
  const double2 *Gd = nullptr;      // dense mode: [N_r][M]
  int64_t m_atoms = 0, m_pad = 0;
  int n_r = 0, k_pad = 0;
  double inv_sigma = 1.0;
  const double2 *dt = nullptr;      // raw d [N_r] (scaled by inv_sigma in-kernel)
  const double2 *v0 = nullptr;      // power-iteration start vector [M]
  float *Gp = nullptr;              // packed operator [m_pad][k_pad]
  double2 *b = nullptr;             // running b [M]
  double2 *u0part = nullptr;        // [grid][N_r]
  unsigned *maxbits = nullptr;      // max |G~| as float bits (f16x3 scaling), may be null
  unsigned long long *bmax = nullptr;  // max_j |b_j| as fp64 bits, may be null
  int grid = 0;
};

// k_forward_pix writing the tensor-core K~ build's X operand directly (scaled
// fp16 hi/lo Morton-group slabs, see sf_ktc.cu) instead of the fp32 panel Gp
struct FwdSlabs {
  __half *xs = nullptr;  // per scene: Xh | Xl | ...; nullptr = write Gp as before
  int64_t xs_stride = 0, slab_stride = 0, ngrp = 0;
  const int32_t *grp_pix = nullptr;  // [8 * ngrp] pixel of each Morton slot, or -1
  int *exps = nullptr;               // per scene {ex, ey}
  float qrow_max = 0.f;
  int nb = 0;
};
struct PixelForwardArgs {
  const double *omega = nullptr;  // [N_r]
  int n_r = 0;
  const double *tau = nullptr;    // [N]
  int64_t n = 0, n_pad = 0;
  int k_pad = 0;
  double inv_sigma = 1.0;
  const double *sig = nullptr;    // device {1/sigma, sigma^2}; overrides inv_sigma
  const double2 *d = nullptr;     // raw d [N_r]
  const double2 *hv0 = nullptr;   // H v0 [N]
  double2 *Ft = nullptr;          // [N][N_r]
  float *Gp = nullptr;            // packed [n_pad][k_pad]
  double2 *dbeta = nullptr;       // [N] this pulse's F~^H d~
  double2 *u0part = nullptr;      // [grid][N_r]
  unsigned *maxbits = nullptr;
  int grid = 0;
  int batch = 1;                  // scenes (grid rows); inputs at sc * in_stride doubles
  int64_t in_stride = 0;
  FwdSlabs slabs;
};

// sf_pixel.cu
sf_status launch_stage_batch(const double *raw, int n_r, int B, int64_t off_d, int64_t off_g,
                             int64_t off_s, int64_t stride, double *in, cudaStream_t st);
sf_status launch_forward_pix(const PixelForwardArgs &a, cudaStream_t st);
sf_status launch_fold(const double2 *dbeta, double2 *beta, int64_t n, const double *pdiag,
                      double *L, long long *counters, double *diag, double sigma2, double2 *bp,
                      cudaStream_t st, const double *sig = nullptr, int batch = 1,
                      int64_t in_stride = 0);
sf_status launch_hv0(const int64_t *ptr, const int32_t *atom, const double *w, int64_t n,
                     const double2 *v, double2 *out, cudaStream_t st);
sf_status launch_bupdate(const int32_t *idx, const double *w, int width, int64_t m,
                         const double2 *beta, double2 *b, unsigned long long *bmax,
                         cudaStream_t st, int batch = 1,
                         int64_t n_pix = 0);
sf_status launch_hz(const int64_t *ptr, const int32_t *atom, const double *w, int64_t n,
                    int64_t n_pad, const double *z, float *x, cudaStream_t st, int batch = 1,
                    int64_t zstride = 0, int64_t xstride = 0);
// x = H z from the entry-major transpose of H's CSR (ents <= 64 entries per
// pixel): thread = (scene, pixel), bitwise equal to k_hz (see sf_pixel.cu)
sf_status launch_hz_ell(const int32_t *atomT, const double *wT, int ents, int64_t n, int64_t n_pad,
                        const double *z, float *x, cudaStream_t st, int batch, int64_t zstride,
                        int64_t xstride);
constexpr int kPeerMaxRanks = 16;
struct PeerSlots {  // one channel / parity: every rank's slot array as mapped here
  double *p[kPeerMaxRanks] = {};
  int world = 0;
};
sf_status launch_pix_reduce(const float *P, int nt, int64_t n_pad, double *ypix, cudaStream_t st,
                            int batch = 1, const PeerSlots *peers = nullptr, size_t peer_off = 0);
sf_status launch_atom_step(const int32_t *idx, const double *w, int width, int64_t m,
                           const double *ypix, const double2 *b, double *zd, double *cprev,
                           const double *scal, const double *wv, int kstep, double *c_out,
                           cudaStream_t st, int batch = 1,
                           int64_t m_pad = 0, int64_t n_pad = 0);
bool is_atom_step_kernel(const void *f);
// Argument values of a captured k_atom_step graph node (kernel parameter order).
struct AtomStepNodeArgs {
  const int32_t *idx;
  const double *wt;
  int width;
  int64_t m;
  const double *ypix;
  const double2 *b;
  double *zd, *cprev;
  const double *scal, *wv;
  int kstep;
  double *c_out;
  int64_t m_pad, n_pad;
};
sf_status launch_pix_to_atom(const float *B, int ntp, const int32_t *idx, const double *w,
                             int width, int64_t m, double *A, cudaStream_t st);

// sf_geom.cu
sf_status launch_simulate_echo(const double *omega, int n_r, const double *gammas, int n_pulses,
                               const double *xyz, const double2 *rho, int64_t n, double2 *d,
                               cudaStream_t st);
// Batched launchers (trailing batch / stride arguments): scene s of a batched
// engine uses each buffer at base + s * (its per-scene size); batch = 1 is the
// single-scene engine.
sf_status launch_pixel_delays(const double *xyz, int64_t n, const double *gamma_dev,
                              double *tau, int *zero_flag, cudaStream_t st, int batch = 1,
                              int64_t in_stride = 0);
sf_status launch_forward_t(const double *omega, int n_r, const double *tau,
                           int64_t n, double2 *Ft, cudaStream_t st);
sf_status launch_delay_phase(const double *omega, int n_r, const double *tau,
                             int64_t n, double2 *F, cudaStream_t st);
sf_status launch_compose(const ComposeArgs &a, cudaStream_t st);
sf_status launch_kgram(const float *Gp, int64_t m_atoms, int n_r, int k_pad,
                       int nsplit, double2 *Kpart, cudaStream_t st);
sf_status launch_fq(const int64_t *qptr, const int32_t *qcol, const double *qval,
                    const double2 *Ft, int64_t n, int n_r, double2 *W, cudaStream_t st, int batch = 1);
sf_status launch_kgram_px(const double2 *Ft, const double2 *W, int64_t n, int n_r, int nsplit,
                          double2 *Kpart, cudaStream_t st, int batch);
sf_status launch_kreduce(const double2 *Kpart, int nsplit, const double2 *u0part,
                         int nu0, int n_r, int upper_only, double scale, double2 *K, float2 *Kf,
                         double2 *u0, cudaStream_t st, const double *sig = nullptr, int batch = 1,
                         int64_t in_stride = 0);
// apply = 1: L += max(inc, 0) with the fallback, counters++ (in-order use);
// apply = 0: only diag = {result, iterations, converged, |dA|_F} (pipelined use).
sf_status launch_power_iter(const double2 *K, const float2 *Kf, const double2 *u0,
                            int n_r, double rel_tol, int max_iter, double *L,
                            long long *counters, double *diag, cudaStream_t st, int apply = 1, int batch = 1);
sf_status launch_start_vector(int64_t n, uint64_t salt, double2 *v, cudaStream_t st);

// sf_gram.cu  (Re(A) tiles += Gp[I]^T-style products over the tile list)
// Gram update A = Ain + P^T P over the given tiles (Ain == A: in place)
sf_status launch_gram(int precision, const float *Gp, int k_pad, const int2 *tiles,
                      int64_t n_tiles, int nt, const float *Ain, float *A, cudaStream_t st);
sf_status launch_split_panels(const float *Gp, int64_t m_pad, int k_pad, const unsigned *maxbits,
                              int *exp_out, __half *Gh, cudaStream_t st, int batch = 1);
sf_status launch_gram_f16x3(const __half *Gh, int k_pad, int nt, const int2 *items, int n_items,
                            const int *exp_in, const float *Ain, float *A, int grid, cudaStream_t st, int batch = 1,
                            int64_t gh_stride = 0, int64_t a_stride = 0);
// diagonal tiles of the row-major upper-triangle store: A_II <- (A_II + A_II^T)/2
sf_status launch_symmetrize_diag(float *A, int nt, cudaStream_t st);

// sf_dirichlet.cu  (closed-form pixel Gram for a uniform frequency grid)
struct __align__(16) DirPix {
  double u;  // tau delta / (2 pi)
  float c, s;  // cos, sin(w_c tau); 0 for padded pixels
};
sf_status launch_dirichlet_prep(const double *tau, int64_t n_pix, int64_t dpad, const double *in,
                                int64_t in_stride, int n_r, DirPix *tab, int *flag,
                                cudaStream_t st, int batch = 1);
sf_status launch_gram_dirichlet(const DirPix *tab, int64_t dpad, const int2 *tiles,
                                int64_t n_tiles, int nt, const double *in, int64_t in_stride,
                                int64_t off_s, int n_r, const float *Ain, float *A, int grid,
                                cudaStream_t st, int batch, int64_t a_stride,
                                unsigned long long *next);
bool omega_uniform(const double *w, int n_r);


// Batch-oracle step size (sf_batch.cu): matrix-free power iteration on
// A = sum_k G_k^H G_k / sigma_k^2 in M space.
struct BatchLipArgs {
  const double *omega = nullptr, *gammas = nullptr, *inv_s2 = nullptr, *xyz = nullptr;
  int n_r = 0, n_pulses = 0, ell_width = 0;
  int64_t n = 0, m = 0;
  const int64_t *csr_ptr = nullptr;
  const int32_t *csr_atom = nullptr, *ell_idx = nullptr;
  const double *csr_w = nullptr, *ell_w = nullptr;
  const double2 *v0 = nullptr;
  double2 *work = nullptr;  // 2m + 2n + n_pulses * n_r complex, then 2 doubles
  unsigned long long *bmax_scratch = nullptr;
};
sf_status batch_lipschitz(const BatchLipArgs &a, double rel_tol, int max_iter, double *lam_out,
                          int *converged, cudaStream_t st);

// Morton tiles of <= 64 pixels with their Q neighbourhoods (sf_qtiles.cu).
struct QTileHost {
  int tiles = 0, max_union = 0, mc = 16;
  std::vector<int32_t> pix_off, pix_list, union_off, union_list, ent_off;
  std::vector<int16_t> ent_u;
  std::vector<double> ent_q;
};
sf_status build_q_tiles(const double *xyz, int64_t n, const int64_t *qptr, const int32_t *qcol,
                        const double *qval, QTileHost &out);

// Tensor-core K~ = F~ Q F~^H (sf_ktc.cu), on the Morton tiles of QTileHost.
struct KtcArgs {
  const float *X = nullptr;  // Gp [n_pad][k_pad]: [Re F~ | Im F~ | 0]
  int k_pad = 0, nb = 0;     // nb = ceil(k_pad / 128)
  const unsigned *maxbits = nullptr;  // max |X| (float bits)
  int tiles = 0;
  int tile_begin = 0, tile_end = 0;  // this rank's tiles (sharded: a contiguous range)
  int64_t ngrp = 0;          // pixel groups (8 Morton positions each) = 8 * tiles
  const int32_t *grp_pix = nullptr;  // [8 * ngrp] pixel id of each Morton slot, or -1
  const int32_t *ug_off = nullptr, *ug_list = nullptr;  // per tile: groups of its Q neighbourhood
  const int32_t *qchunk_off = nullptr;                  // per tile: first Q panel chunk
  const __half *qpanels = nullptr;
  int eq = 0;
  float qrow_max = 0.f;
  int cps = 0;               // K chunks (2 groups) per split of k_ktc_z
  __half *xs = nullptr;      // per scene: Xh | Xl | Yh | Yl slabs, each slab_stride halves
  int64_t slab_stride = 0;   // nb * ngrp * 1024
  int64_t xs_stride = 0;     // 4 * slab_stride
  int presplit = 0;        // Xh / Xl and exps already written (by k_forward_pix)
  float *zpart = nullptr;  // per scene: [cap + 2][nb(nb+1)/2][128][128] (partials, fp64 sum)
  int *exps = nullptr;     // per scene {ex, ey}
  int64_t x_stride = 0;    // batched scenes (grid y): X / zpart floats per scene
  int64_t z_stride = 0;
};
struct KtcHost {
  std::vector<__half> panels;
  std::vector<int32_t> chunk_off, ug_off, ug_list, grp_pix;
};
sf_status build_ktc_panels(const QTileHost &qt, KtcHost &out, int *eq_out, float *qrow_max);
int ktc_splits(const KtcArgs &a);
sf_status launch_ktilde_tc_partial(const KtcArgs &a, int grid, cudaStream_t st, int batch);
sf_status launch_ktilde_assemble(const KtcArgs &a, int grid, const double2 *u0part, int nu0,
                                 int n_r, double2 *K, float2 *Kf, double2 *u0, cudaStream_t st,
                                 int batch);
double *ktc_zsum(const KtcArgs &a, int grid);  // the fp64 Z blocks inside zpart
sf_status launch_ktilde_tc(const KtcArgs &a, int grid, const double2 *u0part, int nu0, int n_r,
                           double2 *K, float2 *Kf, double2 *u0, cudaStream_t st, int batch);

// sf_exact.cu (keep_complex atom-mode statistics)
sf_status launch_herk_c64(const double2 *G, int n_r, int64_t m, double inv_s2, double2 *A,
                          cudaStream_t st);
sf_status launch_kgram_c64(const double2 *G, int64_t m, int n_r, double inv_s2, int nsplit,
                           double2 *Kpart, cudaStream_t st);
sf_status launch_pack_re(const double2 *A, int64_t m, const int2 *tiles, int64_t n_tiles,
                         float *T, cudaStream_t st);
sf_status launch_seam_fista64(const double *gram, const double *corr, int64_t m, double tau,
                              double thresh, const double *w, int steps, double *z, double *cprev,
                              double *y, cudaStream_t st);
sf_status launch_dense_residual(const double2 *G, const double2 *d, int n_r, int64_t m,
                                const double *c, double inv_s2, double2 *r, double *grad,
                                double *quad, cudaStream_t st);

// sf_fista.cu
sf_status launch_bmax(const double2 *b, int64_t m_atoms, unsigned long long *bmax,
                      cudaStream_t st);
sf_status launch_fista_setup(const double *L, const unsigned long long *bmax, double lam,
                             double lam_rel, double *scal, cudaStream_t st, double t0 = 1.0,
                             int steps = 0, double *wv = nullptr, int batch = 1);
const void *fista_setup_kernel();
// One-scene pixel-mode FISTA prologue: k_fista_setup, k_fista_init and the
// first x = H z (k_hz, reading c0, which equals z at step 0) as one launch of
// independent block roles -- two dependent launch boundaries fewer per call.
struct PrologueArgs {
  const double *L = nullptr;
  const unsigned long long *bmax = nullptr;
  double lam = 0.0, lam_rel = 0.0, t0 = 1.0;
  double *scal = nullptr, *wv = nullptr;
  int steps = 0;
  const double *c0 = nullptr;
  int64_t m_atoms = 0, m_pad = 0;
  double *zd = nullptr, *cprev = nullptr;
  const int64_t *ptr = nullptr;
  const int32_t *atom = nullptr;
  const double *w = nullptr;
  int64_t n = 0, n_pad = 0;
  float *x = nullptr;
  int init_blocks = 0, hz_blocks = 0;
};
bool fista_prologue_ok(int64_t n_pad, int batch);
PrologueArgs make_prologue_args(const double *L, const unsigned long long *bmax, double lam,
                                double lam_rel, double *scal, double t0, int steps, double *wv,
                                const double *c0, int64_t m_atoms, int64_t m_pad, double *zd,
                                double *cprev, const int64_t *ptr, const int32_t *atom,
                                const double *w, int64_t n, int64_t n_pad, float *x);
sf_status launch_fista_prologue(const PrologueArgs &a, cudaStream_t st);
const void *fista_prologue_kernel();
sf_status launch_fista_init(const double *c0, int64_t m_atoms, int64_t m_pad,
                            double *zd, double *cprev, float *z32, cudaStream_t st, int batch = 1,
                            int64_t zstride = 0);
// storage of tile (I,J): upper-triangle index when sym, else I*nt + J
// reverse != 0 walks the tile list backwards (alternate FISTA steps: the tiles
// the previous step read last are still in L2 when this one starts)
sf_status launch_gemv(const float *A, const int2 *tiles, int64_t n_tiles,
                      const float *z32, float *P, int nt, int sym, int grid,
                      cudaStream_t st, int batch = 1,
                      int64_t xstride = 0, int reverse = 0, int dense = 0,
                      unsigned long long *bytes = nullptr);
sf_status launch_fista_step(const float *P, int nt, const double2 *b,
                            const double *corr, int64_t m_atoms, int64_t m_pad,
                            double *zd, double *cprev, float *z32,
                            const double *scal, double w, double *c_out,
                            cudaStream_t st);
// pack a dense fp64 [m][m] matrix into tiles; unpack tiles into dense fp64
sf_status launch_pack_tiles(const double *dense, int64_t m, const int2 *tiles,
                            int64_t n_tiles, float *A, cudaStream_t st);
sf_status launch_unpack_tiles(const float *A, const int2 *tiles, int64_t n_tiles,
                              int64_t m, int sym, double *dense, cudaStream_t st);

// sf_misc.cu
sf_status launch_pulse_metrics(const int64_t *csr_ptr, const int32_t *csr_atom,
                               const double *csr_w, int64_t n, const double *c, int64_t m,
                               const uint8_t *mask, const double2 *truth, const double2 *bp,
                               double inv_count, double threshold, double *scratch, double *out,
                               cudaStream_t st);
sf_status launch_reconstruct(const int64_t *csr_ptr, const int32_t *csr_atom,
                             const double *csr_w, int64_t n_pixels,
                             const double *c, double *img, cudaStream_t st);
sf_status launch_soft_threshold(const double *u, int64_t n, int is_complex,
                                double alpha, double *out, cudaStream_t st);
sf_status launch_zgemv(const double2 *X, int64_t n, const double2 *v,
                       double2 *w, cudaStream_t st);
sf_status launch_compose_ell_dense(const double2 *F, int n_r, int64_t n,
                                   const int32_t *ell_idx, const double *ell_w,
                                   int64_t m, int ell_width, double2 *G,
                                   cudaStream_t st);

// sf_shard.cu
void plan_items(int nt, int rank, int world, int64_t *i0, int64_t *i1, int64_t *ntiles);
void local_lists(int nt, int64_t i0, int64_t i1, std::vector<int2> &items_out,
                 std::vector<int2> &tiles_out);
sf_status nccl_unique_id(void *out128);
sf_status nccl_comm_init(void **comm, int world, const void *uid128, int rank);
sf_status nccl_allreduce_f64(double *buf, size_t count, void *comm, cudaStream_t st);
void nccl_comm_destroy(void *comm);
sf_status nccl_comm_dup(void *comm, int rank, void **out);
// in-process loopback group (emulated ranks on one device, sf_shard.cu)
constexpr int kLoopChannels = 2;  // 0: FISTA y_pix, 1: operator-phase K~ partials
struct LoopGroup;
sf_status loop_create(int world, LoopGroup **out);
void loop_destroy(LoopGroup *g);
int loop_world(const LoopGroup *g);
sf_status loop_allreduce_f64(LoopGroup *g, int ch, int rank, double *buf, size_t n,
                             cudaStream_t st);

// peer-memory group (ranks = processes of one node exchanging through each
// other's device memory, sf_shard.cu)
struct PeerGroup;
int64_t peer_blob_size();
sf_status peer_create(int device, int rank, int world, size_t cap_y, size_t cap_k,
                      uint64_t *shared_seq, PeerGroup **out);
sf_status peer_export(PeerGroup *g, void *blob);
sf_status peer_import(PeerGroup *g, const void *blobs);
void peer_destroy(PeerGroup *g);
int peer_world(const PeerGroup *g);
int peer_rank(const PeerGroup *g);
size_t peer_cap(const PeerGroup *g, int ch);
PeerSlots peer_targets(PeerGroup *g, int ch, size_t *offset);
sf_status peer_allreduce_f64(PeerGroup *g, int ch, double *buf, size_t n, cudaStream_t st,
                             bool pushed);

__host__ __device__ inline int64_t tri_index(int I, int J, int nt) {
  return (int64_t)I * nt - (int64_t)I * (I - 1) / 2 + (J - I);
}

}  // namespace sf
