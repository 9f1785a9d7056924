/*
 * sarfista_b200.h -- C ABI of the B200-native Online-FISTA engine.
 *
 * Drop-in boundary for the per-pulse hot path of the reference package
 * `sarfista` (arXiv 2603.08582).  Every entry point below names the
 * reference interface it replaces (file:line under the reference tree
 * `pkg/src/sarfista/`).  Plain pointers and sizes only: no torch, no C++.
 *
 * Conventions
 *   - Complex arrays are interleaved (re, im) doubles, i.e. numpy complex128.
 *   - `mem` selects where a caller buffer lives: SF_MEM_HOST (pageable or
 *     pinned host memory) or SF_MEM_DEVICE (a device pointer on the engine's
 *     GPU).  Device buffers are borrowed for the duration of the call only.
 *   - All work is issued on the engine's stream (sf_set_stream); calls that
 *     return values to host memory synchronise that stream.
 *   - Threading: one engine is single-writer (reference SPEC.md:364); calls
 *     on one engine must be serialised.  Distinct engines are independent.
 *   - Errors: every call returns sf_status; sf_last_error() gives a
 *     thread-local message.  SF_EINVAL maps to Python ValueError, SF_ESTATE
 *     to RuntimeError (mirrors solver.py:218-219), SF_ENOMEM to MemoryError.
 */
#ifndef SARFISTA_B200_H
#define SARFISTA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SF_ABI_VERSION 3

typedef enum sf_status {
  SF_OK = 0,
  SF_EINVAL = 1,      /* bad argument / shape (ValueError)            */
  SF_ESTATE = 2,      /* call not valid in this state (RuntimeError)  */
  SF_ECUDA = 3,       /* CUDA runtime error                           */
  SF_ENOMEM = 4,      /* device allocation failed                     */
  SF_ENCCL = 5,       /* NCCL error / NCCL unavailable                */
  SF_EUNSUPPORTED = 6 /* no sm_100 device / feature not built         */
} sf_status;

enum { SF_MEM_HOST = 0, SF_MEM_DEVICE = 1 };

/* Gram-update arithmetic. */
enum {
  SF_PREC_TF32X3 = 0, /* tcgen05 kind::tf32, hi/lo split, 3 MMAs            */
  SF_PREC_TF32 = 1,   /* tcgen05 kind::tf32, 1 MMA                         */
  SF_PREC_FP32 = 2,   /* SIMT fp32 FFMA                                    */
  SF_PREC_F16X3 = 3,  /* tcgen05 kind::f16, scaled fp16 hi/lo, 3 MMAs      */
  SF_PREC_DIRICHLET = 4 /* pixel mode, uniformly spaced omega only: the sum
                           over frequencies in closed form (Dirichlet kernel),
                           O(1) per stored entry, HBM read-modify-write bound */
};

/* Where the sufficient statistics live.  G = F H with a static dictionary H
 * gives A = H^T B H, B = sum F^H F / sigma^2 (N x N), b = H^T beta, so
 * geometric pulses can be accumulated in pixel space (N^2 instead of M^2
 * state, same iterates up to rounding).  Dense pulses need atom space. */
enum {
  SF_MODE_ATOM = 0,  /* Re(A) M x M tiles; geometric and dense pulses        */
  SF_MODE_PIXEL = 1  /* Re(B) N x N tiles + beta; geometric pulses only      */
};

typedef struct sf_engine sf_engine;

/* Engine descriptor.  The dictionary is given as an ELL table: atom j owns
 * ell_width (pixel index, weight) pairs; unused slots have index -1.
 * pixel_xyz may be NULL when only dense pulses (sf_accumulate_dense) are used. */
typedef struct sf_desc {
  int32_t abi_version;      /* SF_ABI_VERSION                               */
  int32_t device;           /* CUDA device ordinal                          */
  int64_t m_atoms;          /* M  (dictionary.py:57-63 m_atoms)             */
  int32_t n_freq;           /* N_r samples per pulse (geometry.py:78-90)    */
  int32_t ell_width;        /* max pixels per atom (0 if no dictionary)     */
  int64_t n_pixels;         /* N  (scene.py:77-79)                          */
  const int32_t *ell_idx;   /* host [m_atoms][ell_width]                    */
  const double *ell_w;      /* host [m_atoms][ell_width]                    */
  const double *pixel_xyz;  /* host [n_pixels][3] (scene.py:93-105)         */
  int32_t precision;        /* SF_PREC_*                                    */
  int32_t power_max_iter;   /* power-iteration cap, 0 = 500 (solver.py:139)  */
  double l_floor;           /* SufficientStatistics.empty l_floor (solver.py:97) */
  double power_rel_tol;     /* stopping tolerance, <= 0 = 1e-6; a negative value
                               means exactly 0 (fault injection: never converges) */
  int32_t mode;             /* SF_MODE_*                                    */
  int32_t batch;            /* independent scenes sharing dictionary, grid and
                               frequencies (0/1 = one; > 1 = BASELINE cfg2-style
                               batch, pixel mode, f16x3 or dirichlet); every per-scene
                               array of the calls below is then [batch][...] */
  int32_t keep_complex;     /* atom mode, dense pulses: also keep the complex
                               A (M x M complex128) exactly as the reference does
                               (solver.py:88-109, 191-193), update it in fp64 and
                               derive the fp32 Re(A) tiles FISTA reads from it;
                               K~ for the power iteration then comes from the fp64
                               operator.  Small M (reference-API drop-in use).  */
} sf_desc;

/* ---- engine lifetime ------------------------------------------------------ */
/* SufficientStatistics.empty (solver.py:96-109): allocates the packed
 * symmetric Re(A) tile store, b, L = l_floor on the device. */
sf_status sf_create(const sf_desc *desc, sf_engine **out);
/* Check the device (sm_100) and create its CUDA context ahead of the first
 * engine (optional; the drop-in package calls it at import). */
sf_status sf_init_device(int32_t device);
sf_status sf_destroy(sf_engine *eng);
/* cudaStream_t passed as void*; NULL = the legacy default stream.  Until the
 * first call the engine issues on a private non-blocking stream. */
sf_status sf_set_stream(sf_engine *eng, void *stream);
sf_status sf_synchronize(sf_engine *eng);
/* Re-zero A and b, L = l_floor, counters = 0. */
sf_status sf_reset(sf_engine *eng, double l_floor);
/* m_pad (tile-padded M), tile edge, number of stored tiles, device bytes. */
sf_status sf_info(const sf_engine *eng, int64_t *m_pad, int32_t *tile,
                  int64_t *n_tiles, int64_t *device_bytes);

/* ---- per-pulse update ------------------------------------------------------ */
/* accumulate() (solver.py:186-206) for a geometric pulse: the forward operator
 * F = exp(-j w tau) (geometry.py:97-107, kernels.py:27-29) and G = F H
 * (dictionary.py:151-157) are synthesised on the device from gamma and omega;
 * A += Re(G^H G)/sigma2, b += G^H d/sigma2, L += lambda_max(G^H G/sigma2)
 * (power iteration solver.py:139-175 restated in N_r space) with the
 * Frobenius fallback of solver.py:196-199.
 *   gamma  [3] platform position, omega [n_freq], d [n_freq] complex, all in
 *   `mem`.  Host inputs are validated before any work is queued (increasing
 *   frequencies, geometry.py:44-46; platform on a pixel, geometry.py:102-103);
 *   for device inputs the pixel check is recorded on the device and reported
 *   by the next sf_get_scalars. */
sf_status sf_accumulate_geom(sf_engine *eng, const double *gamma,
                             const double *omega, const double *d,
                             double sigma2, int32_t mem);
/* accumulate() for an explicit operator (tests, matrix-R pulses whitened on
 * the host): G [n_freq][m_atoms] complex, d [n_freq] complex. */
sf_status sf_accumulate_dense(sf_engine *eng, const double *G, const double *d,
                              int32_t n_freq, double sigma2, int32_t mem);

/* ---- FISTA ------------------------------------------------------------------ */
/* online_fista_pulse() (solver.py:209-226) + fista_inner (kernels.py:78-103).
 * Reads c0 [m_atoms] (never modified), writes c_out [m_atoms]; both in `mem`.
 * lam > 0 uses that lambda; lam <= 0 and lam_rel > 0 uses
 * lambda = lam_rel * max_j |b_j| computed on the device.  t0 is the carried
 * momentum scalar (solver.py:224); *t_out receives the advanced scalar. */
sf_status sf_fista(sf_engine *eng, const double *c0, double *c_out,
                   int32_t mem, double lam, double lam_rel, int32_t steps,
                   double t0, double *t_out);

/* ---- state readback / restore --------------------------------------------- */
sf_status sf_get_scalars(sf_engine *eng, double *L, int64_t *pulse_count,
                         int64_t *fallbacks, double *last_lambda);
/* Last power iteration: {increment, iterations, converged, |dA|_F}. */
sf_status sf_get_power_diag(sf_engine *eng, double *out4);
/* Roofline probe: a plain streaming read of the engine's current tile store
 * (the bytes one FISTA matvec reads), `iters` launches back to back on the
 * engine stream after one warm-up read; *us = mean microseconds per read.
 * Gives the measured ceiling (L2- or HBM-resident, as the store is) that the
 * matvec is compared with in bench.py. */
sf_status sf_probe_store_read(sf_engine *eng, int32_t iters, double *us);
/* Roofline probe: `iters` back-to-back launches of the FISTA matvec kernel on
 * the current tile store and input vector (pixel mode, after a FISTA call;
 * its partial-slot scratch is overwritten), after one warm-up launch; *us =
 * mean microseconds per launch (the kernel alone, same residency).  dense != 0
 * reads every tile element (the support-blind ceiling); 0 is the product's
 * support-aware read. */
sf_status sf_probe_matvec(sf_engine *eng, int32_t iters, int32_t dense, double *us);
/* y = Re(B) x with the product matvec kernels (pixel mode, one scene): x
 * [n_pad] float32 and y [n_pixels] float64, both DEVICE pointers; dense != 0
 * forces the support-blind read (tests: both reads are bitwise equal).  Uses
 * the FISTA scratch; call between pulses. */
sf_status sf_apply_store(sf_engine *eng, const float *x, double *y, int32_t dense);
/* b [m_atoms] complex */
sf_status sf_get_b(sf_engine *eng, double *b, int32_t mem);
/* Re(A) as a dense symmetric [m_atoms][m_atoms] float64 matrix. */
sf_status sf_get_A_re(sf_engine *eng, double *A_re, int32_t mem);
/* Restore (checkpoint resume, solver.py:335-369): A_re dense symmetric,
 * b complex; either pointer may be NULL to leave that part untouched.
 * Atom-space engines only (pixel-space state: sf_set_pixel_stats). */
sf_status sf_set_stats(sf_engine *eng, const double *A_re, const double *b,
                       double L, int64_t pulse_count, int64_t fallbacks,
                       int32_t mem);
/* Pixel-space state of an SF_MODE_PIXEL engine: Re(B) dense symmetric
 * [n_pixels][n_pixels] and beta [n_pixels] complex (b = H^T beta is derived). */
sf_status sf_get_pixel_stats(sf_engine *eng, double *B_re, double *beta,
                             int32_t mem);
sf_status sf_set_pixel_stats(sf_engine *eng, const double *B_re,
                             const double *beta, double L, int64_t pulse_count,
                             int64_t fallbacks, int32_t mem);
/* Raw packed tile store of the symmetric matrix (Re(A) or Re(B)) for
 * checkpoints: sf_tile_store returns the number of tiles this rank owns, the
 * tile-grid edge nt and their (I, J) pairs (int32 x 2 each, may be NULL);
 * sf_copy_tiles moves them (fp32, 128x128 each, engine layout) out of
 * (to_engine = 0) or into (to_engine = 1) the engine, in that order. */
sf_status sf_tile_store(sf_engine *eng, int64_t *n_local, int64_t *nt,
                        int32_t *tile_ij);
sf_status sf_copy_tiles(sf_engine *eng, float *buf, int32_t to_engine,
                        int32_t mem);
/* Back-projection accumulator of the baseline (baseline.py:23-33):
 * image_sum [n_pixels] complex = sum_k F_k^H d_k over the accumulated
 * geometric pulses, folded on the device (pixel-space engines). */
sf_status sf_get_bp(sf_engine *eng, double *image_sum, int64_t *pulse_count,
                    int32_t mem);
/* keep_complex engines: the complex A [m_atoms][m_atoms] (stats.A,
 * solver.py:88-109) and its restore (load_checkpoint, solver.py:335-369;
 * the dataclass constructor SufficientStatistics(A=..., b=..., L=...)). */
sf_status sf_get_A(sf_engine *eng, double *A, int32_t mem);
sf_status sf_set_stats_complex(sf_engine *eng, const double *A, const double *b, double L,
                               int64_t pulse_count, int64_t fallbacks, int32_t mem);
/* batch_objective / batch_gradient (solver.py:243-264) for one whitened dense
 * pulse: quad_out = |d - G c|^2 / sigma2; grad_inout += Re(G^H (G c - d)) / sigma2.
 * G [n_r][m] complex, d [n_r] complex, c [m] real, all host memory. */
sf_status sf_dense_residual(int32_t device, const double *G, const double *d, int32_t n_r,
                            int64_t m, const double *c, double sigma2, double *quad_out,
                            double *grad_inout);
/* Per-pulse reconstruction metrics on the device (replaces the host metrics of
 * reference harness.py:288-304 / metrics.py:31-56 and the residual of
 * harness.py:306-318): image = H c; c [m_atoms] float64, mask [n_pixels] uint8
 * (truth support), truth [n_pixels] complex128 or NULL (then res = |image|^2),
 * all DEVICE pointers.  out8 (host) = {count(|c| > threshold), sum |image| on
 * the mask, off the mask, sum |BP image| on, off (BP = |sum F^H d| / pulses;
 * zeros before the first pulse or in atom mode), sum |image - truth|^2, pixels
 * on, pixels off}.  Deterministic (fixed-order reductions). */
sf_status sf_pulse_metrics(sf_engine *eng, const double *c, const uint8_t *mask,
                           const double *truth, double threshold, double *out8);
/* Restore the back-projection sum (checkpoint resume; pairs with sf_get_bp). */
sf_status sf_set_bp(sf_engine *eng, const double *image_sum, int32_t mem);
/* reconstruct() (solver.py:294-299): img [n_pixels] = H c. */
sf_status sf_reconstruct(sf_engine *eng, const double *c, double *img,
                         int32_t mem);
/* Per-phase device times (ms) of the last accumulate / fista call.  Calls are
 * timed from the first sf_last_timings call on (or while sf_profile is on):
 * before that the per-call events are not recorded and 0 is reported. */
sf_status sf_last_timings(sf_engine *eng, float *accumulate_ms,
                          float *fista_ms);
/* ---- batch oracle (solver.py:267-291) ----------------------------------------
 * Top eigenvalue of A = sum_k G_k^H G_k / sigma_k^2 over n_pulses geometric
 * pulses (gammas [n_pulses][3], omega [n_r], sigma2 [n_pulses], host), by the
 * reference's power iteration (solver.py:139-175) run matrix-free on the
 * device; *converged = 0 returns the last Rayleigh value (solver.py:175). */
sf_status sf_batch_lipschitz(sf_engine *eng, const double *gammas,
                             const double *omega, const double *sigma2,
                             int32_t n_pulses, double rel_tol, int32_t max_iter,
                             double *lam, int32_t *converged);
/* ---- batched scenes (sf_desc.batch = B > 1; BASELINE cfg2) -----------------
 * One pulse for every scene: gammas [B][3], omega [n_r] (shared), d [B][n_r]
 * complex, sigma2 [B].  sf_fista then takes c0 / c_out as [B][m_atoms] (one
 * momentum t for all scenes); the single-scene getters report scene 0. */
sf_status sf_accumulate_geom_batch(sf_engine *eng, const double *gammas,
                                   const double *omega, const double *d,
                                   const double *sigma2, int32_t mem);
/* Per-scene L, pulse count, fallbacks ([B] each; NULL to skip). */
sf_status sf_get_batch_scalars(sf_engine *eng, double *L, int64_t *pulse_count,
                               int64_t *fallbacks);
/* Per-kernel CUDA-event timing on the engine stream.  enable != 0 starts a
 * fresh record; kinds: SF_K_GEMV (FISTA y = Re(A) z partials, one record per
 * matvec launch), SF_K_GRAM (tile update), SF_K_STEP (atom mode: reduce +
 * shrink; pixel mode: the whole FISTA loop), SF_K_OPERATOR (delays, F,
 * compose, K~, power iteration), SF_K_FISTA (one whole sf_fista call),
 * SF_K_KTILDE (the tensor-core K~ build alone, pixel mode), SF_K_FOLD (the
 * state update's second half: fold, b = H^T beta; pixel mode, incl. its wait
 * for the pulse's power iteration). */
enum { SF_K_GEMV = 0, SF_K_GRAM = 1, SF_K_STEP = 2, SF_K_OPERATOR = 3,
       SF_K_LIPSCHITZ = 4 /* K~ build + power iteration (side stream) */,
       SF_K_FISTA = 5, SF_K_KTILDE = 6, SF_K_FOLD = 7 };
sf_status sf_profile(sf_engine *eng, int32_t enable);
sf_status sf_profile_read(sf_engine *eng, int32_t kind, int64_t *launches,
                          double *total_ms);
/* Tile-store bytes the FISTA matvec requested since sf_profile(eng, 1): the
 * support-aware read loads only the live slabs / rows of each tile, so this is
 * the algorithmic byte count of the profiled launches (SF_K_GEMV). */
sf_status sf_profile_bytes(sf_engine *eng, int64_t *gemv_bytes);

/* ---- one scene over several GPUs (pixel-space engines) ----------------------
 * The Gram work items (2x2 super-tiles of the stored triangle) are split into
 * contiguous, tile-balanced ranges; rank r updates and multiplies with its own
 * tiles only, and each FISTA step sums the partial y_pix over ranks with one
 * NCCL all-reduce (fp64, N values).  The K~ build is split by Morton pixel
 * tiles: each pulse, rank r builds the Z-block partials of its contiguous tile
 * range and one all-reduce (fp64, (k_pad/128)(k_pad/128+1)/2 blocks of 128^2,
 * on a second communicator) sums them.  Everything else is computed
 * redundantly.
 * sf_plan_shard is host-only (no device).  sf_shard_init must precede the
 * first pulse; world == 1 with a NULL id runs the sharded code path alone. */
sf_status sf_plan_shard(int64_t n_dim, int32_t rank, int32_t world,
                        int64_t *item_begin, int64_t *item_end,
                        int64_t *tiles_local);
sf_status sf_nccl_unique_id(void *out128);
sf_status sf_shard_init(sf_engine *eng, int32_t rank, int32_t world,
                        const void *unique_id128);
/* Emulated ranks on ONE device (tests of the sharded engine path without
 * several GPUs): the engines of one process, each driven by its own host
 * thread in lockstep, exchange through a loopback group instead of NCCL --
 * every exchange copies the rank's partial into a device slot, meets the other
 * ranks at a host barrier, and sums the slots in rank order on the rank's
 * stream after stream-event waits (no kernel waits on another).  Same work
 * partition and exchange points as sf_shard_init.  The group must outlive the
 * engines sharded into it; a rank that stops calling makes the others' next
 * exchange fail with SF_ESTATE after 120 s instead of hanging. */
typedef struct sf_loopback sf_loopback;
sf_status sf_loopback_create(int32_t world, sf_loopback **group);
void sf_loopback_destroy(sf_loopback *group);
sf_status sf_shard_init_loopback(sf_engine *eng, int32_t rank, sf_loopback *group);
/* Peer-memory exchange: one process per GPU on one node, no collective library.
 * Every rank owns slot arrays in its device memory and maps every other rank's
 * (CUDA IPC; NVLink peer access).  Per FISTA step the slot-reduction kernel
 * stores the rank's partial y_pix straight into its slot on EVERY rank (fused
 * reduce + push), an interprocess event marks the push, the ranks' host threads
 * meet at a sequence counter in shared host memory, each stream waits on every
 * rank's event and sums the slots in rank order (identical bits everywhere);
 * the K~ partials travel the same way once per pulse.  No kernel waits on
 * another rank's kernel.  Set-up: sf_shard_sizes (slot sizes of an engine) ->
 * sf_peer_create on every rank with the SAME zero-initialised shared array of
 * 2 x 16 uint64 (e.g. POSIX shared memory) -> sf_peer_export, all-gather the
 * sf_peer_blob_size()-byte blobs in rank order by any means -> sf_peer_import
 * -> sf_shard_init_peer before the first pulse.  The group outlives its
 * engine; a rank that stops calling makes the others' next exchange fail with
 * SF_ESTATE after 120 s. */
typedef struct sf_peer_group sf_peer_group;
sf_status sf_shard_sizes(sf_engine *eng, int64_t *cap_y, int64_t *cap_k);
sf_status sf_peer_create(int32_t device, int32_t rank, int32_t world, int64_t cap_y,
                         int64_t cap_k, uint64_t *shared_seq, sf_peer_group **group);
int64_t sf_peer_blob_size(void);
sf_status sf_peer_export(sf_peer_group *group, void *blob);
sf_status sf_peer_import(sf_peer_group *group, const void *blobs);
void sf_peer_destroy(sf_peer_group *group);
sf_status sf_shard_init_peer(sf_engine *eng, sf_peer_group *group);

/* ---- engine-less seam functions (kernels.py:27-116 plugin seam) ----------- */
/* delay_phase_matrix (kernels.py:27-29, 66-76): out [n_r][n] complex (host). */
sf_status sf_delay_phase_matrix(int32_t device, const double *omegas,
                                int32_t n_r, const double *delays, int64_t n,
                                double *out);
/* fista_inner (kernels.py:32-53, 78-103) on a host gram_re [m][m]. */
sf_status sf_fista_inner(int32_t device, const double *gram_re,
                         const double *corr_re, const double *c0, int64_t m,
                         double t0, double tau, double thresh, int32_t steps,
                         double *c_out, double *t_out);
/* hermitian_top_eigenvalue (solver.py:139-175) on a host complex [n][n]. */
sf_status sf_hermitian_top_eigenvalue(int32_t device, const double *X,
                                      int64_t n, double rel_tol,
                                      int32_t max_iter, double *lam,
                                      int32_t *converged);
/* compose (dictionary.py:151-157): G [n_r][m] = F [n_r][n] @ H, H as ELL. */
sf_status sf_compose_ell(int32_t device, const double *F, int32_t n_r,
                         int64_t n, const int32_t *ell_idx,
                         const double *ell_w, int64_t m, int32_t ell_width,
                         double *G);
/* Noise-free pulse simulation (harness.py:221-234, d = F rho before noise) for
 * n_pulses platform positions gammas [n_pulses][3]: d [n_pulses][n_r] complex,
 * rho [n] complex (real scenes pass Im = 0); host memory. */
sf_status sf_simulate_echo(int32_t device, const double *omegas, int32_t n_r,
                           const double *gammas, int32_t n_pulses,
                           const double *pixel_xyz, const double *rho, int64_t n,
                           double *d);
/* soft_threshold (solver.py:229-240): real (is_complex=0) or complex input. */
sf_status sf_soft_threshold(int32_t device, const double *u, int64_t n,
                            int32_t is_complex, double alpha, double *out);

/* ---- diagnostics ------------------------------------------------------------ */
const char *sf_last_error(void);
int32_t sf_abi_version(void);
/* Number of kernels this library launched on the calling thread so far. */
int64_t sf_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SARFISTA_B200_H */
