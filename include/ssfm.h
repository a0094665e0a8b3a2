/*
 * ssfm.h -- C-ABI of the B200-native sparse Levenberg-Marquardt core
 * (bundle adjustment + global positioning) of InstantSfM (arXiv 2510.13310).
 *
 * This is the drop-in boundary that replaces the reference package's
 * native layer and the numpy/scipy hot path under `lm_solve`:
 *
 *   reference (sparsesfm, /root/reference/pkg/src/sparsesfm)      -> here
 *   ----------------------------------------------------------------------
 *   BAProblem.__init__            ba.py:35-64                      ssfm_create_ba
 *   GPProblem.__init__/fix_gauge  gp.py:33-67, gp.py:193-201       ssfm_create_gp
 *   problem.cost(theta)           ba.py:133-138, gp.py:103-107     ssfm_cost
 *   problem.linearize(theta)      ba.py:140-194, gp.py:109-128     ssfm_linearize
 *   jtj_fill_cy / jtr_fill_cy     _kernels/_core.pyx:18-97         (inside ssfm_linearize)
 *   apply_damping                 sparse_block.py:406-426          (inside ssfm_solve_normal)
 *   solve_normal -> _solve_schur  lm.py:537-720                    ssfm_solve_normal
 *   schur_fill_cy + dense S@p     _core.pyx:100-160, lm.py:656     (implicit S*p, inside the PCG)
 *   problem.post_step / renormalize  ba.py:196-197, lm.py:104-117,
 *                                 gp.py:130-147                    ssfm_post_step
 *   lm_solve                      lm.py:727-800                    ssfm_lm_solve
 *   JtJPattern.off_keys           sparse_block.py:219-323          ssfm_export_pattern
 *
 * Conventions
 *   - Plain pointers and sizes only. Array pointers are DEVICE pointers on the
 *     handle's device unless a parameter says "host". Streams are passed as
 *     `void*` (a cudaStream_t; NULL = legacy default stream).
 *   - theta is the reference parameter vector, same layout (lm.py, ba.py:68-81,
 *     gp.py:71-80): BA [C x (q4,t3)] ++ [P x 3] ++ [C focal | 1 shared | none];
 *     GP [C x 3] ++ [P x 3] ++ [N scales | none in depth mode].
 *   - All arithmetic is IEEE fp64.
 *   - Every entry point returns an ssfm_status; ssfm_last_error() gives the
 *     message of the last failure on the calling thread.
 *   - A handle is not thread-safe; separate handles may run concurrently.
 */
#ifndef SSFM_H
#define SSFM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes, 1:1 with the reference exception taxonomy (errors.py:4-77). */
typedef enum {
  SSFM_OK = 0,
  SSFM_SINGULAR_BLOCK = 1,      /* errors.SingularBlock      (errors.py:20)  */
  SSFM_CG_STALL = 2,            /* errors.CGStall            (errors.py:24)  */
  SSFM_SOLVER_FAILURE = 3,      /* errors.SolverFailure      (errors.py:28)  */
  SSFM_ZERO_QUATERNION = 4,     /* errors.ZeroQuaternion     (errors.py:39)  */
  SSFM_EMPTY_PROBLEM = 5,       /* errors.EmptyProblem       (errors.py:43)  */
  SSFM_MISSING_DEPTH = 6,       /* errors.MissingDepth       (errors.py:47)  */
  SSFM_LAYOUT_MISMATCH = 7,     /* errors.LayoutMismatch     (errors.py:12)  */
  SSFM_DIMENSION_MISMATCH = 8,  /* errors.DimensionMismatch  (errors.py:16)  */
  SSFM_INVALID_ARGUMENT = 9,    /* ValueError / IndexError                    */
  SSFM_CUDA_ERROR = 10,
  SSFM_COMM_ERROR = 11,        /* peer exchange of a sharded handle failed / timed out */
  SSFM_PARSE_ERROR = 12,       /* errors.ParseError "line N: reason" (errors.py:51) */
  SSFM_COUNT_MISMATCH = 13,    /* errors.CountMismatch      (errors.py:59)  */
  SSFM_DUPLICATE_OBSERVATION = 14 /* errors.DuplicateObservation (errors.py:63) */
} ssfm_status;

/* Termination reasons of SolveReport.termination (lm.py:61-83). */
typedef enum {
  SSFM_TERM_MAX_ITER = 0,
  SSFM_TERM_CONVERGED_COST = 1,
  SSFM_TERM_CONVERGED_GRAD = 2,
  SSFM_TERM_SOLVER_FAILURE = 3
} ssfm_termination;

enum { SSFM_PINHOLE = 0, SSFM_BAL_RADIAL = 1 };   /* scene.py:19-20 */
enum { SSFM_LOSS_TRIVIAL = 0, SSFM_LOSS_HUBER = 1, SSFM_LOSS_CAUCHY = 2 }; /* scene.py:233-242; Cauchy: an extension */

/* LMConfig (lm.py:36-58). solver: 0 = schur_pcg (the only device solver). */
typedef struct {
  int32_t max_iterations;
  double lambda0, lambda_up, lambda_down, lambda_min, lambda_max;
  double rel_cost_tol, grad_tol;
  int32_t cg_max_iters;
  double cg_tol;
} ssfm_lm_config;

/* IterationRecord (lm.py:61-69). */
typedef struct {
  int32_t iteration;
  int32_t step_accepted;
  int32_t cg_iters;
  int32_t status;          /* in-step failure that caused a rejection, else 0 */
  double cost_before, cost_after, lam;
  int64_t wall_time_ns;    /* host clock around the iteration, like lm.py:755 */
  double device_ms;        /* CUDA-event time of the iteration on the stream */
} ssfm_iter_record;

/* BAProblem(scene, loss, optimize_focal, shared_focal), ba.py:35-64.
 * Observation arrays are in the scene's observation order (residual order). */
typedef struct {
  int32_t num_cameras;
  int32_t num_points;
  int64_t num_obs;
  int32_t model;           /* SSFM_PINHOLE | SSFM_BAL_RADIAL */
  int32_t optimize_focal;
  int32_t shared_focal;
  int32_t loss_kind;
  double loss_delta;
  const int32_t* cam_idx;  /* [N] device */
  const int32_t* pt_idx;   /* [N] device */
  const double* pixels;    /* [N,2] device */
  const double* pps;       /* [C,2] device, principal points */
  const double* dists;     /* [C,2] device, bal radial (k1,k2) */
  const double* focals;    /* [C] device, used when optimize_focal == 0 */
} ssfm_ba_desc;

/* GPProblem(rays, fixed_rotations, cam_idx, pt_idx, num_points, loss,
 * depth_mode, depths) + fix_gauge, gp.py:33-67 / gp.py:193-201. */
typedef struct {
  int32_t num_cameras;
  int32_t num_points;
  int64_t num_obs;
  int32_t depth_mode;
  int32_t gauge_fixed;
  int32_t loss_kind;
  double loss_delta;
  const int32_t* cam_idx;  /* [N] device */
  const int32_t* pt_idx;   /* [N] device */
  const double* rays;      /* [N,3] device, unit world rays (make_rays) */
  const double* depths;    /* [N] device ray distances, depth mode only (else NULL) */
} ssfm_gp_desc;

typedef struct ssfm_handle ssfm_handle;

const char* ssfm_last_error(void);
const char* ssfm_version(void);

/* Build a problem: copies the inputs into the handle's device arena and builds
 * the point-major / camera-major orderings, segments and work tiles on the
 * device (replaces JtJPattern / JtrPattern / _SchurPlan construction,
 * sparse_block.py:219-363, lm.py:236-483). */
int ssfm_create_ba(const ssfm_ba_desc* desc, void* stream, ssfm_handle** out);
int ssfm_create_gp(const ssfm_gp_desc* desc, void* stream, ssfm_handle** out);
int ssfm_destroy(ssfm_handle* h);

/* ---- grow-only device arena (Workspace, lm.py:86-101; the spec's unified
 * memory pool) -------------------------------------------------
 * Handles created with ssfm_create_*_in take every device allocation from the
 * arena (bump allocation). Destroying the last live handle resets it, so the
 * next stage's handle (GP -> BA) reuses the same HBM without cudaMalloc; a
 * stage that needs more adds a chunk, and an idle arena coalesces its chunks
 * into one of the high-water size. reserve_bytes (may be 0) is allocated up
 * front. The arena must outlive its handles (ssfm_arena_destroy fails with
 * SSFM_INVALID_ARGUMENT while handles are live). device: the current device
 * (-1). ssfm_arena_info: capacity, high-water mark, live handles and the
 * number of cudaMalloc calls the arena made (any pointer may be NULL). */
typedef struct ssfm_arena ssfm_arena;
int ssfm_arena_create(int32_t device, int64_t reserve_bytes, ssfm_arena** out);
int ssfm_arena_destroy(ssfm_arena* arena);
int ssfm_arena_info(ssfm_arena* arena, int64_t* capacity, int64_t* high_water, int32_t* live_handles,
                    int64_t* chunk_mallocs);
int ssfm_create_ba_in(const ssfm_ba_desc* desc, ssfm_arena* arena, void* stream, ssfm_handle** out);
int ssfm_create_gp_in(const ssfm_gp_desc* desc, ssfm_arena* arena, void* stream, ssfm_handle** out);

/* Device block cache. ssfm_destroy hands a handle's device blocks to a
 * per-process cache (exact-size reuse: re-creating a handle of the same shape
 * skips cudaMalloc/cudaFree, 40-190 ms at C5), capped by SSFM_BLOCK_CACHE_GB or
 * a quarter of the device's HBM. A failed allocation releases the cache and
 * retries. ssfm_trim_cache frees the cached blocks of `device` (-1: all
 * devices); ssfm_cache_bytes = bytes currently cached. */
int ssfm_trim_cache(int32_t device, int64_t* freed_bytes);
int64_t ssfm_cache_bytes(void);

int64_t ssfm_num_params(const ssfm_handle* h);
int64_t ssfm_num_residuals(const ssfm_handle* h);
int64_t ssfm_device_bytes(const ssfm_handle* h);

/* cost(theta) -> *cost_host (blocking). ba.py:133-138 / gp.py:103-107. */
int ssfm_cost(ssfm_handle* h, const double* theta, double* cost_host, void* stream);

/* linearize(theta): fills the handle's compact Jacobian and the block
 * normal-equation pieces. Optional exports in the reference layout
 * (ba.py:185-193, gp.py:118-128): r [total_residuals], J [N x 22 | 21 | 18]
 * row-major per entry, grad = J^T r [total_params] (jtr, sparse_block.py:388).
 * *grad_max_host (may be NULL) = max |J^T r| (lm.py:762). */
int ssfm_linearize(ssfm_handle* h, const double* theta, double* r_out,
                   double* J_out, double* grad_out, double* grad_max_host,
                   void* stream);

/* solve_normal(apply_damping(jtj, lambda), ...) (lm.py:537-720) on the state of
 * the last ssfm_linearize; delta [total_params] device. Returns SSFM_OK,
 * SSFM_SINGULAR_BLOCK or SSFM_CG_STALL (a rejection inside lm_solve). */
int ssfm_solve_normal(ssfm_handle* h, double lambda, const ssfm_lm_config* cfg,
                      double* delta, int32_t* cg_iters_host, void* stream);

/* post_step in place (renormalize lm.py:104-117 / GP gauge gp.py:130-147). */
int ssfm_post_step(ssfm_handle* h, double* theta, void* stream);

/* lm_solve (lm.py:727-800). theta in/out (device). recs: host array of cap
 * records; *n_recs = records written; *termination = ssfm_termination.
 * Returns SSFM_SOLVER_FAILURE (records still valid) when the linear solve
 * fails with lambda at lambda_max. */
int ssfm_lm_solve(ssfm_handle* h, double* theta, const ssfm_lm_config* cfg,
                  ssfm_iter_record* recs, int32_t cap, int32_t* n_recs,
                  int32_t* termination, void* stream);

/* ba.prune (ba.py:223-261) on the device: points seen by fewer than two
 * cameras and cameras left without observations are dropped to a fixed point.
 * cam_idx / pt_idx [n] int32, camera_map [C] / point_map [P] int32 (old ->
 * new, -1 removed), obs_mask [n] uint8: device arrays. *n_cam_out, *n_pt_out,
 * *n_obs_out: survivors. SSFM_EMPTY_PROBLEM when nothing survives. */
int ssfm_prune(int64_t n, const int32_t* cam_idx, const int32_t* pt_idx, int32_t C, int32_t P,
               int32_t* camera_map, int32_t* point_map, uint8_t* obs_mask, int32_t* n_cam_out,
               int32_t* n_pt_out, int64_t* n_obs_out, void* stream);

/* The CUDA device a handle lives on. */
int32_t ssfm_handle_device(const ssfm_handle* h);

/* Several devices in one process (dist.connect_local): enable direct access
 * from `device` to `peer` before their handles' exchange regions are
 * connected (ssfm_comm_connect with region pointers). SSFM_COMM_ERROR when
 * the devices cannot access each other. */
int ssfm_enable_peer_access(int32_t device, int32_t peer);

/* How lm_solve runs its loop on this handle: 1 = the whole LM loop as one
 * CUDA graph (accept/reject, lambda and termination decided on the device,
 * one read-back per solve; single-rank BA handles, SSFM_LM_GRAPH=0 disables),
 * -1 = host loop (graph unavailable), 0 = not decided yet (no solve ran). */
int32_t ssfm_lm_mode(const ssfm_handle* h);

/* Reference-equivalent integer structures, bit-exact with the reference:
 *  - obs_pt_order [N] int32: stable point-major permutation of observations
 *  - obs_cam_order [N] int32: stable camera-major permutation
 *  - off_keys: JtJPattern.off_keys (sparse_block.py:263-266), int32 [K,2]
 *    sorted (a<b), written when off_keys != NULL and cap >= K; *n_off = K.
 *  - slots: _SchurPlan retained slots (lm.py:338-384), int32 [S,2] sorted by
 *    retained pair code, written when slots != NULL and cap >= S; *n_slots = S.
 * All outputs are device pointers (any may be NULL). */
int ssfm_export_pattern(ssfm_handle* h, int32_t* obs_pt_order,
                        int32_t* obs_cam_order, int32_t* off_keys,
                        int64_t off_cap, int64_t* n_off, int32_t* slots,
                        int64_t slot_cap, int64_t* n_slots, void* stream);

/* Timing hooks for bench.py: per-kernel-class accumulated device time of the
 * last lm_solve (ms) and launch counts. kind: 0 = PCG operator (S*p), 1 =
 * linearize, 2 = all, 3..7 = BA PCG phases measured inside the persistent
 * kernel by block 0 (point or fused pass, camera pass, q = S p, x/r/z update,
 * p update; each including its grid barrier). */
int ssfm_profile_get(const ssfm_handle* h, int32_t kind, double* ms,
                     int64_t* launches, double* bytes);
int ssfm_profile_enable(ssfm_handle* h, int32_t on);

/* ---- point-sharded multi-GPU solve -------------------
 * Each rank creates its handle from ITS shard: every camera (replicated), a
 * contiguous range of points renumbered from 0 and all observations of those
 * points (theta = [7C poses | 3 P_local points | focals]). Camera-side sums
 * and scalar reductions are exchanged through peer memory (csrc/comm.cuh);
 * the camera half of S*p is exchanged inside the persistent PCG kernel every
 * CG iteration. Replicated quantities are combined in rank order on every
 * rank, so all ranks hold bitwise-identical camera parameters and take the
 * same LM / CG decisions. After ssfm_comm_connect every call that computes
 * (cost, linearize, solve_normal, lm_solve) is collective over the ranks.
 *
 * ssfm_comm_init: allocate this rank's exchange region; *ipc_handle_out (64
 *   bytes, may be NULL) receives its cudaIpcMemHandle_t, *region_out (may be
 *   NULL) its device pointer. nranks <= 16. BA handles only.
 * ssfm_comm_connect: map the peers' regions, from IPC handles (nranks x 64
 *   bytes, one process per GPU) or from raw device pointers (several handles
 *   of one process on one device); entries for this rank are ignored. */
int ssfm_comm_init(ssfm_handle* h, int32_t rank, int32_t nranks, void* ipc_handle_out,
                   void** region_out);
int ssfm_comm_connect(ssfm_handle* h, const void* ipc_handles, void* const* regions);

/* reproj_rmse statistics (synth_metrics.py:312-325) on the device: sum of
 * squared (unweighted) pixel errors and the number of observations in front of
 * their camera, for theta (device). rmse = sqrt(*sum_sq / *count). BA only. */
int ssfm_reproj_stats(ssfm_handle* h, const double* theta, double* sum_sq, int64_t* count, void* stream);

/* ---- generic block algebra (the reference's public sparse_block API) -----
 * Device pointers; the contribution schedules are the reference's JtJPattern
 * (sparse_block.py:219-323) and JtrPattern (:326-363), built by the caller.
 * Results are bit-identical to the reference's Cython fills.
 * ssfm_block_jtj   replaces jtj_fill_cy (_core.pyx:18-58): out_data[key blocks]
 * ssfm_block_jtr   replaces jtr_fill_cy (_core.pyx:61-97): out[param scalars]
 * ssfm_block_scale_diag replaces scale_diag_inplace (sparse_block.py:429-439):
 *                  data[diag_idx[k]] *= factor */
int ssfm_block_jtj(const double* entry_data, const int64_t* entry_off, const int32_t* entry_h,
                   const int32_t* entry_w, const int64_t* contrib_a, const int64_t* contrib_b,
                   const int64_t* seg_start, const int64_t* key_out_off, int64_t nkeys,
                   double* out_data, void* stream);
int ssfm_block_jtr(const double* entry_data, const int64_t* entry_off, const int32_t* entry_h,
                   const int32_t* entry_w, const int32_t* by_entry, const int64_t* seg_start,
                   const int64_t* seg_out, const int64_t* res_row, int64_t nsegs,
                   const double* residuals, double* out, void* stream);
int ssfm_block_scale_diag(double* data, const int64_t* diag_idx, int64_t n, double factor, void* stream);

/* ---- dense solver (lm.py:124-220; LMConfig(solver="dense")) -------------
 * ssfm_dense_scatter: A[dst[k]] = data[src[k]] (materialize_dense with the
 *   caller's _DensePlan indices; A is n x n row-major, zero-initialised).
 * ssfm_dense_solve: in place on A: pin zero diagonals (SSFM_SINGULAR_BLOCK if
 *   the gradient entry is non-zero), reject negative diagonals, Jacobi
 *   equilibration, Cholesky (cuSOLVER potrf, loaded with dlopen on first use),
 *   x = solution of A x = b. All pointers device. */
int ssfm_dense_scatter(const double* data, const int64_t* dst, const int64_t* src, int64_t m,
                       double* A, void* stream);
int ssfm_dense_solve(double* A, const double* b, double* x, int64_t n, void* stream);

/* ---- Schur PCG on an explicit BlockNormalSystem ---------------------------
 * ssfm_schur_solve replaces _solve_schur (lm.py:537-704) for a damped system
 * held in the reference's block storage (sparse_block.py:162-216: `data`,
 * `gradient` = -J^T r). The plan is the integer schedule of _SchurPlan
 * (lm.py:236-483), built once per pattern by the caller (generic._SchurXPlan):
 * retained blocks (pose / focal / gp_center) form the reduced system, point
 * blocks (point / gp_point, width 3) are eliminated, and scale blocks
 * (gp_scale, width 1) are eliminated first. All pointers are device pointers.
 * Returns SSFM_OK, SSFM_SINGULAR_BLOCK (masked scale / point direction with a
 * non-zero gradient, det <= 0, singular preconditioner block, masked retained
 * direction with a non-zero reduced gradient) or SSFM_CG_STALL. */
typedef struct {
  int64_t n_params, n_ret, n_rblk, n_pt, n_u, n_slots, n_sc, n_direct;
  const int64_t* ret_s_off;   /* [n_rblk+1] reduced offset of each retained block */
  const int64_t* ret_theta;   /* [n_ret] theta row of each reduced scalar */
  const int64_t* pre_off;     /* [n_rblk+1] offset of each w x w preconditioner block */
  const int64_t* direct_dst;  /* [n_direct] S[dst[k]] = data[src[k]] (row-major n_ret x n_ret) */
  const int64_t* direct_src;
  const int64_t* pt_diag;     /* [n_pt] data offset of the point's 3x3 diagonal block */
  const int64_t* pt_theta;    /* [n_pt] theta row of the point's first scalar */
  const int32_t* u_w;         /* [n_u] U entry (retained x point coupling): retained width */
  const int32_t* u_ret;       /*        retained block (local index) */
  const int32_t* u_pt;        /*        point (local index) */
  const int64_t* u_off;       /* [n_u+1] offset in the U store (w x 3 row-major per entry) */
  const int64_t* u_gather;    /* [u_off[n_u]] data index of every U scalar */
  const int32_t* u_by_ret;    /* [n_u] entries grouped by retained block, entry order */
  const int64_t* ret_useg;    /* [n_rblk+1] */
  const int32_t* u_by_pt;     /* [n_u] entries grouped by point, entry order */
  const int64_t* pt_useg;     /* [n_pt+1] */
  const int64_t* slot_seg;    /* [n_slots+1] contribution segment of each S slot */
  const int32_t* slot_ra;     /* [n_slots] retained blocks of the slot, ra <= rb */
  const int32_t* slot_rb;
  const int32_t* con_ua;      /* [slot_seg[n_slots]] U entries (a, b) of each contribution */
  const int32_t* con_ub;
  const int64_t* sc_diag;     /* [n_sc] data offset of the scale's 1x1 diagonal */
  const int64_t* sc_theta;    /* [n_sc] theta row of the scale */
  const int64_t* sc_uc;       /* [n_sc] data offset of the 3 retained-scale couplings */
  const int64_t* sc_up;       /* [n_sc] data offset of the 3 point-scale couplings */
  const int32_t* sc_c;        /* [n_sc] retained block (width 3) */
  const int32_t* sc_p;        /* [n_sc] point */
  const int32_t* sc_u;        /* [n_sc] U entry joining (sc_c, sc_p) */
  const int32_t* sc_by_c;     /* scales grouped by retained block */
  const int64_t* c_scseg;     /* [n_rblk+1] */
  const int32_t* sc_by_p;     /* scales grouped by point */
  const int64_t* p_scseg;     /* [n_pt+1] */
  const int32_t* sc_by_u;     /* scales grouped by U entry */
  const int64_t* u_scseg;     /* [n_u+1] */
} ssfm_schur_plan;

int ssfm_schur_solve(const ssfm_schur_plan* plan, const double* data, const double* gradient,
                     const ssfm_lm_config* cfg, double* delta, int32_t* cg_iters_host, void* stream);

/* Diagnostic (BA): number of Jacobian entries where the camera-major copy
 * (written by the camera-tile linearize pass) differs bitwise from the
 * point-major copy, after ssfm_linearize. Expected 0. */
int ssfm_check_jacobian(ssfm_handle* h, int64_t* mismatches, void* stream);

/* Diagnostic (BA and GP): mean time (ms) of one standalone launch of a pass
 * of the two-pass Schur operator over the current linearization, reps
 * launches after warm-up. which: 0 = point pass (point-major records, camera
 * vector gather -> y), 1 = camera pass (camera-major records, y gather ->
 * tile sums), 2 = both back to back. Call after ssfm_solve_normal. */
int ssfm_bench_operator(ssfm_handle* h, int32_t which, int32_t reps, double* ms_out, void* stream);

/* Which Schur operator the PCG kernel of this handle runs (no reference
 * counterpart; it replaces the dense S@p of lm.py:656). *slot_groups = 0: the
 * two-pass operator (point-major then camera-major Jacobian reads); >= 1: the
 * fused single-pass operator with the 8 camera slots split over that many CTAs
 * (fused.cuh). *grid / *threads: the persistent kernel's launch geometry.
 * *smem_bytes: dynamic shared memory per CTA. Any pointer may be NULL. */
int ssfm_operator_info(const ssfm_handle* h, int32_t* slot_groups, int32_t* grid,
                       int32_t* threads, int64_t* smem_bytes);

/* ---- accuracy metrics on device-resident scenes ----------------------------
 * ssfm_rotation_auc   replaces synth_metrics.rotation_auc (synth_metrics.py:
 *   281-309): q_est/q_true [C][4] device (w,x,y,z, unnormalised), taus/auc host
 *   [ntau] (1..16), auc on the reference's 0-100 scale.
 * ssfm_center_moments  the Umeyama moments of synth_metrics.align (:225-238):
 *   x (estimate), y (truth) [n][3] device; out host [17] = mx(3), my(3),
 *   cov = yc^T xc / n (9, row-major), var_x, sum |x - y|^2 (center_rmse, :260).
 *   The 3x3 SVD and sign fix are host logic, as in the reference.
 * ssfm_apply_sim3  the scene transform of align (:244-256): rot [9] row-major,
 *   trans [3], rq_conj [4] host; quats [C][4], centers [C][3], points [P][3]
 *   device, transformed in place. */
int ssfm_rotation_auc(const double* q_est, const double* q_true, int32_t C, const double* taus, int32_t ntau,
                      double* auc, void* stream);
int ssfm_center_moments(const double* x, const double* y, int32_t n, double* out, void* stream);
int ssfm_apply_sim3(const double* rot, const double* trans, double scale, const double* rq_conj, double* quats,
                    double* centers, int32_t C, double* points, int64_t P, void* stream);

/* ssfm_make_rays: gp.make_rays (gp.py:150-177) input preparation on the device,
 * bit-identical to numpy: rays [n][3] = normalize(R(q)^T ((u-cx)/f, (v-cy)/f, 1));
 * with depths (or NULL), ray_depths [n] = depth * |dirs|. Device pointers;
 * cam_idx int64 [n], pixels [n][2], pps [C][2], focals [C], quats [C][4]. */
int ssfm_make_rays(int64_t n, const int64_t* cam_idx, const double* pixels, const double* pps, const double* focals,
                   const double* quats, const double* depths, double* rays, double* ray_depths, void* stream);

/* ---- BAL problem files (io.read_bal, io.py:83-131) ------------------------
 * Array-native host reader: ssfm_bal_read parses `path` (the reference's token,
 * error-message and line-number rules) and returns counts[3] = C, P, N;
 * ssfm_bal_take copies out cam_idx / pt_idx [N] int64, pixels [N][2],
 * cam_params [C][9] (angle-axis, translation, focal, k1, k2), points [P][3]
 * (host arrays); ssfm_bal_free releases the reader. Errors: SSFM_PARSE_ERROR,
 * SSFM_COUNT_MISMATCH (trailing tokens), SSFM_DUPLICATE_OBSERVATION. */
typedef struct ssfm_bal ssfm_bal;
int ssfm_bal_read(const char* path, ssfm_bal** out, int64_t* counts);
int ssfm_bal_take(ssfm_bal* reader, int64_t* cam_idx, int64_t* pt_idx, double* pixels, double* cam_params,
                  double* points);
void ssfm_bal_free(ssfm_bal* reader);

#ifdef __cplusplus
}
#endif

#endif /* SSFM_H */
