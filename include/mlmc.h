/*
 * mlmc.h -- C-ABI of the B200-native MPML hot path (arXiv 2503.05533).
 *
 * The library (paper_2503_05533_b200/libmlmc.so, sm_100a) computes, for one
 * level l of the multilevel hierarchy and a batch of samples, the coupled
 * differences Y_l = Q~_l(omega) - Q~_{l-1}(omega) of the paper's MLMC estimator
 * (Eq. (3)), each Q~ obtained by solving the P1 FE system
 * A(omega) x = b of -div(a grad u) = 1 on (0,1)^2 (Eq. (19)) only to
 * the relative residual the adaptive algorithm permits (Eq. (2), P:70-73;
 * Eq. (16)), and returns the per-level sums Algorithm 2 needs
 * (P:357-379).  Citation keys: P:n = PAPER.md line n; Rk = reading k of
 * DESIGN.md section 3.
 *
 * Conventions for every entry point
 *  - Return value: MLMC_OK (0) or one of the MLMC_E* codes below.  A failing
 *    call leaves outputs unspecified; mlmc_last_error() gives a message.
 *  - Pointers are plain host or device pointers; no framework types.  "dev"
 *    means CUDA device memory on the ctx's device, "host" means ordinary (or
 *    pinned) host memory.  The caller owns every buffer it passes; the
 *    library never frees or retains caller memory beyond the call, except the
 *    workspace bound with mlmc_bind_workspace (borrowed until rebound or
 *    mlmc_destroy).
 *  - A ctx is bound to one device and one CUDA stream; it is not thread-safe.
 *  - Sample identity: (seed, level, global index) fully determines the random
 *    input xi (Philox4x32-10, R12), so results do not depend on batching,
 *    rank count or call order.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns MLMC_ECUDA.
 */
#ifndef MLMC_H
#define MLMC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes (mirroring the SPEC exit codes 0/2/3/4) ---------- */
#define MLMC_OK      0
#define MLMC_EINVAL  2   /* invalid argument / configuration */
#define MLMC_ESOLVER 3   /* a solve failed (no convergence, breakdown, overflow) */
#define MLMC_ELMAX   4   /* Algorithm 2 reached L_max with the bias test failing (R2) */
#define MLMC_ECUDA   5   /* CUDA error, no device, or kernel image missing */
#define MLMC_ENOMEM  6   /* workspace too small / allocation failed */

#define MLMC_MAX_LEVELS 16
#define MLMC_SUMS_LEN   12   /* doubles per mlmc_level_sums */
#define MLMC_SAMPLE_LEN 8    /* doubles per per-sample record */

/* ---- problem definition ----------------------------------------------------
 * field = MLMC_FIELD_EXPCOV_KL: log a is a centred Gaussian field with
 *   covariance sigma2 * exp(-|x1-y1|/corr_len - |x2-y2|/corr_len), truncated
 *   to its m largest Karhunen-Loeve modes (BASELINE configs; R11).
 * field = MLMC_FIELD_PAPER_EQ20: Eq. (20): log a = sum_{j<=m}
 *   omega_j j^-q_decay sin(2 pi j x1) cos(2 pi j x2), omega_j ~ N(0, sigma2)
 *   (the paper's s is m here).
 * Mesh level l has h_l = 1/(h0_inv * refine^l), refine must be 2,
 * levels 0..L_max; h0_inv * 2^L_max <= 512.                                  */
typedef enum { MLMC_FIELD_EXPCOV_KL = 0, MLMC_FIELD_PAPER_EQ20 = 1 } mlmc_field;

typedef struct {
    int32_t field;
    int32_t m;          /* KL terms (1..1024) */
    double  sigma2;     /* variance of log a (EXPCOV) / of omega_j (EQ20) */
    double  corr_len;   /* EXPCOV correlation length, > 0 */
    double  q_decay;    /* EQ20 decay exponent */
    int32_t h0_inv;     /* 1/h0 (>= 2) */
    int32_t refine;     /* m of P:308; only 2 is supported */
    int32_t L_max;      /* finest level the plan supports */
    int32_t device;     /* CUDA device ordinal */
} mlmc_problem;

/* ---- solver and precision (Algorithm 1's quadruple) -------------
 * solver = MLMC_SOLVER_MINRES: unpreconditioned MINRES from x0 = 0, all
 *   arithmetic binary64, stop at the first k with phibar_k/||b|| <=
 *   tol (Eq. (2) with C = 1, R9).  u_* fields ignored.
 * solver = MLMC_SOLVER_CHOL_IR: Algorithm 1: banded Cholesky in
 *   u_f (MLMC_FMT_E4M3 / F16 / F32 / F64), initial and correction substitutions in
 *   u_s (F32 or F64, R24; F16 with an E4M3 / F16 factor and u <= F32, as the paper's
 *   "hh.." quads), residual in u_r and x in u (u = u_r, F64, F32 or F16 -- the
 *   paper's "..ss" / "..hh" quads of Table 1 right; binary16 arithmetic
 *   computed in binary32 and rounded once per operation), stop when ||r||/||b|| < tol
 *   (P:120), at most max_iter refinement steps.
 * solver = MLMC_SOLVER_MGCG (NEXT-4 of SURVEY section 8(f), h = 1/8 .. 1/512): conjugate gradients in
 *   binary64 preconditioned by one symmetric multigrid V(1,1) cycle in binary32 (nested P1 meshes,
 *   Galerkin-exact coarse operators, red-black Gauss-Seidel), the same stopping rule ||r_k||/||b|| <=
 *   tol (r_k the CG recurrence residual) and the same records; iterations are CG steps.  u_* ignored.
 *   h >= 1/64: every grid on chip; h <= 1/128: one CTA per system over workspace scratch.
 * solver = MLMC_SOLVER_CG (NEXT-4; h = 1/8 .. 1/64): plain conjugate gradients in binary64 from x0 = 0,
 *   the other Krylov method the paper names for these SPD systems; stopping rule and records as
 *   MG-PCG, default max_iter as MINRES, cost model as MINRES (iterations x n).  u_* ignored.
 * max_iter = 0 selects the default (MINRES: 16n+1000 -- loss of orthogonality
 * at coefficient contrasts ~1e7 takes well over n steps; IR: 50).
 * MINRES reports phibar_k/||b|| (the stopping quantity) as the residual and
 * computes Q from the scalar recurrence of 1^T x_k (R26); with
 * MLMC_FLAG_VERIFY it also carries x_k and reports ||b - A x_k||/||b||, with
 * bit-identical Q (meshes h >= 1/64, the on-chip tile kernel; EINVAL on the
 * finer meshes, whose kernels keep no x_k).                                 */
typedef enum { MLMC_FMT_E4M3 = 0, MLMC_FMT_F16 = 1, MLMC_FMT_F32 = 2, MLMC_FMT_F64 = 3 } mlmc_fmt;
typedef enum { MLMC_SOLVER_MINRES = 0, MLMC_SOLVER_CHOL_IR = 1, MLMC_SOLVER_MGCG = 2, MLMC_SOLVER_CG = 3 } mlmc_solver;

#define MLMC_FLAG_VERIFY 1   /* MINRES: also keep x_k and report the true residual */
#define MLMC_FLAG_ESCALATE 2 /* MINRES / CHOL_IR: a failed solve (max_iter, breakdown, limiting accuracy) is
                                solved again by MG-PCG to the same tolerance; if that converges the sample's
                                status is 4 */
#define MLMC_FLAG_C2F 4      /* on prec_fine, MINRES both halves, fine mesh h = 1/16, 1/32 or 1/64 (NEXT-4,
                                P:97-102, R32): the fine half starts from x0 = P x_c, the P1 interpolation of
                                the coarse half's solution of the same sample (solved first), instead of 0; the
                                stopping rule stays ||b - A x_k|| <= tol ||b|| (phibar_k <= tol ||b||), the
                                reported iterations are the fine half's from x0 */

typedef struct {
    int32_t solver;
    int32_t u_f, u_s, u, u_r;   /* mlmc_fmt codes */
    int32_t max_iter;
    int32_t flags;              /* MLMC_FLAG_* */
} mlmc_precision;

/* ---- per-level accumulators (Algorithm 2 steps 5-6) -------------
 * Layout: MLMC_SUMS_LEN doubles, so a rank-sum is a plain double all-reduce
 * (the two *_max fields need a MAX reduction).
 * cost = deterministic work model (R5): MINRES iters * n per solve; IR
 * n*bw^2*bits(u_f)/64 + steps*4*n*bw per solve; summed over fine + coarse.  */
typedef struct {
    double sum_y, sum_y2;        /* sum_k Y^(k), sum_k (Y^(k))^2 */
    double sum_qf, sum_qc;       /* sum of fine / coarse QoIs */
    double sum_cost;
    double n;                    /* samples accumulated */
    double n_fail;               /* samples with a non-converged / failed solve */
    double iters_f, iters_c;     /* summed MINRES iterations or IR steps */
    double iters_f_max, iters_c_max;
    double n_escalated;          /* samples with a solve repaired by escalation (status 4; not failures) */
} mlmc_level_sums;

/* per-sample record (MLMC_SAMPLE_LEN doubles, sample-major):
 *   [0] Q_f   [1] Q_c (0 at level 0)   [2] iters_f   [3] iters_c
 *   [4] relative residual of the fine solve (MINRES: phibar/||b||, or the true
 *       ||b-Ax||/||b|| with MLMC_FLAG_VERIFY; IR: the true residual)  [5] coarse
 *   [6] status_f  [7] status_c   (0 ok, 1 max_iter, 2 breakdown, 3 non-finite, 4 ok after escalation) */

typedef struct mlmc_ctx mlmc_ctx;   /* opaque */

/* ---- plan ------------------------------------------------------------------
 * mlmc_plan_levels: validate `problem`, compute the KL eigenpairs on the host
 * (1D transcendental equations, R11), and upload each level's synthesis data
 * to the device lazily on first use of the level: the matrix Phi_l[p][k]
 * (2 N_l^2 triangle centroids x m, binary64) where the separable form does not
 * apply (h = 1/8 with K > 16 one-dimensional modes, or K > 32), else the
 * separable form's four N_l x K tables of the 1D functions and the K x K mode
 * map (K = number of 1D modes in use).  Creates its own stream unless
 * one is bound later.  Errors: EINVAL (bad problem), ECUDA (no device).
 * The ctx owns its plan data; free with mlmc_destroy.                        */
int  mlmc_plan_levels(const mlmc_problem* problem, mlmc_ctx** out);
void mlmc_destroy(mlmc_ctx* ctx);
const char* mlmc_strerror(int code);
const char* mlmc_last_error(const mlmc_ctx* ctx);

/* Geometry of mesh level l: N = 1/h, n = (N-1)^2 unknowns, P = 2N^2 triangles,
 * band width bw = N-1.  Errors: EINVAL if l is outside 0..L_max.            */
typedef struct { int32_t N, n, P, bw; double h; } mlmc_level_info;
int mlmc_level_info_get(const mlmc_ctx* ctx, int level, mlmc_level_info* out);

/* Device workspace needed to process `batch` coupled samples of `level` per
 * kernel pass (larger n are processed in passes) with MINRES solves.
 * Host-only.                                                                */
int mlmc_workspace_bytes(const mlmc_ctx* ctx, int level, uint64_t batch, size_t* out);

/* The same for the given fine / coarse precisions (either may be NULL =
 * MINRES): Cholesky-IR solves (K4) also need a factor scratch of one factor
 * per resident warp segment -- it depends on the format and on the device's
 * occupancy, so this query needs the device (ECUDA without one).            */
int mlmc_workspace_bytes_prec(const mlmc_ctx* ctx, int level, uint64_t batch, const mlmc_precision* prec_fine,
                              const mlmc_precision* prec_coarse, size_t* out);

/* Lend the library a device buffer (>= 256-byte aligned) and the cudaStream_t
 * all later work is ordered on (NULL = the legacy default stream; before the
 * first bind the ctx uses a private stream).  The buffer stays borrowed until
 * rebound or mlmc_destroy.  Errors: EINVAL (NULL buffer / misaligned).       */
int mlmc_bind_workspace(mlmc_ctx* ctx, void* dev_ptr, size_t bytes, void* cuda_stream);

/* ---- the hot path -----------------------------------------------------------
 * mlmc_sample_level: for global sample indices first_index .. first_index+n-1
 * of `level`: xi = Philox(seed, level, index) (R12); the KL field on the
 * level-l and level-(l-1) meshes from the SAME xi; P1 assembly
 * (centroid rule, R10); fine solve to tol_fine with prec_fine and
 * coarse solve to tol_coarse with prec_coarse (R8; ignored at level 0); Q =
 * int_D u_h; Y = Q_f - Q_c (Y = Q_f at level 0).
 *   out_sums   host, required: the level's sums over these n samples.
 *   per_sample optional (NULL to skip), host or dev, n * MLMC_SAMPLE_LEN doubles.
 * Synchronises the bound stream before returning.  n = 0 is valid (zero sums).
 * Errors: EINVAL (level, tolerances <= 0 or >= 1 for MINRES, formats),
 * ENOMEM (no / too small workspace for one sample), ECUDA.  A solve failure
 * is NOT an error here: it is counted in n_fail and flagged per sample.      */
int mlmc_sample_level(mlmc_ctx* ctx, int level, uint64_t n, uint64_t seed, uint64_t first_index,
                      const mlmc_precision* prec_fine, const mlmc_precision* prec_coarse,
                      double tol_fine, double tol_coarse,
                      mlmc_level_sums* out_sums, double* per_sample);

/* Same computation, fully asynchronous on the bound stream: sums_dev (dev,
 * MLMC_SUMS_LEN doubles) is overwritten with this call's sums; per_sample_dev
 * optional (dev).  No host synchronisation.                                 */
int mlmc_sample_level_async(mlmc_ctx* ctx, int level, uint64_t n, uint64_t seed, uint64_t first_index,
                            const mlmc_precision* prec_fine, const mlmc_precision* prec_coarse,
                            double tol_fine, double tol_coarse,
                            double* sums_dev, double* per_sample_dev);

/* Several levels in one call (one round of Algorithm 2 step 4 / one fixed-N
 * MLMC pass): entry q processes n[q] samples of levels[q] from first_index[q]
 * with prec_fine[q]/prec_coarse[q] and tol_fine[q]/tol_coarse[q] exactly as
 * mlmc_sample_level would, and writes its sums to sums_dev + q*MLMC_SUMS_LEN
 * (dev).  The levels run concurrently on internal priority streams (largest
 * work first) forked from and joined back into the bound stream; the bound
 * workspace is split between them (each level still processes its samples in
 * passes if its slice is small).  Asynchronous; errors as mlmc_sample_level. */
int mlmc_sample_levels_async(mlmc_ctx* ctx, int nlev, const int* levels, const uint64_t* n, uint64_t seed,
                             const uint64_t* first_index, const mlmc_precision* prec_fine,
                             const mlmc_precision* prec_coarse, const double* tol_fine,
                             const double* tol_coarse, double* sums_dev);

/* Several levels with caller-supplied random inputs, concurrently (the host-buffer path of one fixed-N
 * MLMC step): entry q processes n[q] samples of levels[q] from xi[q] (n[q]*m doubles, host -- pinned
 * makes the copy asynchronous -- or dev) exactly as mlmc_sample_level_xi would; out_sums (host) gets
 * nlev records, per_sample (optional array of nlev pointers, each NULL, host or dev, n[q] *
 * MLMC_SAMPLE_LEN doubles) the per-sample records.  All copies and kernels run on internal streams
 * forked from the bound one; synchronises it once before returning.  Errors as mlmc_sample_level. */
int mlmc_sample_levels_xi(mlmc_ctx* ctx, int nlev, const int* levels, const uint64_t* n, const double* const* xi,
                          const mlmc_precision* prec_fine, const mlmc_precision* prec_coarse, const double* tol_fine,
                          const double* tol_coarse, mlmc_level_sums* out_sums, double* const* per_sample);

/* Caller-supplied random inputs (the SPEC's coupled_sample(l, omega)): exactly
 * mlmc_sample_level, except that xi (n*m doubles, sample-major, host or dev;
 * standard normals, the field's omega = sqrt(sigma2) xi) replaces the Philox
 * draw.  Host xi is copied to the device inside the call (pinned memory makes
 * the copy asynchronous).  Errors as mlmc_sample_level; EINVAL if xi is NULL. */
int mlmc_sample_level_xi(mlmc_ctx* ctx, int level, uint64_t n, const double* xi,
                         const mlmc_precision* prec_fine, const mlmc_precision* prec_coarse,
                         double tol_fine, double tol_coarse,
                         mlmc_level_sums* out_sums, double* per_sample);

/* ---- per-kernel accounting -------------------------------------------------
 * Every kernel the library launches is counted per (kind, mesh N); with
 * profiling on, each launch is also bracketed by CUDA events on the bound
 * stream and its device time accumulated.  mlmc_profile_enable resets the
 * table; mlmc_profile_read synchronises the stream and copies at most `max`
 * entries (count = entries available).                                       */
enum { MLMC_K_RNG = 0, MLMC_K_FIELD = 1, MLMC_K_MINRES = 2, MLMC_K_CHOL_IR = 3, MLMC_K_SUMS = 4,
       MLMC_K_ORDER = 5 /* longest-first job order of a MINRES launch: a kernel of its own only after the
                           P x m field synthesis; the separable field kernel forms it in its last CTA
                           (counted as MLMC_K_FIELD) */ };
typedef struct { int32_t kind; int32_t N; uint64_t launches; double ms; } mlmc_kernel_stat;
int mlmc_profile_enable(mlmc_ctx* ctx, int on);
int mlmc_profile_read(mlmc_ctx* ctx, mlmc_kernel_stat* stats, int max, int* count);

/* ---- Algorithm 2 -------------------------------------------------
 * Cross-rank reduction callback: reduce `count` doubles in place across all
 * ranks (op 0 = SUM, 1 = MAX); return 0 on success.  Called once per round
 * with the per-level sums; with world = 1 it may be NULL.                    */
typedef int (*mlmc_allreduce_fn)(double* buf, int count, int op, void* user);

typedef struct {
    double  k_p;         /* Eq. (16) safety constant (0.05); <= 0 = standard MLMC */
    double  fixed_tol;   /* standard-MLMC solver tolerance (used when k_p <= 0) */
    double  r_bias;      /* the "r" of the bias test, R1: default 1 */
    int32_t N_init;      /* R6: default 100 */
    int32_t policy;      /* 0 = MINRES everywhere (paper-minres), 1 = Table 1 IR quads (paper-ir: hhss /
                            ssss / ssdd on h >= 1/32 where eps_l allows them, else wider; MINRES beyond),
                            3 = auto: per mesh, the fastest admissible solver / precision
                            timed on a pilot batch (see mlmc_auto_choice),
                            2 = MG-PCG on h <= 1/32 and MINRES on h = 1/8, 1/16 (NEXT-4) */
    int32_t rank, world; /* this process's slice of every level's new indices */
    int32_t max_rounds;  /* safety cap (default 100) */
    uint64_t seed;
    int32_t on_fail;     /* a solve that misses its tolerance (max_iter, breakdown; R15): 0 = stop with
                            MLMC_ESOLVER, 1 = keep the sample (Q of the last iterate) and count it in
                            mlmc_result.n_fail, 2 = escalate (MINRES / IR solves carry MLMC_FLAG_ESCALATE: a
                            failed one is solved again by MG-PCG; what still fails is kept and counted as with 1)
                            -- never resampled in any case */
    int32_t reserved0;
} mlmc_adaptive_opts;

typedef struct {
    double   estimate;                   /* Eq. (3): sum_l hat Y_l */
    int32_t  L, rounds, code;            /* code: MLMC_OK or MLMC_ELMAX */
    int32_t  n_fail;                     /* solves that missed their tolerance (kept under on_fail = 1) */
    uint64_t N[MLMC_MAX_LEVELS];         /* samples drawn per level (all ranks) */
    double   eps[MLMC_MAX_LEVELS];       /* eps_l of the last round */
    double   mean[MLMC_MAX_LEVELS];      /* hat Y_l */
    double   var[MLMC_MAX_LEVELS];       /* s_l^2 (Eq. (4), 1/N_l) */
    double   cost[MLMC_MAX_LEVELS];      /* C_l (R5) */
    double   solve_seconds;              /* wall time inside mlmc_sample_level calls */
} mlmc_result;

/* Run Algorithm 2 to RMSE eps (R16: TOL = eps).  Every rank calls this with
 * identical arguments except opts->rank; all ranks return identical results,
 * and the results (estimate, N, mean, var, cost) are bit-identical for any
 * world size: the level sums are exact 256-bit fixed-point totals exchanged
 * through the same all-reduce.
 * Errors: EINVAL, ECUDA, ESOLVER (a failed solve under the abort policy),
 * ELMAX (result still filled).                                              */
int mlmc_adaptive_run(mlmc_ctx* ctx, double eps, const mlmc_adaptive_opts* opts,
                      mlmc_allreduce_fn allreduce, void* user, mlmc_result* out);

/* Policy 3 (auto) of mlmc_adaptive_run: on first use of a mesh the controller times every candidate --
 * MG-PCG, on h >= 1/32 the Cholesky-IR quads the level tolerance admits (q/h/s factors with binary16/32
 * vectors, h/s factors with binary64 vectors), and MINRES last -- on a pilot batch of its own (seed ^ a
 * constant, never part of the estimate; 8..512 samples by mesh size; kernel device time) and keeps the
 * fastest whose pilot solves all converged; MINRES first runs 200 steps and is dropped when they already
 * cost more than the best candidate's solve or their residual decay extrapolates to a slower one; pilot times are summed across ranks so all ranks agree.  A
 * choice is kept in the context per (mesh, tolerance class: >= 1e-3, >= 1e-5, below) for later runs.
 * mlmc_auto_choice returns the latest precision chosen for mesh N (= 1/h) and its pilot cost in device
 * ms per sample.  Errors: EINVAL (no choice made for N).                                                */
int mlmc_auto_choice(const mlmc_ctx* ctx, int N, mlmc_precision* out, double* ms_per_sample);
/* Record a choice for mesh N and tolerance class tol_class (0: tol >= 1e-3, 1: >= 1e-5, 2: below) before a
 * policy-3 run, so that the run does not time pilots: a run driven by recorded choices (e.g. the ones
 * mlmc_auto_choice reported on another box) takes the same decisions everywhere.  ms_per_sample reads -1
 * for a recorded choice.  Errors: EINVAL (N not a mesh of the plan, class out of range, solver not built
 * for N).                                                                                                */
int mlmc_auto_choice_set(mlmc_ctx* ctx, int N, int tol_class, const mlmc_precision* p);

/* The same controller over a caller-supplied host sampler instead of the GPU
 * (CPU tests of Algorithm 2 and of the multi-rank exchange).  The sampler must
 * draw n coupled samples of `level` from global index first_index with the
 * given precisions / tolerances and write MLMC_SUMS_LEN sums; return 0 on
 * success.  Levels 0..L_max, h_l = 1/(h0_inv 2^l).  Host-only.              */
typedef int (*mlmc_level_sampler_fn)(int level, uint64_t n, uint64_t first_index,
                                     const mlmc_precision* prec_fine, const mlmc_precision* prec_coarse,
                                     double tol_fine, double tol_coarse, double* sums, void* user);
int mlmc_adaptive_run_host(int h0_inv, int L_max, double eps, const mlmc_adaptive_opts* opts,
                           mlmc_level_sampler_fn sampler, void* sampler_user,
                           mlmc_allreduce_fn allreduce, void* user, mlmc_result* out);

/* ---- K3d: MINRES of ONE sample over row slabs ----------
 * The finest levels hold few samples (N_L ~ 100) and each
 * is one serial MINRES chain, which sets the critical path of an
 * adaptive run.  K3d solves ONE system -- sample (seed, level, index) on the
 * mesh of `mesh_level` (level or level-1, i.e. the fine or the coarse half) --
 * with the same method and stopping rule as mlmc_sample_level's MINRES (R9,
 * R26, R27), its grid split into row slabs: rank r of `world` owns interior
 * rows j0 <= j < j1 (an even split of 1..N-1, >= 2 rows each) and keeps rows
 * j0-2 .. j1+1 of five binary64 planes in a caller-allocated device workspace.
 * One MINRES step = mlmc_dd_pass, then the CALLER's exchange, then
 * mlmc_dd_scalar:
 *   - all-reduce (SUM, in place, identical result on every rank) of the 3
 *     doubles at byte offset layout.sums_off of the workspace;
 *   - halo rows: mlmc_dd_exchange_rows(layout, step) gives byte offsets of
 *     [send to rank-1, receive from rank-1, send to rank+1, receive from
 *     rank+1] (-1 = no neighbour), each `pitch` doubles; rank r's send to
 *     rank r+1 is rank r+1's receive from rank r.
 * With world = 1 nothing is exchanged and mlmc_dd_run_local runs the solve
 * (chunks of 32 steps as one CUDA graph).  All launches are on the ctx's
 * stream.  Errors: EINVAL (bad level / partition / tolerance), ENOMEM (work-
 * space smaller than layout.bytes), ECUDA.                                     */
typedef struct {
    int32_t N, rank, world, j0, j1, rows, pitch, tiles;
    uint64_t bytes;          /* device workspace bytes (caller allocates, owns) */
    uint64_t plane_off[5];   /* Lanczos vectors P0, P1, P2 (rotating), cE, cN: rows x pitch doubles */
    uint64_t sums_off;       /* 3 doubles: partial sums of the last pass (SUM-all-reduce in place) */
    uint64_t state_off, partials_off, counter_off, rpart_off, xi_off, a_off;   /* internal */
} mlmc_dd_layout;
typedef struct mlmc_dd mlmc_dd;
/* host only: the partition and workspace layout of rank/world on mesh N = 1/h (m KL terms) */
int  mlmc_dd_layout_get(int N, int m, int rank, int world, mlmc_dd_layout* out);
/* host only: the halo rows of the exchange that follows pass `step` (0, 1, ...) */
int  mlmc_dd_exchange_rows(const mlmc_dd_layout* layout, int step, int64_t offs[4]);
/* bind a slab solver to ctx (dev_ws: >= layout.bytes of device memory, borrowed until destroy) */
int  mlmc_dd_create(mlmc_ctx* ctx, int mesh_level, int rank, int world, void* dev_ws, size_t bytes,
                    mlmc_dd** out);
/* field of sample (seed, level, index) on the slab's mesh, planes, state reset (async) */
int  mlmc_dd_begin(mlmc_dd* dd, uint64_t seed, int level, uint64_t index, double tol, int max_iter);
int  mlmc_dd_pass(mlmc_dd* dd);     /* one pass: p_{j+1}, t_{j+1}, partial sums (async; no-op when done) */
int  mlmc_dd_scalar(mlmc_dd* dd);   /* Givens step + stopping test on the reduced sums (async) */
/* synchronous: out = {Q (h^2 1^T x), MINRES iterations, phibar/||b||, status (0 ok, 1 max_iter,
 * 3 non-finite), done (0/1)} -- Q valid once done */
int  mlmc_dd_result(mlmc_dd* dd, double out[5]);
int  mlmc_dd_run_local(mlmc_dd* dd, double out[5]);   /* world = 1: the whole solve, then mlmc_dd_result */
/* The exchange FUSED into the solve kernel over peer memory (world <= 8): the slab tiles store their boundary
 * rows straight into the neighbours' ghost rows, each rank's leader CTA stores its rank partial into every
 * rank's table and bumps every rank's arrival counter (system-scope atomics), and every rank adds the world
 * partials in rank order -- one kernel for the whole solve, no host round trip per step.
 *   mlmc_dd_run_peer: this rank's part; peer_ws[q] = rank q's dd workspace as mapped on THIS device (CUDA IPC /
 *   symmetric memory over NVLink; peer_ws[rank] = its own).  Every rank must call it (the ranks wait on one
 *   another inside the kernel) after every rank's mlmc_dd_begin has completed.  Synchronous.
 *   mlmc_dd_run_emulated: all `world` ranks of one solve whose slab solvers live on this ctx's device
 *   (dds[q] = rank q), in ONE cooperative launch -- the single-GPU test of the same kernel.  Synchronous.
 * out as mlmc_dd_result (every rank holds the same result).  Errors: EINVAL, ECUDA (cooperative launch
 * not possible).                                                                                          */
int  mlmc_dd_run_peer(mlmc_dd* dd, void* const* peer_ws, double out[5]);
int  mlmc_dd_run_emulated(mlmc_dd* const* dds, int world, double out[5]);
/* Peer mapping for mlmc_dd_run_peer (one process per GPU): mlmc_dd_ipc_handle gives a 64-byte CUDA IPC handle
 * of the allocation holding this rank's workspace and the workspace's byte offset in it; a peer process opens
 * it with mlmc_dd_ipc_open (*ptr = the workspace as mapped on the peer's device, *base = the mapping to pass to
 * mlmc_dd_ipc_close).  Errors: EINVAL, ECUDA.                                                              */
int  mlmc_dd_ipc_handle(mlmc_dd* dd, void* handle64, uint64_t* offset);
int  mlmc_dd_ipc_open(mlmc_ctx* ctx, const void* handle64, uint64_t offset, void** ptr, void** base);
int  mlmc_dd_ipc_close(mlmc_ctx* ctx, void* base);
void mlmc_dd_destroy(mlmc_dd* dd);

/* ---- host-only helpers (no device needed; used by the controller) ---------- */
/* Eq. (16): eps[l] = sqrt(k_p) h_l^2 for l < L, eps[L] = k_p h_L^2. */
int mlmc_eps_schedule(int L, double h0, double k_p, double* eps_out);
/* Algorithm 2 step 7, real-valued N_l; C[l] must be > 0.             */
int mlmc_optimal_samples(int nlev, const double* V, const double* C, double tol, double* N_out);
/* The m retained KL modes (R11): 1-based 1D indices ik, jk, eigenvalues lam
 * (descending), and the first `nroots` 1D roots w (w[i-1] for 1D mode i).    */
int mlmc_kl_modes(double sigma2, double corr_len, int m, int32_t* ik, int32_t* jk, double* lam,
                  double* w, int nroots);

/* ---- diagnostics (device) ---------------------------------------------------
 * Run only the field stages for samples first_index.. of `level` on the mesh
 * of level `mesh_level` (level or level-1): xi_dev gets n*m normals, a_dev
 * gets n*2N^2 triangle coefficients a_T (tri 2*(j*N+i) = lower, +1 = upper
 * triangle of cell (i,j)).  Either output may be NULL.  Synchronous.        */
int mlmc_debug_field(mlmc_ctx* ctx, int level, int mesh_level, uint64_t n, uint64_t seed,
                     uint64_t first_index, double* xi_dev, double* a_dev);

/* Job trace of the on-chip MINRES kernels (h >= 1/256), for schedule analysis (tools/step_trace.py): with
 * dev_buf != NULL every system solve started afterwards appends {start, end (globaltimer ns), smid << 32 | N,
 * (cluster rank * 2 + half: 0 fine, 1 coarse) << 32 | job} as 4 uint64 to dev_buf (device, cap records); with dev_buf == NULL the trace is
 * stopped (after a device synchronisation) and *count = records written (may exceed cap).  Only the
 * MLMC_TUNING build records; the production build returns EINVAL.                                   */
int mlmc_debug_trace(mlmc_ctx* ctx, void* dev_buf, uint32_t cap, uint32_t* count);

#ifdef __cplusplus
}
#endif
#endif /* MLMC_H */
