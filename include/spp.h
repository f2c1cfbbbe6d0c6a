/*
 * spp.h -- C ABI of the B200-native solver for singularly perturbed convection-diffusion
 * on Shishkin meshes (hot path of arXiv 2108.13468).
 *
 *   -eps Lap(u) - c . grad(u) + r u = f  on (0,1)^dim,  u = 0 on the boundary
 *   (eq:1D / eq:2D), first-order upwind finite differences (eq:stencil_1d,
 *   P:242-247; 5-point stencil P:964-987) on a (tensor-product) Shishkin mesh (eq:tau 1D,
 *   P:278-284; eq:tau exponential), solved by FGMRES right-
 *   preconditioned with the paper's block preconditioner: 1D eq:block_M; 2D
 *   eq:2D blocks = downstream Gauss-Seidel on I, line solves on
 *   Y and X, full-coarsening multigrid on the corner
 *   (P:1263-1287).
 *
 * Everything runs in sm_100a CUDA kernels in fp64.  No CPU fallback: every entry point that
 * computes returns SPP_E_CUDA if no usable device is present.
 *
 * Conventions
 *   - N ("n" below) = number of mesh intervals per axis; interior unknowns (N-1)^dim.
 *   - Grid functions passed through the ABI are "compact": (N-1)^dim doubles, x fastest,
 *     index (j-1)*(N-1) + (i-1) for node (x_i, y_j), i, j = 1..N-1 (1D: i-1).
 *   - Pointers are host or device (cudaMalloc'd / torch CUDA tensors) as `spp_mem` says.
 *   - Ownership: the caller owns every buffer it passes.  spp_create copies what it needs
 *     into library-owned device memory and keeps no caller pointer.  spp_solve reads f and
 *     writes u_out / res_hist only during the call, on the context's stream, and
 *     synchronises that stream before returning.
 *   - Threading: one context per thread/stream; a context is not thread-safe; there is no
 *     global mutable state except the thread-local error message.
 *   - Errors: status codes only (no exceptions cross the ABI).  Positive = result valid with
 *     a flag set; negative = failure, outputs undefined, spp_last_error() explains.
 */
#ifndef SPP_H
#define SPP_H

#include <stdint.h>

#if defined(__GNUC__)
#define SPP_API __attribute__((visibility("default")))
#else
#define SPP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SPP_OK = 0,
    SPP_NOT_CONVERGED = 1,  /* max_iters reached; last iterate + full history returned */
    SPP_E_ARG = -1,         /* bad argument: N odd/too small, eps not in (0,1], NULL pointer ... */
    SPP_E_MESH = -2,        /* coordinates are not a piecewise-uniform mesh broken at N/2     */
    SPP_E_COEF = -3,        /* c1 <= 0, c2 < 0 or mixed 0/>0 (2D), r < 0, non-finite */
    SPP_E_PIVOT = -4,       /* zero / non-finite Thomas pivot                          */
    SPP_E_MG_CAP = -5,      /* corner MG hit mg_max_cycles in strict mode                      */
    SPP_E_CUDA = -6,        /* CUDA runtime error, or no usable device                         */
    SPP_E_NCCL = -7,        /* NCCL cannot be loaded, a call or the communicator failed, or an
                               exchange did not complete within SPP_NCCL_TIMEOUT_S seconds
                               (default 600): a peer is gone or out of step         */
    SPP_E_NOMEM = -8,       /* device or host allocation failed                                */
    SPP_E_STATE = -9,       /* call not valid in this context state                            */
    SPP_E_NONFINITE = -10   /* NaN/Inf in the Krylov recurrence (beta or a Hessenberg entry):
                               non-finite input data or a preconditioner blow-up (SURVEY 5
                               "NaN/Inf guard on h_{k+1,k}"); outputs undefined               */
} spp_status;

typedef enum { SPP_HOST = 0, SPP_DEVICE = 1 } spp_mem;

typedef enum {
    SPP_STOP_REL_JACOBI = 0, /* ||D^{-1}(f - A u)||_2 <= tol ||D^{-1} f||_2 (recurrence), the
                                BASELINE "relative residual" (reading R11)       */
    SPP_STOP_REL_L2 = 1,     /* ||f - A u||_2 <= tol ||f||_2 (recurrence, unweighted)        */
    SPP_STOP_ABS_L2 = 2,     /* ||f - A u||_2 <= tol (paper 2D: tol = 10 N^{-1} ln N)*/
    SPP_STOP_ABS_MAX = 3     /* true ||f - A u||_inf <= tol (paper 1D: K N^{-1} ln N);
                                1D with side = SPP_LEFT only                                 */
} spp_stop;

typedef enum {
    SPP_RIGHT_FLEXIBLE = 0,  /* FGMRES, right preconditioned, flexible         */
    SPP_LEFT = 1             /* left-preconditioned GMRES, 1D paper mode         */
} spp_side;

typedef struct {
    int32_t dim;             /* 1 or 2                                                       */
    int32_t n;               /* N intervals per axis: even, >= 4 (1D) / >= 8 with N/2 a power
                                of two (2D, full coarsening of the corner)            */
    double eps;              /* perturbation parameter, (0, 1]                               */
    const double *x, *y;     /* HOST node coordinates, N+1 each: x[0]=0, x[N]=1, uniform on
                                [0, x[N/2]] and on [x[N/2], 1] (Shishkin; 2D also
                                any strictly increasing mesh with 0 < x[N/2] <= 1/2, e.g.
                                spp_bakhvalov_mesh); y NULL in 1D.  On a Shishkin mesh the
                                library uses tau = x[N/2] and the formula widths (R12).      */
    const double *c1, *c2, *r; /* coefficient samples at interior nodes (compact layout);
                                c2 NULL in 1D.  Residency per `mem`.  2D: c1 > 0, r >= 0 and
                                either c2 > 0 everywhere (two exponential layers) or c2 = 0
                                everywhere (one parabolic layer along y = 0; the
                                corner then runs the semi-coarsening Galerkin multigrid of
                                P:1192-1261, whose paper tolerance is mg_reduction = 1e-2, and
                                the y mesh wants tau_y = sigma sqrt(eps) ln N, eq:tau
                                parabolic: spp_shishkin_mesh(N, sqrt(eps), sigma, 1)); a
                                mixture is SPP_E_COEF.  Row strips support c2 > 0 only.     */
    spp_mem mem;
} spp_problem;

typedef struct {
    spp_side side;
    spp_stop stop;
    double tol;
    int32_t max_iters;       /* Arnoldi steps (default 200)                           */
    int32_t restart;         /* 0 = no restart (the paper); m > 0 = FGMRES(m), 2D only:
                                after m steps x += sum y_j z_j and the next cycle starts from
                                the true residual, the stop target staying the initial one
                                (reading R23); max_iters counts all steps          */
    double mg_reduction;     /* corner MG relative reduction of ||S_0 rho||_2 (1e-3) */
    int32_t mg_max_cycles;   /* cycle cap (20)                                        */
    int32_t mg_fixed_cycles; /* 0 = adaptive (paper); > 0 = exactly this many (parity mode)  */
    int32_t mg_coarsest;     /* coarsen until <= this many points per axis (4)        */
    int32_t fixed_iters;     /* 0 = run to tolerance; > 0 = exactly this many Arnoldi steps  */
    int32_t mg_strict;       /* 1 = return SPP_E_MG_CAP when the cap is hit                  */
    int32_t reserved[7];
} spp_options;

typedef struct {
    int32_t iters;           /* Arnoldi steps = preconditioner applications         */
    int32_t converged;
    int32_t mg_cycles_total, mg_cycles_min, mg_cycles_max, mg_cap_hits, applies;
    int32_t kernel_launches; /* CUDA kernels launched by this call                           */
    double res0, res_final;  /* monitored residual (per `stop`) at start / end               */
    double true_res_l2_rel;     /* ||f - A u||_2 / ||f||_2 after the solve                   */
    double true_res_jacobi_rel; /* ||D^{-1}(f - A u)||_2 / ||D^{-1} f||_2                    */
    double setup_s, solve_s;    /* device time of the last spp_setup / this spp_solve        */
} spp_stats;

typedef struct spp_ctx spp_ctx;

/* Defaults: right/flexible, SPP_STOP_REL_JACOBI, tol 1e-8, 200 iterations, MG 1e-3 / 20 /
 * adaptive / coarsest 4.
 * Option validation (spp_create, spp_create_dist, spp_batch1d_create return SPP_E_ARG):
 * restart < 0, restart > 0 in 1D, in row strips or with fixed_iters > 0; 2D with side = SPP_LEFT
 * or stop = SPP_STOP_ABS_MAX; 1D with exactly one of
 * side = SPP_LEFT / stop = SPP_STOP_ABS_MAX (the left GMRES of P:828-833 always stops on the
 * true max-norm residual, and that stop exists only there); tol <= 0 or not finite. */
SPP_API void spp_default_options(int32_t dim, spp_options *o);

/* Shishkin mesh on the host (eq:tau 1D P:278-284 / eq:tau exponential P:914-928):
 * tau = min(1/2, sigma*eps*ln(n)/beta); n/2 uniform intervals on [0,tau] and on [tau,1].
 * x_out: n+1 doubles (host).  SPP_E_ARG for odd n < 4, eps not in (0,1], sigma/beta <= 0. */
SPP_API spp_status spp_shishkin_mesh(int32_t n, double eps, double sigma, double beta, double *x_out);

/* Bakhvalov-Shishkin graded mesh on the host (reading R21): the
 * graded layer-adapted mesh of Remark rem:not just S-meshes with the transition point
 * at index n/2: x_i = -(sigma eps/beta) ln(1 - 2(1 - 1/n) i/n) for i <= n/2, uniform
 * on [tau, 1], tau = sigma eps ln(n)/beta (the Shishkin transition point); tau > 1/2: the uniform
 * mesh i/n.  Same arguments and errors as spp_shishkin_mesh.  2D problems accept this (or any
 * strictly increasing mesh with x[0] = 0, x[n] = 1, 0 < x[n/2] <= 1/2): the operator then uses
 * the coordinate differences as widths and the corner multigrid geometric interpolation weights;
 * 1D problems need the Shishkin mesh (SPP_E_MESH otherwise). */
SPP_API spp_status spp_bakhvalov_mesh(int32_t n, double eps, double sigma, double beta, double *x_out);

/* Validate the problem, allocate the device workspace on `cuda_stream` (NULL = legacy default
 * stream) and run the setup (coefficients, corner multigrid levels, line factorisations;
 * counted in time-to-solution as the paper does). */
SPP_API spp_status spp_create(const spp_problem *p, const spp_options *o, void *cuda_stream, spp_ctx **out);

/* Re-run the setup for new coefficient samples on the same mesh (c2 NULL in 1D). */
SPP_API spp_status spp_setup(spp_ctx *c, const double *c1, const double *c2, const double *r, spp_mem mem);

/* Solve A u = f.  f, u_out: compact grid functions with residency `mem`.  res_hist (host,
 * may be NULL) receives the monitored residual, iters+1 entries truncated at res_hist_cap.
 * st (host, may be NULL).  Returns SPP_OK, SPP_NOT_CONVERGED or an error. */
SPP_API spp_status spp_solve(spp_ctx *c, const double *f, double *u_out, spp_mem mem,
                     double *res_hist, int32_t res_hist_cap, spp_stats *st);

/* Test hooks (per-kernel parity with the oracle).  in/out are DEVICE pointers in the compact
 * layout of the stage:  global grid (N-1)^2 for MATVEC, PRECOND, MII, MYY, MXX;
 * corner block (N/2)^2 for CORNER_SOLVE, and level-l corner grids (n_l)^2 for GS_SWEEP,
 * VCYCLE, RESTRICT (in: level l, out: level l+1), PROLONG_ADD (in: level l+1, out: level l,
 * accumulated), LEVEL_RESIDUAL (in: [b | e] stacked, out: rho).
 *   MATVEC     out = A in (unweighted, difference form)
 *   PRECOND    out = M^{-1} in                      (cycles_out: corner MG cycles)
 *   MII        out = in with region I replaced by M_II^{-1} in_I
 *   MYY / MXX  out = in with region Y / X replaced by its line solves, using `out`'s current
 *              values as the already-solved neighbours (call MII first; out is in/out)
 *   CORNER_RHS out (corner, (N/2)^2) = b_C built from in (global) and out's X/Y neighbours --
 *              in is the stacked pair [q | z] (2*(N-1)^2)
 *   GS_SWEEP   out = one downstream GS sweep of A_l e = b from e = out, b = in
 *   VCYCLE     out = V(1,1) cycle on level l for rhs in, zero initial guess
 *   CORNER_SOLVE out = M_CC^{-1} in (adaptive cycles; cycles_out).
 * Hooks that drive exactly the kernels and arguments of the BASELINE-mode solve:
 *   MII_JACOBI out = in with region I replaced by M_II^{-1} (D in): the z-form chained sweep the
 *              Jacobi-weighted FGMRES runs (its preconditioner input is D v, reading R11)
 *   POST_SMOOTH  level l: in = [b | e | e_c] stacked (n_l^2, n_l^2, n_{l+1}^2); out = one GS sweep
 *              of A_l x = b from x0 = e + P e_c (the fused prolongation + right-hand-side kernel
 *              and the sweep of the V-cycle's post-smoothing, with b stored as b/D as there)
 *   RESID_RESTRICT level l: in = [R | e] stacked; out (level l+1) = S^{-1} P^T S (R - A_l e) / D_{l+1},
 *              the general residual-restriction kernel with the V-cycle's z-form scalings (R read
 *              as R/D, the coarse right-hand side stored divided by its diagonal)
 *   PRE_RESTRICT level l: in = R; out (level l+1) = S^{-1} P^T S (R - A_l e) / D_{l+1} with e = one
 *              downstream GS sweep of A_l e = R from zero: the V-cycle's pre-smoothing followed by
 *              its residual-restriction, which forms R - A_l e as aW e_W + aS e_S (P:1205-1209,
 *              P:1276-1280) */
typedef enum {
    SPP_STAGE_MATVEC = 0, SPP_STAGE_MII = 1, SPP_STAGE_MYY = 2, SPP_STAGE_MXX = 3,
    SPP_STAGE_CORNER_RHS = 4, SPP_STAGE_GS_SWEEP = 5, SPP_STAGE_VCYCLE = 6,
    SPP_STAGE_CORNER_SOLVE = 7, SPP_STAGE_PRECOND = 8, SPP_STAGE_RESTRICT = 9,
    SPP_STAGE_PROLONG_ADD = 10, SPP_STAGE_LEVEL_RESIDUAL = 11, SPP_STAGE_MII_JACOBI = 12,
    SPP_STAGE_POST_SMOOTH = 13, SPP_STAGE_RESID_RESTRICT = 14, SPP_STAGE_PRE_RESTRICT = 15
} spp_stage;
SPP_API spp_status spp_apply_stage(spp_ctx *c, spp_stage s, int32_t level, const double *in, double *out,
                           int32_t *cycles_out);

/* Total CUDA kernels launched by this context since spp_create (setup + solves + hooks). */
SPP_API int64_t spp_kernel_launches(const spp_ctx *c);

/* Number of corner MG levels and the unknowns per axis of level l. */
SPP_API int32_t spp_mg_levels(const spp_ctx *c);
SPP_API int32_t spp_mg_level_n(const spp_ctx *c, int32_t l);

/* Per-kernel-class device timing (CUDA events on the context stream).  enable != 0 records
 * events around every launch of the listed classes during subsequent spp_solve calls.
 * spp_profile_get returns, for class k, the launch count, total milliseconds and the
 * algorithmic bytes moved accumulated since the last reset.
 * Classes: 0 spmv, 1 sweep_I, 2 lines_XY, 3 mg_sweep (tiled GS sweeps of the corner levels),
 * 4 mg_resid_restrict, 5 mg_prolong (GS right-hand side + prolongation), 6 mg_update,
 * 7 krylov_vec (MGS and vector ops), 8 setup, 9 other, 10 mg_coarse (fused coarse V-cycle),
 * 11 exchange (row strips: the copies / NCCL group of one exchange step, on the strip's stream). */
#define SPP_PROF_CLASSES 12
SPP_API spp_status spp_profile_enable(spp_ctx *c, int32_t enable);
SPP_API spp_status spp_profile_reset(spp_ctx *c);
SPP_API spp_status spp_profile_get(const spp_ctx *c, int32_t k, int64_t *launches, double *ms, double *bytes);
SPP_API const char *spp_profile_name(int32_t k);

SPP_API void spp_destroy(spp_ctx *c);

/* ---- Batched 1D solves (the 1D method of P:375-386 / P:828-833) ----
 * nprob independent problems -eps_p u'' - c_p u' + r_p u = f_p on their own Shishkin meshes,
 * each solved exactly as a single spp_create(dim=1)/spp_solve would (same kernels' setup and
 * Krylov body, one CTA per problem; results are bitwise those of the single solve), with one
 * set of options for the whole batch.
 *   n, eps     host, nprob entries: N_p (even, 4 <= N_p <= 8192) and eps_p in (0,1].
 *   x          host, concatenated meshes: problem p's N_p+1 coordinates start at
 *              sum_{q<p} (N_q+1); each is validated as in spp_create (SPP_E_MESH).
 *   c, r       concatenated interior samples with residency `mem`: problem p's N_p-1 values
 *              start at sum_{q<p} (N_q-1) (the same layout for f and u below).  Copied at
 *              create; SPP_E_COEF names the first problem with c <= 0 or r < 0.
 *   o          options shared by every problem (NULL = spp_default_options(1)); max_iters <= 512.
 * spp_batch1d_solve: f, u_out concatenated as c; iters_out, converged_out, res_out (host, may be
 * NULL; nprob entries) receive each problem's iterations, convergence flag and final monitored
 * residual.  st (may be NULL): iters = max over problems, applies = sum, converged = all,
 * setup_s / solve_s device times.  Returns SPP_OK if every problem converged, else
 * SPP_NOT_CONVERGED (results still valid).  Errors at create leave *out NULL and are reported
 * by spp_last_error(NULL); errors at solve by spp_batch1d_last_error(b).
 * spp_batch1d_setup: re-run the setup for new c, r (same layout and residency rules as at
 * create) on the same problems and meshes, reusing the device workspace. */
typedef struct spp_batch1d spp_batch1d;
SPP_API spp_status spp_batch1d_create(int32_t nprob, const int32_t *n, const double *eps, const double *x,
                              const double *c, const double *r, spp_mem mem, const spp_options *o,
                              void *cuda_stream, spp_batch1d **out);
SPP_API spp_status spp_batch1d_setup(spp_batch1d *b, const double *c, const double *r, spp_mem mem);
SPP_API spp_status spp_batch1d_solve(spp_batch1d *b, const double *f, double *u_out, spp_mem mem,
                             int32_t *iters_out, int32_t *converged_out, double *res_out, spp_stats *st);
SPP_API int32_t spp_batch1d_nprob(const spp_batch1d *b);
SPP_API int64_t spp_batch1d_launches(const spp_batch1d *b);
SPP_API const char *spp_batch1d_last_error(const spp_batch1d *b);
SPP_API void spp_batch1d_destroy(spp_batch1d *b);

/* ---- Row strips across GPUs --------------------------------------
 * A 2D problem split into row strips: strip r owns the interior rows [J[r], J[r+1]) of every grid
 * function (J[0] = 1, J[P] = N), with one strip boundary at row N/2+1 (the X/I | C/Y split of
 * eq:2D blocks).  The solve computes the same method as spp_create/spp_solve (same
 * iterations and corner cycles; results equal to rounding): halos of one row for
 * the stencil, the certified warm-up / smoothing halos of the strip above for the line chains
 * and the corner multigrid strips, the exact M_II sweep relayed strip to strip, the vertical
 * M_YY lines solved as column blocks, and every dot product as all-gathered per-strip partial
 * sums.  spp_setup / spp_solve / spp_destroy take a strip context like any other;
 * spp_apply_stage returns SPP_E_STATE for it.
 *
 * spp_strip_partition: the default J (host, nranks+1 entries): ceil(P/2) strips share rows
 *   1..N/2 and the others rows N/2+1..N-1, evenly.  SPP_E_ARG if they do not fit.
 * spp_create_strips: nstrips strips of a whole problem on the calling device with a loopback
 *   transport (device copies between the strips' buffers): the decomposition's own test and
 *   validation mode.  p and spp_solve's f / u are whole ((N-1)^2 compact).  nstrips = 1 is
 *   spp_create.
 * spp_create_dist: one strip per process (one GPU each), NCCL over `nccl_comm` (an ncclComm_t of
 *   nranks ranks, rank = this process; see spp_nccl_*).  local->c1, c2, r and spp_solve's f / u
 *   hold this rank's rows j0 .. j1-1 only ((j1-j0)(N-1) compact values, row j0 first); x, y are
 *   the whole meshes.  Every rank must pass its own [j0, j1): they must tile 1..N-1 in rank order
 *   with a boundary at N/2+1 (SPP_E_ARG otherwise).  Collective: every rank calls it, and every
 *   later spp_setup / spp_solve, in the same order.  The caller keeps the communicator alive
 *   until spp_destroy.  SPP_E_NCCL if NCCL cannot be loaded or fails.
 * spp_nccl_unique_id / spp_nccl_comm_create / spp_nccl_comm_destroy: an NCCL communicator for
 *   spp_create_dist (rank 0 makes the 128-byte id, the caller broadcasts it, every rank
 *   creates).  NCCL is loaded at run time (SPP_NCCL_LIB, else the libnccl.so.2 in the process).
 * spp_dist_info: ranks, corner levels smoothed on strips, and the transfers / bytes / exchange
 *   steps this rank took part in since create (1, 0, 0 ... for a one-GPU context).
 * spp_dist_plan: host-only exchange schedule of one FGMRES iteration for a synthetic geometry
 *   (partition j, D strip levels of certified halo `halo`, line warm-up `warm`): 11 int64 per
 *   block (step, src, dst, role, slot, src offset, dst offset, width, rows, pitch, 0) for the
 *   blocks `rank` sends or receives (rank < 0: all), at most cap written; returns the count or
 *   SPP_E_ARG.  For testing the multi-process orchestration without GPUs. */
SPP_API spp_status spp_strip_partition(int32_t n, int32_t nranks, int32_t *j);
SPP_API spp_status spp_create_strips(const spp_problem *p, int32_t nstrips, const spp_options *o, void *cuda_stream,
                                     spp_ctx **out);
SPP_API spp_status spp_create_dist(const spp_problem *local, int32_t j0, int32_t j1, void *nccl_comm, int32_t rank,
                                   int32_t nranks, const spp_options *o, void *cuda_stream, spp_ctx **out);
SPP_API spp_status spp_nccl_unique_id(uint8_t *id);
SPP_API spp_status spp_nccl_comm_create(const uint8_t *id, int32_t nranks, int32_t rank, void **comm);
SPP_API void spp_nccl_comm_destroy(void *comm);
SPP_API spp_status spp_dist_info(const spp_ctx *c, int32_t *nranks, int32_t *strip_levels, int64_t *xfers,
                                 double *bytes, int64_t *exchanges);
SPP_API int32_t spp_dist_plan(int32_t n, int32_t nranks, const int32_t *j, int32_t d_levels, int32_t halo, int32_t warm,
                              int32_t rank, int64_t *out, int32_t cap);

/* Last error message for this context (or the thread-local one when c == NULL). */
SPP_API const char *spp_last_error(const spp_ctx *c);

/* Library version string. */
SPP_API const char *spp_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPP_H */
