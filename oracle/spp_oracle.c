/*
 * spp_oracle.c -- plain, slow, single-threaded fp64 CPU ORACLE for the hot path of
 * arXiv 2108.13468 (MacLachlan, Madden, Nhan: "A boundary-layer preconditioner for
 * singularly perturbed convection diffusion").
 *
 * *** TEST INFRASTRUCTURE ONLY. ***  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.  The product
 * path (paper_2108_13468_b200/) never links, imports or executes anything here, and this
 * file shares no code, header, table or helper with the CUDA path.
 *
 * Citation key:  P:a-b = /root/reference/PAPER.md lines a..b (section / equation named
 * next to it);  S:a-b = SPEC.md lines;  "reading Rk" = DESIGN.md section "Readings".
 *
 * Every routine follows the paper step by step, in its order and notation; no blocking,
 * fusion or reordering.  Compiled with -O2 -ffp-contract=off (no FMA contraction).
 *
 * Parity pins (tests/test_oracle_*.py, all `-m "not gpu"`):
 *   mesh ............ closed-form tau, piecewise uniformity
 *   operator 1D/2D .. M-matrix sign pattern, A*1 = r exactly (difference form), uniform-mesh
 *                     stencil of P:349-351, dense brute force (numpy) on N<=16,
 *                     Table 1 to 4 digits, Table 6 to 4 digits,
 *                     first-order convergence to the cfg2 manufactured solution
 *   precond 1D ...... Theorem block_fact unit eigenvectors; eigen band;
 *                     Table 2 iteration counts exactly
 *   precond 2D ...... equals a dense solve with M-hat built from A by the block rules of
 *                     eq:2D blocks [corner solved to 1e-14]; N-hat >= 0
 *                     (P:1120-1124); Table 7 iteration counts exactly;
 *                     5 corner V-cycles per apply
 *   corner MG ....... converges to the dense A_CC^{-1} b (numpy); Galerkin-free check that
 *                     level 0 equals A_CC (reading R8); linearity of the V-cycle
 *   FGMRES .......... A = I converges in 1 step; Arnoldi orthonormality; recurrence residual
 *                     equals the true Jacobi-weighted residual
 *   O1 direct ....... banded LU vs numpy dense solve on tiny meshes
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_NOT_CONVERGED 1
#define ORC_E_ARG (-1)
#define ORC_E_PIVOT (-4)
#define ORC_E_NOMEM (-8)
#define ORC_E_NONFINITE (-10)   /* NaN/Inf beta or Hessenberg entry (SURVEY 5 NaN/Inf guard) */

/* ===================================================================================== */
/*  Mesh                                                                                 */
/* ===================================================================================== */

/* Shishkin mesh, eq:tau 1D and eq:tau exponential:
 *   tau = min(1/2, sigma*eps*ln(N)/beta),  N/2 uniform intervals on [0,tau] and on [tau,1].
 * The paper's 1D choice is sigma=2, beta=C_lower; its 2D choice sigma=5/2;
 * BASELINE uses sigma=2, beta=1 (B:7-11).  x has N+1 entries. */
int orc_mesh(int N, double eps, double sigma, double beta, double *x)
{
    if (N < 4 || (N % 2) != 0 || !(eps > 0.0) || eps > 1.0 || !(sigma > 0.0) || !(beta > 0.0))
        return ORC_E_ARG;
    double tau = sigma * eps * log((double)N) / beta;
    if (tau > 0.5) tau = 0.5;
    int n = N / 2;
    double h = tau / n, H = (1.0 - tau) / n;
    for (int i = 0; i < n; i++) x[i] = i * h;
    x[n] = tau;
    for (int i = n + 1; i < N; i++) x[i] = tau + (i - n) * H;
    x[N] = 1.0;
    return ORC_OK;
}

/* Bakhvalov-Shishkin mesh (reading R21): the graded layer-adapted mesh the
 * paper's Remark rem:not just S-meshes names ("graded (e.g., Bakhvalov) meshes"),
 * with the transition point at index N/2 that the block preconditioner needs:
 *   x_i = -(sigma eps / beta) ln(1 - 2 (1 - 1/N) i / N),  i = 0 .. N/2   (graded layer),
 *   x_i = tau + (i - N/2) (1 - tau) / (N/2),               i = N/2 .. N   (uniform),
 * tau = x_{N/2} = sigma eps ln(N) / beta, the Shishkin transition point.  tau > 1/2: the
 * uniform mesh x_i = i/N (no layer to resolve). */
int orc_mesh_bs(int N, double eps, double sigma, double beta, double *x)
{
    if (N < 4 || (N % 2) != 0 || !(eps > 0.0) || eps > 1.0 || !(sigma > 0.0) || !(beta > 0.0))
        return ORC_E_ARG;
    int n = N / 2;
    double s = sigma * eps / beta;
    double tau = s * log((double)N);
    if (tau > 0.5) {
        for (int i = 0; i <= N; i++) x[i] = (double)i / N;
        x[N] = 1.0;
        return ORC_OK;
    }
    x[0] = 0.0;
    for (int i = 1; i < n; i++) x[i] = -s * log(1.0 - 2.0 * (1.0 - 1.0 / N) * i / N);
    x[n] = tau;
    double H = (1.0 - tau) / n;
    for (int i = n + 1; i < N; i++) x[i] = tau + (i - n) * H;
    x[N] = 1.0;
    return ORC_OK;
}

/* 1 if x is the piecewise-uniform (Shishkin) mesh broken at N/2, to rounding. */
static int mesh_is_shishkin(const double *x, int N)
{
    int n = N / 2;
    double t = x[n], h = t / n, H = (1.0 - t) / n;
    for (int i = 0; i <= N; i++) {
        double want = i <= n ? i * h : t + (i - n) * H;
        if (fabs(x[i] - want) > 1e-12 * (fabs(want) + h)) return 0;
    }
    return 1;
}

/* Mesh width h_i = x_i - x_{i-1} on the piecewise-uniform mesh, evaluated
 * from the formula tau/(N/2) resp. (1-tau)/(N/2) with tau = x_{N/2} (reading R12:
 * formula, not coordinate differences).  Valid for i = 1..N. */
static double mesh_h(const double *x, int N, int i)
{
    int n = N / 2;
    double tau = x[n];
    return (i <= n) ? tau / n : (1.0 - tau) / n;
}

/* Width h_i for the 2D operator: the Shishkin formula (reading R12) on a piecewise-uniform mesh;
 * on any other (graded) mesh the coordinate differences h_i = x_i - x_{i-1} of P:964-968. */
static double mesh_w(const double *x, int N, int i, int graded)
{
    return graded ? x[i] - x[i - 1] : mesh_h(x, N, i);
}

/* ===================================================================================== */
/*  Dense-ish helpers                                                                    */
/* ===================================================================================== */

static double dot(size_t n, const double *a, const double *b)
{
    double s = 0.0;
    for (size_t i = 0; i < n; i++) s += a[i] * b[i];
    return s;
}

/* Thomas algorithm without pivoting ("Thomas' algorithm"; safe for these
 * diagonally dominant M-matrices, Lemma diag_dom).  Row k:
 *   lo[k]*x[k-1] + di[k]*x[k] + up[k]*x[k+1] = rhs[k],  k = 0..m-1 (lo[0], up[m-1] unused). */
int orc_thomas(int m, const double *lo, const double *di, const double *up,
               const double *rhs, double *x)
{
    double *cp = (double *)malloc(sizeof(double) * (size_t)(m > 0 ? m : 1));
    if (!cp) return ORC_E_NOMEM;
    double den = di[0];
    if (!(den != 0.0) || !isfinite(den)) { free(cp); return ORC_E_PIVOT; }
    cp[0] = (m > 1) ? up[0] / den : 0.0;
    x[0] = rhs[0] / den;
    for (int k = 1; k < m; k++) {
        den = di[k] - lo[k] * cp[k - 1];
        if (!(den != 0.0) || !isfinite(den)) { free(cp); return ORC_E_PIVOT; }
        cp[k] = (k < m - 1) ? up[k] / den : 0.0;
        x[k] = (rhs[k] - lo[k] * x[k - 1]) / den;
    }
    for (int k = m - 2; k >= 0; k--) x[k] -= cp[k] * x[k + 1];
    free(cp);
    return ORC_OK;
}

/* ===================================================================================== */
/*  1D problem: -eps u'' - c u' + r u = f, u(0)=u(1)=0   (eq:1D)                 */
/* ===================================================================================== */

/* Upwind stencil eq:stencil_1d at node i = 1..N-1 (array index i-1):
 *   [ -eps/(h_i hb_i),  eps/hb_i (1/h_i + 1/h_{i+1}) + c_i/h_{i+1} + r_i,
 *     -eps/(h_{i+1} hb_i) - c_i/h_{i+1} ]
 * stored in difference form (reading R12): aW = eps/(hb_i h_i), aE = eps/(hb_i h_{i+1}) +
 * c_i/h_{i+1}, diagonal D = (aW + aE) + r. */
void orc1_coef(int N, double eps, const double *x, const double *c, const double *r,
               double *aW, double *aE, double *D)
{
    for (int i = 1; i <= N - 1; i++) {
        double hi = mesh_h(x, N, i), hi1 = mesh_h(x, N, i + 1);
        double hb = 0.5 * (hi + hi1);
        aW[i - 1] = eps / (hb * hi);
        aE[i - 1] = eps / (hb * hi1) + c[i - 1] / hi1;
        D[i - 1] = (aW[i - 1] + aE[i - 1]) + r[i - 1];
    }
}

/* y = A u in difference form: (Au)_i = aW_i (u_i - u_{i-1}) + aE_i (u_i - u_{i+1}) + r_i u_i,
 * u_0 = u_N = 0 (homogeneous Dirichlet). */
void orc1_matvec(int N, const double *aW, const double *aE, const double *r,
                 const double *u, double *y)
{
    int m = N - 1;
    for (int k = 0; k < m; k++) {
        double uw = (k > 0) ? u[k - 1] : 0.0, ue = (k < m - 1) ? u[k + 1] : 0.0;
        y[k] = aW[k] * (u[k] - uw) + aE[k] * (u[k] - ue) + r[k] * u[k];
    }
}

/* Exact discrete solution U^E = A^{-1} f (O1): Thomas on the assembled tridiagonal, then
 * difference-form iterative refinement x <- x + A^{-1}(f - A_diff x). */
int orc1_direct(int N, const double *aW, const double *aE, const double *D, const double *r,
                const double *f, double *u)
{
    int m = N - 1;
    double *lo = malloc(sizeof(double) * m), *up = malloc(sizeof(double) * m);
    double *res = malloc(sizeof(double) * m), *cor = malloc(sizeof(double) * m);
    if (!lo || !up || !res || !cor) { free(lo); free(up); free(res); free(cor); return ORC_E_NOMEM; }
    for (int k = 0; k < m; k++) { lo[k] = -aW[k]; up[k] = -aE[k]; }
    int st = orc_thomas(m, lo, D, up, f, u);
    for (int it = 0; it < 8 && st == ORC_OK; it++) {
        orc1_matvec(N, aW, aE, r, u, res);
        for (int k = 0; k < m; k++) res[k] = f[k] - res[k];
        st = orc_thomas(m, lo, D, up, res, cor);
        for (int k = 0; k < m; k++) u[k] += cor[k];
    }
    free(lo); free(up); free(res); free(cor);
    return st;
}

/* Preconditioner eq:block_M: M = A with A_II replaced by its upper-triangular
 * part, i.e. the sub-diagonal entries zeroed in rows N_L+2 .. N-1, N_L = N/2 (the transition
 * point is in L; row N_L+1 keeps A_IL).  M z = q is one
 * Thomas solve. */
int orc1_precond(int N, const double *aW, const double *aE, const double *D,
                 const double *q, double *z)
{
    int m = N - 1, NL = N / 2;
    double *lo = malloc(sizeof(double) * m), *up = malloc(sizeof(double) * m);
    if (!lo || !up) { free(lo); free(up); return ORC_E_NOMEM; }
    for (int i = 1; i <= m; i++) {
        lo[i - 1] = (i >= NL + 2) ? 0.0 : -aW[i - 1];
        up[i - 1] = -aE[i - 1];
    }
    int st = orc_thomas(m, lo, D, up, q, z);
    free(lo); free(up);
    return st;
}

/* ===================================================================================== */
/*  Generic Krylov drivers (operator + preconditioner callbacks)                          */
/* ===================================================================================== */

typedef struct {
    size_t n;
    void *ctx;
    void (*A)(void *ctx, const double *x, double *y);     /* y = A x (unweighted)         */
    int (*Minv)(void *ctx, const double *q, double *z);    /* z = M^{-1} q                 */
    const double *D;                                       /* diagonal of A (Jacobi weight)*/
} orc_sys;

typedef struct {
    int iters, converged, breakdown, status;
    double res0, res_final;
} orc_kstats;

static void apply_givens(double *h, double *cs, double *sn, double *g, int k)
{
    for (int i = 0; i < k; i++) {
        double t = cs[i] * h[i] + sn[i] * h[i + 1];
        h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
        h[i] = t;
    }
    double den = hypot(h[k], h[k + 1]);
    if (den == 0.0) { cs[k] = 1.0; sn[k] = 0.0; }
    else { cs[k] = h[k] / den; sn[k] = h[k + 1] / den; }
    h[k] = den;
    h[k + 1] = 0.0;
    g[k + 1] = -sn[k] * g[k];
    g[k] = cs[k] * g[k];
}

/* Flexible GMRES (Saad 2003, cited P:1306-1308), right-preconditioned, modified
 * Gram-Schmidt, x0 = 0.  restart = 0: no restart (the paper, "no restarts" P:831);
 * restart = m > 0: FGMRES(m) (SURVEY 8(b) `restart`, reading R23): after m Arnoldi steps without
 * convergence the iterate is formed, x <- x + sum_j y_j z_j, and the process restarts from the
 * true residual r = W (f - A x) (Saad 2003, the restarted Algorithm 9.6), the stopping target
 * staying the one of the initial residual.  With restart >= the steps taken, every operation is
 * the unrestarted one.
 *   weighted = 1 (BASELINE mode, reading R11): run on (W A) x = W f with W = D^{-1}; the
 *     preconditioner for W A is (W M)^{-1} = M^{-1} D, so z_k = M^{-1}(D v_k).
 *   weighted = 0 (paper mode): plain A x = f, z_k = M^{-1} v_k.
 *   stop_abs = 0: |g_{k+1}| <= tol * beta (relative);  stop_abs = 1: |g_{k+1}| <= tol
 *     (the paper's ||R|| <= 10 N^{-1} ln N, Euclidean).
 *   fixed_iters > 0: run exactly that many Arnoldi steps in total (parity mode, reading R17).
 * hist[0] = beta, hist[k+1] = |g_{k+1}| of the k-th step overall (recurrence residual, S:534;
 * after a restart the recurrence starts from the true residual of the restart). */
int orc_fgmres_r(const orc_sys *s, const double *f, double *x, int weighted, int stop_abs,
                 double tol, int maxit, int fixed_iters, int restart, double *hist, int hist_cap,
                 orc_kstats *st)
{
    size_t n = s->n;
    memset(st, 0, sizeof(*st));
    const int mr = (restart > 0 && restart < maxit) ? restart : maxit;   /* steps per cycle */
    double **V = calloc((size_t)mr + 1, sizeof(double *));
    double **Z = calloc((size_t)mr + 1, sizeof(double *));
    double *H = calloc((size_t)(mr + 1) * (mr + 1), sizeof(double)); /* column k at H + k*(mr+1) */
    double *cs = calloc((size_t)mr + 1, sizeof(double)), *sn = calloc((size_t)mr + 1, sizeof(double));
    double *g = calloc((size_t)mr + 2, sizeof(double)), *y = calloc((size_t)mr + 1, sizeof(double));
    double *q = malloc(sizeof(double) * n), *w = malloc(sizeof(double) * n);
    if (!V || !Z || !H || !cs || !sn || !g || !y || !q || !w) { st->status = ORC_E_NOMEM; goto done; }
    int ld = mr + 1;

    V[0] = malloc(sizeof(double) * n);
    if (!V[0]) { st->status = ORC_E_NOMEM; goto done; }
    for (size_t i = 0; i < n; i++) V[0][i] = weighted ? f[i] / s->D[i] : f[i];
    double beta = sqrt(dot(n, V[0], V[0]));
    st->res0 = beta;
    if (!isfinite(beta)) { st->status = ORC_E_NONFINITE; goto done; }
    if (hist_cap > 0) hist[0] = beta;
    memset(x, 0, sizeof(double) * n);
    if (beta == 0.0) { st->converged = 1; st->res_final = 0.0; goto done; }
    double target = stop_abs ? tol : tol * beta;
    int total = 0;                                  /* Arnoldi steps over all cycles */
    for (;;) {                                      /* restart cycles (one when restart = 0) */
        for (size_t i = 0; i < n; i++) V[0][i] /= beta;
        memset(g, 0, sizeof(double) * ((size_t)mr + 2));
        g[0] = beta;
        int k, stop = 0;
        for (k = 0; k < mr && total < maxit; k++) {
            /* z_k = M^{-1}(s v_k) */
            for (size_t i = 0; i < n; i++) q[i] = weighted ? s->D[i] * V[k][i] : V[k][i];
            if (!Z[k]) Z[k] = malloc(sizeof(double) * n);
            if (!Z[k]) { st->status = ORC_E_NOMEM; goto done; }
            int ps = s->Minv(s->ctx, q, Z[k]);
            if (ps < 0) { st->status = ps; goto done; }
            /* w = W A z_k */
            s->A(s->ctx, Z[k], w);
            if (weighted) for (size_t i = 0; i < n; i++) w[i] /= s->D[i];
            /* modified Gram-Schmidt ("modified Gram-Schmidt and Arnoldi steps") */
            double *h = H + (size_t)k * ld;
            for (int j = 0; j <= k; j++) {
                h[j] = dot(n, w, V[j]);
                for (size_t i = 0; i < n; i++) w[i] -= h[j] * V[j][i];
            }
            h[k + 1] = sqrt(dot(n, w, w));
            if (!V[k + 1]) V[k + 1] = malloc(sizeof(double) * n);
            if (!V[k + 1]) { st->status = ORC_E_NOMEM; goto done; }
            /* SURVEY 5 "NaN/Inf guard on h_{k+1,k}": a non-finite entry is a failure, and only an
             * exact zero h_{k+1,k} is a (happy) breakdown */
            for (int j = 0; j <= k + 1; j++) if (!isfinite(h[j])) { st->status = ORC_E_NONFINITE; goto done; }
            int brk = h[k + 1] == 0.0;
            for (size_t i = 0; i < n; i++) V[k + 1][i] = brk ? 0.0 : w[i] / h[k + 1];
            apply_givens(h, cs, sn, g, k);
            double res = fabs(g[k + 1]);
            total++;
            if (total < hist_cap) hist[total] = res;
            st->iters = total;
            st->res_final = res;
            if (brk) { st->breakdown = 1; st->converged = (res <= target); stop = 1; k++; break; }
            if (fixed_iters > 0) { if (total >= fixed_iters) { st->converged = (res <= target); stop = 1; k++; break; } }
            else if (res <= target) { st->converged = 1; stop = 1; k++; break; }
        }
        /* solve the k x k upper-triangular system R y = g, then x += sum_j y_j z_j */
        int kk = k;
        for (int i = kk - 1; i >= 0; i--) {
            double t = g[i];
            for (int j = i + 1; j < kk; j++) t -= H[(size_t)j * ld + i] * y[j];
            y[i] = t / H[(size_t)i * ld + i];
        }
        for (int j = 0; j < kk; j++)
            for (size_t i = 0; i < n; i++) x[i] += y[j] * Z[j][i];
        if (stop || total >= maxit) break;
        /* restart from the true residual v_0 = W (f - A x) */
        s->A(s->ctx, x, w);
        for (size_t i = 0; i < n; i++) V[0][i] = weighted ? (f[i] - w[i]) / s->D[i] : f[i] - w[i];
        beta = sqrt(dot(n, V[0], V[0]));
        if (!isfinite(beta)) { st->status = ORC_E_NONFINITE; goto done; }
        if (beta == 0.0) { st->converged = 1; st->res_final = 0.0; break; }
    }
    st->status = st->converged ? ORC_OK : ORC_NOT_CONVERGED;
done:
    if (V) for (int j = 0; j <= mr; j++) free(V[j]);
    if (Z) for (int j = 0; j <= mr; j++) free(Z[j]);
    free(V); free(Z); free(H); free(cs); free(sn); free(g); free(y); free(q); free(w);
    return st->status;
}

int orc_fgmres(const orc_sys *s, const double *f, double *x, int weighted, int stop_abs,
               double tol, int maxit, int fixed_iters, double *hist, int hist_cap,
               orc_kstats *st)
{
    return orc_fgmres_r(s, f, x, weighted, stop_abs, tol, maxit, fixed_iters, 0, hist, hist_cap, st);
}

/* Left-preconditioned GMRES for the 1D paper experiments (MATLAB gmres, "modified
 * slightly to implement the stopping criterion, and with no restarts"; reading R10):
 * Arnoldi (MGS) on M^{-1}A starting from M^{-1}b, x0 = 0; after every step the iterate x_k is
 * formed and the TRUE residual is tested, ||b - A x_k||_inf <= tol (tol = K N^{-1} ln N,
 * P:812).  hist[k] = ||b - A x_k||_inf. */
int orc_gmres_left(const orc_sys *s, const double *b, double *x, double tol, int maxit,
                   double *hist, int hist_cap, orc_kstats *st)
{
    size_t n = s->n;
    memset(st, 0, sizeof(*st));
    int ld = maxit + 1;
    double **V = calloc((size_t)maxit + 2, sizeof(double *));
    double *H = calloc((size_t)(maxit + 1) * (maxit + 1), sizeof(double));
    double *cs = calloc((size_t)maxit + 1, sizeof(double)), *sn = calloc((size_t)maxit + 1, sizeof(double));
    double *g = calloc((size_t)maxit + 2, sizeof(double)), *y = calloc((size_t)maxit + 1, sizeof(double));
    double *w = malloc(sizeof(double) * n), *t = malloc(sizeof(double) * n);
    if (!V || !H || !cs || !sn || !g || !y || !w || !t) { st->status = ORC_E_NOMEM; goto done; }
    memset(x, 0, sizeof(double) * n);
    /* initial true residual = b (x0 = 0) */
    double r0 = 0.0;
    for (size_t i = 0; i < n; i++) r0 = fmax(r0, fabs(b[i]));
    st->res0 = r0;
    if (hist_cap > 0) hist[0] = r0;
    if (r0 <= tol) { st->converged = 1; st->res_final = r0; goto done; }
    V[0] = malloc(sizeof(double) * n);
    if (!V[0]) { st->status = ORC_E_NOMEM; goto done; }
    int ps = s->Minv(s->ctx, b, V[0]);
    if (ps < 0) { st->status = ps; goto done; }
    double beta = sqrt(dot(n, V[0], V[0]));
    for (size_t i = 0; i < n; i++) V[0][i] /= beta;
    g[0] = beta;
    for (int k = 0; k < maxit; k++) {
        s->A(s->ctx, V[k], t);
        ps = s->Minv(s->ctx, t, w);
        if (ps < 0) { st->status = ps; goto done; }
        double *h = H + (size_t)k * ld;
        for (int j = 0; j <= k; j++) {
            h[j] = dot(n, w, V[j]);
            for (size_t i = 0; i < n; i++) w[i] -= h[j] * V[j][i];
        }
        h[k + 1] = sqrt(dot(n, w, w));
        V[k + 1] = malloc(sizeof(double) * n);
        if (!V[k + 1]) { st->status = ORC_E_NOMEM; goto done; }
        int brk = !(h[k + 1] > 0.0);
        for (size_t i = 0; i < n; i++) V[k + 1][i] = brk ? 0.0 : w[i] / h[k + 1];
        apply_givens(h, cs, sn, g, k);
        int kk = k + 1;
        for (int i = kk - 1; i >= 0; i--) {
            double tt = g[i];
            for (int j = i + 1; j < kk; j++) tt -= H[(size_t)j * ld + i] * y[j];
            y[i] = tt / H[(size_t)i * ld + i];
        }
        memset(x, 0, sizeof(double) * n);
        for (int j = 0; j < kk; j++)
            for (size_t i = 0; i < n; i++) x[i] += y[j] * V[j][i];
        s->A(s->ctx, x, t);
        double rinf = 0.0;
        for (size_t i = 0; i < n; i++) rinf = fmax(rinf, fabs(b[i] - t[i]));
        if (kk < hist_cap) hist[kk] = rinf;
        st->iters = kk;
        st->res_final = rinf;
        if (rinf <= tol || brk) { st->converged = (rinf <= tol); st->breakdown = brk; break; }
    }
    st->status = st->converged ? ORC_OK : ORC_NOT_CONVERGED;
done:
    if (V) for (int j = 0; j <= maxit + 1; j++) free(V[j]);
    free(V); free(H); free(cs); free(sn); free(g); free(y); free(w); free(t);
    return st->status;
}

/* ----- 1D solver entry point ----- */
typedef struct { int N; const double *aW, *aE, *r, *D; } ctx1d;
static void cb1_A(void *c, const double *x, double *y)
{
    ctx1d *k = (ctx1d *)c;
    orc1_matvec(k->N, k->aW, k->aE, k->r, x, y);
}
static int cb1_M(void *c, const double *q, double *z)
{
    ctx1d *k = (ctx1d *)c;
    return orc1_precond(k->N, k->aW, k->aE, k->D, q, z);
}

/* side: 0 = right/flexible (FGMRES), 1 = left (paper 1D mode, true inf-norm residual).
 * weighted/stop_abs as orc_fgmres (ignored for side 1).  iters etc. in out[0..4]:
 * out_i[0]=iters, [1]=converged;  out_d[0]=res0, [1]=res_final. */
int orc1_solve(int N, double eps, const double *x, const double *c, const double *r,
               const double *f, int side, int weighted, int stop_abs, double tol, int maxit,
               int fixed_iters, double *u, double *hist, int hist_cap, int *out_i, double *out_d)
{
    int m = N - 1;
    double *aW = malloc(sizeof(double) * m), *aE = malloc(sizeof(double) * m), *D = malloc(sizeof(double) * m);
    if (!aW || !aE || !D) { free(aW); free(aE); free(D); return ORC_E_NOMEM; }
    orc1_coef(N, eps, x, c, r, aW, aE, D);
    ctx1d k = {N, aW, aE, r, D};
    orc_sys s = {(size_t)m, &k, cb1_A, cb1_M, D};
    orc_kstats st;
    int rc = (side == 1) ? orc_gmres_left(&s, f, u, tol, maxit, hist, hist_cap, &st)
                         : orc_fgmres(&s, f, u, weighted, stop_abs, tol, maxit, fixed_iters, hist, hist_cap, &st);
    out_i[0] = st.iters; out_i[1] = st.converged;
    out_d[0] = st.res0; out_d[1] = st.res_final;
    free(aW); free(aE); free(D);
    return rc;
}

/* ===================================================================================== */
/*  2D problem: -eps Lap u - c.grad u + r u = f on (0,1)^2, u = 0 on the boundary        */
/*  (eq:2D), tensor Shishkin mesh, two exponential layers (c1, c2 > 0).         */
/* ===================================================================================== */

/* One multigrid level of the corner block. */
typedef struct {
    int nl;                     /* unknowns per axis                                       */
    double *aW, *aS;            /* [nl+2], index m = 1..nl                                  */
    double *aE, *aN, *rr, *D;   /* [nl*nl], idx (l-1)*nl + (m-1)                           */
    double *hb, *kb;            /* [nl+2]: hbar_m, kbar_l -> S_l = diag(hbar_m kbar_l)     */
    double *e, *rho, *b;        /* work vectors [nl*nl]                                    */
    /* [nl+2]: geometric interpolation weights of an odd node q of this level from the next
     * coarser level's nodes at its left / right (x) and below / above (y): the linear
     * interpolant on this level's 1D meshes; 1/2 on a uniform corner */
    double *wxl, *wxr, *wyl, *wyr;
} orc_level;

/* One level of the semi-coarsening Galerkin multigrid for the corner when the layer along y = 0
 * is parabolic (c2 = 0). */
typedef struct {
    int nx, ny;                 /* unknowns in x (halved per level) and y (n on every level)  */
    double *a;                  /* [nx*ny*9] stencil: a[p*9 + (dj+1)*3 + (di+1)] is the entry of
                                   row (i,j) at column (i+di, j+dj); 0 outside the block        */
    double *wW, *wE;            /* [nx*ny] interpolation weights of an odd-x node from the coarse
                                   nodes at x_{i-1} and x_{i+1} (operator-induced) */
    double *e, *rho, *b;        /* work [nx*ny]                                                */
} orc_plev;

typedef struct {
    int N, n, m;                /* N intervals; n = N/2 (corner size); m = N-1              */
    int gx, gy;                 /* graded (non-Shishkin) mesh in x / y: widths from coordinates */
    int par;                    /* c2 = 0: one parabolic + one exponential layer */
    int PL;                     /* parabolic corner: levels of the semi-coarsening hierarchy  */
    orc_plev pl[24];
    double eps;
    double *aW, *aS;            /* [N+1], index 1..N-1                                      */
    double *aE, *aN, *rr, *D;   /* [m*m], idx (j-1)*m + (i-1)                              */
    int L;                      /* number of MG levels (0..L-1); level L-1 is coarsest     */
    orc_level lev[24];
    double mg_red;              /* 1e-3                                            */
    int mg_cap, mg_fixed;       /* 20; fixed-cycle parity mode (reading R17)       */
    /* statistics of the last solve */
    long mg_cycles_total;
    int mg_min, mg_max, mg_cap_hits, applies;
    int *cycle_log; int cycle_log_cap;
    double *bC, *zC;            /* corner work [n*n]                                       */
} orc2d;

#define IX(i, j, m) ((size_t)((j) - 1) * (size_t)(m) + (size_t)((i) - 1))

static inline double at2(const double *u, int m, int i, int j)
{
    return (i < 1 || j < 1 || i > m || j > m) ? 0.0 : u[IX(i, j, m)];
}

/* 5-point upwind stencil in difference form (reading R12):
 *   aW_i  = eps/(hbar_i h_i)                      aS_j  = eps/(kbar_j k_j)
 *   aE_ij = eps/(hbar_i h_{i+1}) + c1_ij/h_{i+1}  aN_ij = eps/(kbar_j k_{j+1}) + c2_ij/k_{j+1}
 *   D_ij  = ((aW + aE) + (aS + aN)) + r_ij
 * (the paper's centre entry equals D; its off-diagonals are -aW, -aE, -aS, -aN). */
static void orc2_coef(orc2d *P, const double *x, const double *y, const double *c1,
                      const double *c2, const double *r)
{
    int N = P->N, m = P->m;
    double eps = P->eps;
    int gx = P->gx, gy = P->gy;
    for (int i = 1; i <= m; i++) {
        double hi = mesh_w(x, N, i, gx), hi1 = mesh_w(x, N, i + 1, gx), hb = 0.5 * (hi + hi1);
        P->aW[i] = eps / (hb * hi);
        double kj = mesh_w(y, N, i, gy), kj1 = mesh_w(y, N, i + 1, gy), kb = 0.5 * (kj + kj1);
        P->aS[i] = eps / (kb * kj);
    }
    for (int j = 1; j <= m; j++) {
        double kj = mesh_w(y, N, j, gy), kj1 = mesh_w(y, N, j + 1, gy), kb = 0.5 * (kj + kj1);
        for (int i = 1; i <= m; i++) {
            double hi = mesh_w(x, N, i, gx), hi1 = mesh_w(x, N, i + 1, gx), hb = 0.5 * (hi + hi1);
            size_t p = IX(i, j, m);
            P->aE[p] = eps / (hb * hi1) + c1[p] / hi1;
            P->aN[p] = eps / (kb * kj1) + c2[p] / kj1;
            P->rr[p] = r[p];
            P->D[p] = ((P->aW[i] + P->aE[p]) + (P->aS[j] + P->aN[p])) + r[p];
        }
    }
}

/* y = A u, difference form, zero Dirichlet values outside (reading R12). */
void orc2_matvec_raw(const orc2d *P, const double *u, double *y)
{
    int m = P->m;
    for (int j = 1; j <= m; j++)
        for (int i = 1; i <= m; i++) {
            size_t p = IX(i, j, m);
            double c = u[p];
            y[p] = P->aW[i] * (c - at2(u, m, i - 1, j)) + P->aE[p] * (c - at2(u, m, i + 1, j))
                 + P->aS[j] * (c - at2(u, m, i, j - 1)) + P->aN[p] * (c - at2(u, m, i, j + 1))
                 + P->rr[p] * c;
        }
}

/* ----- corner multigrid ----- */

/* Level l keeps every 2^l-th layer node of the corner, plus the corner boundary nodes
 * x_0 and x_{n+1} (reading R8), and re-discretises ("rediscretization") with the same
 * stencil formula on that 1D mesh: widths 2^l * tau/(N/2) inside the corner and the first
 * coarse width (1-tau)/(N/2) for the last interval; c1, c2, r sampled at the coarse nodes.
 * On a graded mesh (NEXT-4) the level's 1D mesh is X_q = x_{q 2^l} (q = 0..nl), X_{nl+1} =
 * x_{n+1}, and the widths are its coordinate differences. */
/* the level's 1D widths w[q] = X_q - X_{q-1}, q = 1 .. nl+1 */
static void level_widths(const double *x, int N, int l, int graded, double *w)
{
    int n = N / 2, step = 1 << l, nl = n >> l;
    if (!graded) {
        double h = step * (x[n] / n), H = (1.0 - x[n]) / n;
        for (int q = 1; q <= nl; q++) w[q] = h;
        w[nl + 1] = H;
        return;
    }
    for (int q = 1; q <= nl; q++) w[q] = x[q * step] - x[(q - 1) * step];
    w[nl + 1] = x[n + 1] - x[n];
}
static int build_level(orc2d *P, int l, const double *x, const double *y, const double *c1,
                       const double *c2, const double *r)
{
    orc_level *Lv = &P->lev[l];
    int N = P->N, n = P->n, step = 1 << l, nl = n >> l;
    Lv->nl = nl;
    size_t nn = (size_t)nl * nl;
    Lv->aW = calloc(nl + 2, sizeof(double)); Lv->aS = calloc(nl + 2, sizeof(double));
    Lv->hb = calloc(nl + 2, sizeof(double)); Lv->kb = calloc(nl + 2, sizeof(double));
    Lv->aE = malloc(nn * sizeof(double)); Lv->aN = malloc(nn * sizeof(double));
    Lv->rr = malloc(nn * sizeof(double)); Lv->D = malloc(nn * sizeof(double));
    Lv->e = malloc(nn * sizeof(double)); Lv->rho = malloc(nn * sizeof(double));
    Lv->b = malloc(nn * sizeof(double));
    if (!Lv->aW || !Lv->aS || !Lv->hb || !Lv->kb || !Lv->aE || !Lv->aN || !Lv->rr || !Lv->D ||
        !Lv->e || !Lv->rho || !Lv->b) return ORC_E_NOMEM;
    Lv->wxl = calloc(nl + 2, sizeof(double)); Lv->wxr = calloc(nl + 2, sizeof(double));
    Lv->wyl = calloc(nl + 2, sizeof(double)); Lv->wyr = calloc(nl + 2, sizeof(double));
    double *wx = calloc(nl + 2, sizeof(double)), *wy = calloc(nl + 2, sizeof(double));
    if (!Lv->wxl || !Lv->wxr || !Lv->wyl || !Lv->wyr || !wx || !wy) { free(wx); free(wy); return ORC_E_NOMEM; }
    level_widths(x, N, l, P->gx, wx);                       /* level widths, x axis */
    level_widths(y, N, l, P->gy, wy);                       /* level widths, y axis */
    /* odd node q lies between this level's nodes q-1 and q+1, the coarser level's (q-1)/2 and
     * (q+1)/2: linear interpolation weights from the widths (exactly 1/2 when they are equal) */
    for (int q = 1; q < nl; q += 2) {
        double a = wx[q], b = wx[q + 1];
        Lv->wxl[q] = a == b ? 0.5 : b / (a + b); Lv->wxr[q] = a == b ? 0.5 : a / (a + b);
        a = wy[q]; b = wy[q + 1];
        Lv->wyl[q] = a == b ? 0.5 : b / (a + b); Lv->wyr[q] = a == b ? 0.5 : a / (a + b);
    }
    double eps = P->eps;
    for (int q = 1; q <= nl; q++) {
        double h = wx[q], h1 = wx[q + 1], hb = 0.5 * (h + h1);
        double k = wy[q], k1 = wy[q + 1], kb = 0.5 * (k + k1);
        Lv->aW[q] = eps / (hb * h);  Lv->hb[q] = hb;
        Lv->aS[q] = eps / (kb * k);  Lv->kb[q] = kb;
    }
    for (int lq = 1; lq <= nl; lq++) {
        double k1 = wy[lq + 1], kb = Lv->kb[lq];
        for (int q = 1; q <= nl; q++) {
            double h1 = wx[q + 1], hb = Lv->hb[q];
            size_t g = IX(q * step, lq * step, P->m), p = IX(q, lq, nl);
            Lv->aE[p] = eps / (hb * h1) + c1[g] / h1;
            Lv->aN[p] = eps / (kb * k1) + c2[g] / k1;
            Lv->rr[p] = r[g];
            Lv->D[p] = ((Lv->aW[q] + Lv->aE[p]) + (Lv->aS[lq] + Lv->aN[p])) + r[g];
        }
    }
    free(wx); free(wy);
    (void)N;
    return ORC_OK;
}

/* One downstream point Gauss-Seidel sweep: from the top-right
 * point of the block to the bottom-left, i.e. j descending, i descending; E and N neighbours
 * already updated, W and S old.  In place on e. */
static void mg_gs(const orc_level *Lv, const double *b, double *e)
{
    int nl = Lv->nl;
    for (int j = nl; j >= 1; j--)
        for (int i = nl; i >= 1; i--) {
            size_t p = IX(i, j, nl);
            e[p] = (b[p] + Lv->aW[i] * at2(e, nl, i - 1, j) + Lv->aS[j] * at2(e, nl, i, j - 1)
                         + Lv->aE[p] * at2(e, nl, i + 1, j) + Lv->aN[p] * at2(e, nl, i, j + 1)) / Lv->D[p];
        }
}

/* rho = b - A_l e (difference form). */
static void mg_residual(const orc_level *Lv, const double *b, const double *e, double *rho)
{
    int nl = Lv->nl;
    for (int j = 1; j <= nl; j++)
        for (int i = 1; i <= nl; i++) {
            size_t p = IX(i, j, nl);
            double c = e[p];
            double Ae = Lv->aW[i] * (c - at2(e, nl, i - 1, j)) + Lv->aE[p] * (c - at2(e, nl, i + 1, j))
                      + Lv->aS[j] * (c - at2(e, nl, i, j - 1)) + Lv->aN[p] * (c - at2(e, nl, i, j + 1))
                      + Lv->rr[p] * c;
            rho[p] = b[p] - Ae;
        }
}

/* 1D linear interpolation parents of fine node i: an even node 2I is a coarse
 * node (weight 1); an odd node 2I+1 lies between coarse nodes I and I+1 (weights wl[i], wr[i]:
 * 1/2 each on a uniform corner).  Coarse node 0 is the Dirichlet boundary and is skipped. */
static int parents(int i, int *I, double *w, const double *wl, const double *wr)
{
    if ((i & 1) == 0) { I[0] = i / 2; w[0] = 1.0; return 1; }
    int c = 0;
    if ((i - 1) / 2 >= 1) { I[c] = (i - 1) / 2; w[c] = wl[i]; c++; }
    I[c] = (i + 1) / 2; w[c] = wr[i]; c++;
    return c;
}

/* b_{l+1} = S_{l+1}^{-1} P^T S_l rho_l  (FE rescaling by hbar_i kbar_j, then the
 * transpose of bilinear interpolation as restriction). */
static void mg_restrict(const orc_level *F, const orc_level *C, const double *rho, double *bc)
{
    int nf = F->nl, nc = C->nl;
    memset(bc, 0, sizeof(double) * (size_t)nc * nc);
    for (int j = 1; j <= nf; j++)
        for (int i = 1; i <= nf; i++) {
            int Ii[2], Jj[2]; double wi[2], wj[2];
            int ni = parents(i, Ii, wi, F->wxl, F->wxr), nj = parents(j, Jj, wj, F->wyl, F->wyr);
            double sr = (F->hb[i] * F->kb[j]) * rho[IX(i, j, nf)];
            for (int a = 0; a < ni; a++)
                for (int c = 0; c < nj; c++)
                    bc[IX(Ii[a], Jj[c], nc)] += wi[a] * wj[c] * sr;
        }
    for (int J = 1; J <= nc; J++)
        for (int I = 1; I <= nc; I++)
            bc[IX(I, J, nc)] /= (C->hb[I] * C->kb[J]);
}

/* e_l += P e_{l+1}  (bilinear interpolation). */
static void mg_prolong_add(const orc_level *F, const orc_level *C, const double *ec, double *e)
{
    int nf = F->nl, nc = C->nl;
    for (int j = 1; j <= nf; j++)
        for (int i = 1; i <= nf; i++) {
            int Ii[2], Jj[2]; double wi[2], wj[2];
            int ni = parents(i, Ii, wi, F->wxl, F->wxr), nj = parents(j, Jj, wj, F->wyl, F->wyr);
            double s = 0.0;
            for (int a = 0; a < ni; a++)
                for (int c = 0; c < nj; c++) s += wi[a] * wj[c] * ec[IX(Ii[a], Jj[c], nc)];
            e[IX(i, j, nf)] += s;
        }
}

/* V(1,1) cycle on level l for A_l e = b, zero initial guess ("standard V(1,1)
 * cycling strategy", coarsest grid "four sweeps of the downstream Gauss-Seidel relaxation").
 * Result in Lv->e. */
static void mg_vcycle(orc2d *P, int l, const double *b)
{
    orc_level *Lv = &P->lev[l];
    size_t nn = (size_t)Lv->nl * Lv->nl;
    memset(Lv->e, 0, nn * sizeof(double));
    if (l == P->L - 1) {
        for (int s = 0; s < 4; s++) mg_gs(Lv, b, Lv->e);
        return;
    }
    orc_level *Cv = &P->lev[l + 1];
    mg_gs(Lv, b, Lv->e);                         /* pre-smoothing  */
    mg_residual(Lv, b, Lv->e, Lv->rho);
    mg_restrict(Lv, Cv, Lv->rho, Cv->b);
    mg_vcycle(P, l + 1, Cv->b);                  /* coarse correction (result in Cv->e) */
    mg_prolong_add(Lv, Cv, Cv->e, Lv->e);
    mg_gs(Lv, b, Lv->e);                         /* post-smoothing */
}

static double fe_norm(const orc_level *Lv, const double *v)
{
    int nl = Lv->nl;
    double s = 0.0;
    for (int j = 1; j <= nl; j++)
        for (int i = 1; i <= nl; i++) {
            double t = (Lv->hb[i] * Lv->kb[j]) * v[IX(i, j, nl)];
            s += t * t;
        }
    return sqrt(s);
}

/* ----- corner multigrid, one parabolic and one exponential layer (c2 = 0) -----
 * Semi-coarsening: factor-2 coarsening in x only, y kept.  The finest operator is A_CC with row
 * (i,j) multiplied by hbar_i kbar_j (FE scaling); interpolation to fine node (i,j)
 * (odd i) from the coarse nodes at x_{i-1}, x_{i+1} with the weights of the stencil collapsed in
 * the North-South direction:
 *   wW = -(a_{(i,j),(i-1,j-1)} + a_{(i,j),(i-1,j)} + a_{(i,j),(i-1,j+1)}) / (a_{(i,j),(i,j-1)} + a_{(i,j),(i,j)} + a_{(i,j),(i,j+1)})
 *   wE = the same with the (i+1) column;
 * an even fine node is a coarse node (weight 1); restriction = interpolation^T;
 * coarse operators by the Galerkin triple product R A P, nine-point on coarse
 * grids; downstream point Gauss-Seidel (top-right to bottom-left), V(1,1), four sweeps on the
 * coarsest grid; the coarsest has <= 4 points in x (reading R7). */
#define PST(L, p, di, dj) ((L)->a[(size_t)(p) * 9 + ((dj) + 1) * 3 + ((di) + 1)])

static double pl_at(const orc_plev *L, const double *u, int i, int j)
{
    return (i < 1 || j < 1 || i > L->nx || j > L->ny) ? 0.0 : u[(size_t)(j - 1) * L->nx + (i - 1)];
}

/* interpolation weights of level L from its (next coarser) level */
static void pl_weights(orc_plev *L)
{
    for (int j = 1; j <= L->ny; j++)
        for (int i = 1; i <= L->nx; i++) {
            size_t p = (size_t)(j - 1) * L->nx + (i - 1);
            L->wW[p] = L->wE[p] = 0.0;
            if ((i & 1) == 0) continue;
            double den = PST(L, p, 0, -1) + PST(L, p, 0, 0) + PST(L, p, 0, 1);
            L->wW[p] = -(PST(L, p, -1, -1) + PST(L, p, -1, 0) + PST(L, p, -1, 1)) / den;
            L->wE[p] = -(PST(L, p, 1, -1) + PST(L, p, 1, 0) + PST(L, p, 1, 1)) / den;
        }
}

/* interpolation weight P_{(i,j),(I,j)} of fine node i from coarse node I (0 if not a parent) */
static double pl_P(const orc_plev *F, int i, int j, int I)
{
    size_t p = (size_t)(j - 1) * F->nx + (i - 1);
    if ((i & 1) == 0) return I == i / 2 ? 1.0 : 0.0;
    if (I == (i - 1) / 2) return I >= 1 ? F->wW[p] : 0.0;
    if (I == (i + 1) / 2) return F->wE[p];
    return 0.0;
}

/* C = P^T F P (Galerkin), row by row of the fine operator */
static void pl_galerkin(const orc_plev *F, orc_plev *C)
{
    memset(C->a, 0, sizeof(double) * (size_t)C->nx * C->ny * 9);
    for (int j = 1; j <= F->ny; j++)
        for (int i = 1; i <= F->nx; i++) {
            size_t p = (size_t)(j - 1) * F->nx + (i - 1);
            for (int I = (i - 1) / 2; I <= (i + 1) / 2; I++) {
                if (I < 1 || I > C->nx) continue;
                double wi = pl_P(F, i, j, I);
                if (wi == 0.0) continue;
                for (int dj = -1; dj <= 1; dj++)
                    for (int di = -1; di <= 1; di++) {
                        double a = PST(F, p, di, dj);
                        if (a == 0.0) continue;
                        int i2 = i + di, j2 = j + dj;
                        for (int I2 = (i2 - 1) / 2; I2 <= (i2 + 1) / 2; I2++) {
                            if (I2 < 1 || I2 > C->nx || i2 < 1 || i2 > F->nx) continue;
                            double w2 = pl_P(F, i2, j2, I2);
                            if (w2 == 0.0) continue;
                            size_t q = (size_t)(j - 1) * C->nx + (I - 1);
                            PST(C, q, I2 - I, dj) += wi * a * w2;
                        }
                    }
            }
        }
}

/* downstream point Gauss-Seidel sweep (j descending, i descending), in place */
static void pl_gs(const orc_plev *L, const double *b, double *e)
{
    for (int j = L->ny; j >= 1; j--)
        for (int i = L->nx; i >= 1; i--) {
            size_t p = (size_t)(j - 1) * L->nx + (i - 1);
            double s = b[p];
            for (int dj = -1; dj <= 1; dj++)
                for (int di = -1; di <= 1; di++)
                    if (di || dj) s -= PST(L, p, di, dj) * pl_at(L, e, i + di, j + dj);
            e[p] = s / PST(L, p, 0, 0);
        }
}

static void pl_residual(const orc_plev *L, const double *b, const double *e, double *rho)
{
    for (int j = 1; j <= L->ny; j++)
        for (int i = 1; i <= L->nx; i++) {
            size_t p = (size_t)(j - 1) * L->nx + (i - 1);
            double s = 0.0;
            for (int dj = -1; dj <= 1; dj++)
                for (int di = -1; di <= 1; di++) s += PST(L, p, di, dj) * pl_at(L, e, i + di, j + dj);
            rho[p] = b[p] - s;
        }
}

static void pl_restrict(const orc_plev *F, const orc_plev *C, const double *r, double *bc)
{
    for (int j = 1; j <= C->ny; j++)
        for (int I = 1; I <= C->nx; I++) {
            double s = 0.0;
            for (int i = 2 * I - 1; i <= 2 * I + 1; i++)
                if (i <= F->nx) s += pl_P(F, i, j, I) * r[(size_t)(j - 1) * F->nx + (i - 1)];
            bc[(size_t)(j - 1) * C->nx + (I - 1)] = s;
        }
}

static void pl_prolong_add(const orc_plev *F, const orc_plev *C, const double *ec, double *e)
{
    for (int j = 1; j <= F->ny; j++)
        for (int i = 1; i <= F->nx; i++) {
            double s = 0.0;
            for (int I = (i - 1) / 2; I <= (i + 1) / 2; I++)
                if (I >= 1 && I <= C->nx) s += pl_P(F, i, j, I) * ec[(size_t)(j - 1) * C->nx + (I - 1)];
            e[(size_t)(j - 1) * F->nx + (i - 1)] += s;
        }
}

static void pl_vcycle(orc2d *P, int l, const double *b)
{
    orc_plev *L = &P->pl[l];
    size_t nn = (size_t)L->nx * L->ny;
    memset(L->e, 0, nn * sizeof(double));
    if (l == P->PL - 1) {
        for (int s = 0; s < 4; s++) pl_gs(L, b, L->e);
        return;
    }
    orc_plev *C = &P->pl[l + 1];
    pl_gs(L, b, L->e);
    pl_residual(L, b, L->e, L->rho);
    pl_restrict(L, C, L->rho, C->b);
    pl_vcycle(P, l + 1, C->b);
    pl_prolong_add(L, C, C->e, L->e);
    pl_gs(L, b, L->e);
}

/* the hierarchy, from the corner block of the (level-0) coefficients */
static int pl_build(orc2d *P)
{
    const orc_level *L0 = &P->lev[0];
    int n = P->n, nx = n, l = 0;
    for (;;) {
        orc_plev *L = &P->pl[l];
        L->nx = nx; L->ny = n;
        size_t nn = (size_t)nx * n;
        L->a = calloc(nn * 9, sizeof(double));
        L->wW = calloc(nn, sizeof(double)); L->wE = calloc(nn, sizeof(double));
        L->e = calloc(nn, sizeof(double)); L->rho = calloc(nn, sizeof(double)); L->b = calloc(nn, sizeof(double));
        if (!L->a || !L->wW || !L->wE || !L->e || !L->rho || !L->b) { P->PL = l + 1; return ORC_E_NOMEM; }
        if (l == 0) {
            for (int j = 1; j <= n; j++)
                for (int i = 1; i <= n; i++) {
                    size_t p = IX(i, j, n);
                    double S = L0->hb[i] * L0->kb[j];                /* FE row scaling */
                    PST(L, p, 0, 0) = S * L0->D[p];
                    if (i > 1) PST(L, p, -1, 0) = -S * L0->aW[i];
                    if (i < n) PST(L, p, 1, 0) = -S * L0->aE[p];
                    if (j > 1) PST(L, p, 0, -1) = -S * L0->aS[j];
                    if (j < n) PST(L, p, 0, 1) = -S * L0->aN[p];
                }
        } else {
            pl_galerkin(&P->pl[l - 1], L);
        }
        if (nx <= 4) { P->PL = l + 1; break; }
        pl_weights(L);
        nx /= 2;
        l++;
        if (l >= 24) return ORC_E_ARG;
    }
    return ORC_OK;
}

/* M_CC^{-1}: stationary iteration with the V-cycle until the corner residual, in the
 * FE-rescaled Euclidean norm ||S_0 rho||_2, drops by the relative factor mg_red = 1e-3
 * (reading R6), starting from z = 0; cap mg_cap cycles.  Returns the
 * number of cycles. */
int orc2_corner_solve(orc2d *P, const double *bC, double *zC, int *cap_hit)
{
    orc_level *L0 = &P->lev[0];
    int nl = L0->nl;
    size_t nn = (size_t)nl * nl;
    double *rho = malloc(nn * sizeof(double));
    memset(zC, 0, nn * sizeof(double));
    double b0 = fe_norm(L0, bC);
    int cycles = 0;
    *cap_hit = 0;
    if (P->par) {
        /* the same iteration on the FE-scaled corner system (S A_CC) z = S b_C: the
         * scaled residual S b - (S A_CC) z = S (b - A_CC z) has the norm of reading R6 */
        orc_plev *Q = &P->pl[0];
        double *sb = malloc(nn * sizeof(double));
        for (int j = 1; j <= nl; j++)
            for (int i = 1; i <= nl; i++) sb[IX(i, j, nl)] = (L0->hb[i] * L0->kb[j]) * bC[IX(i, j, nl)];

        for (;;) {
            pl_residual(Q, sb, zC, rho);
            double rn = 0.0;
            for (size_t p = 0; p < nn; p++) rn += rho[p] * rho[p];
            if (P->mg_fixed > 0) { if (cycles >= P->mg_fixed) break; }
            else {
                if (sqrt(rn) <= P->mg_red * b0) break;
                if (cycles >= P->mg_cap) { *cap_hit = 1; break; }
            }
            pl_vcycle(P, 0, rho);
            for (size_t p = 0; p < nn; p++) zC[p] += Q->e[p];
            cycles++;
        }
        free(sb);
        free(rho);
        return cycles;
    }
    for (;;) {
        for (size_t p = 0; p < nn; p++) rho[p] = 0.0;
        mg_residual(L0, bC, zC, rho);
        if (P->mg_fixed > 0) { if (cycles >= P->mg_fixed) break; }
        else {
            if (fe_norm(L0, rho) <= P->mg_red * b0) break;
            if (cycles >= P->mg_cap) { *cap_hit = 1; break; }
        }
        mg_vcycle(P, 0, rho);
        for (size_t p = 0; p < nn; p++) zC[p] += L0->e[p];
        cycles++;
    }
    free(rho);
    return cycles;
}

/* ----- block preconditioner eq:2D blocks, back-substitution I -> Y -> X -> C ----- */

/* M_II: downstream Gauss-Seidel = the upper-triangular part of A_II (E and N
 * kept), swept from the upper-right corner of I to the bottom-left; neighbours outside I are
 * zero.  q is the vector being preconditioned.  Writes z on I. */
void orc2_stage_I(const orc2d *P, const double *q, double *z)
{
    int n = P->n, m = P->m;
    for (int j = m; j >= n + 1; j--)
        for (int i = m; i >= n + 1; i--) {
            size_t p = IX(i, j, m);
            double zE = (i < m) ? z[IX(i + 1, j, m)] : 0.0;
            double zN = (j < m) ? z[IX(i, j + 1, m)] : 0.0;
            z[p] = (q[p] + P->aE[p] * zE + P->aN[p] * zN) / P->D[p];
        }
}

/* M_YY: block downstream Gauss-Seidel with line solves along lines of constant
 * x, ordered right-to-left; each line j = 1..n is tridiagonal (-aS, D, -aN), W dropped, the
 * East neighbour (already solved) and, on the top row j = n, the North neighbour in I (A_YI)
 * moved to the right-hand side.  Thomas per line. */
int orc2_stage_Y(const orc2d *P, const double *q, double *z)
{
    int n = P->n, m = P->m;
    double *lo = malloc(sizeof(double) * n), *di = malloc(sizeof(double) * n);
    double *up = malloc(sizeof(double) * n), *rh = malloc(sizeof(double) * n), *s = malloc(sizeof(double) * n);
    int st = ORC_OK;
    for (int i = m; i >= n + 1 && st == ORC_OK; i--) {
        for (int j = 1; j <= n; j++) {
            size_t p = IX(i, j, m);
            lo[j - 1] = -P->aS[j];
            di[j - 1] = P->D[p];
            up[j - 1] = (j < n) ? -P->aN[p] : 0.0;
            double zE = (i < m) ? z[IX(i + 1, j, m)] : 0.0;
            rh[j - 1] = q[p] + P->aE[p] * zE;
            if (j == n) rh[j - 1] += P->aN[p] * z[IX(i, n + 1, m)];
        }
        st = orc_thomas(n, lo, di, up, rh, s);
        for (int j = 1; j <= n; j++) z[IX(i, j, m)] = s[j - 1];
    }
    free(lo); free(di); free(up); free(rh); free(s);
    return st;
}

/* M_XX: line solves along lines of constant y, swept from the top of the mesh
 * downwards; each line i = 1..n tridiagonal (-aW, D, -aE), S dropped, the North neighbour
 * (line above, already solved) and, at i = n, the East neighbour in I (A_XI) on the rhs.
 * A_XY = 0 for the 5-point stencil. */
int orc2_stage_X(const orc2d *P, const double *q, double *z)
{
    int n = P->n, m = P->m;
    double *lo = malloc(sizeof(double) * n), *di = malloc(sizeof(double) * n);
    double *up = malloc(sizeof(double) * n), *rh = malloc(sizeof(double) * n), *s = malloc(sizeof(double) * n);
    int st = ORC_OK;
    for (int j = m; j >= n + 1 && st == ORC_OK; j--) {
        for (int i = 1; i <= n; i++) {
            size_t p = IX(i, j, m);
            lo[i - 1] = -P->aW[i];
            di[i - 1] = P->D[p];
            up[i - 1] = (i < n) ? -P->aE[p] : 0.0;
            double zN = (j < m) ? z[IX(i, j + 1, m)] : 0.0;
            rh[i - 1] = q[p] + P->aN[p] * zN;
            if (i == n) rh[i - 1] += P->aE[p] * z[IX(n + 1, j, m)];
        }
        st = orc_thomas(n, lo, di, up, rh, s);
        for (int i = 1; i <= n; i++) z[IX(i, j, m)] = s[i - 1];
    }
    free(lo); free(di); free(up); free(rh); free(s);
    return st;
}

/* Corner right-hand side b_C = q_C - A_CX z_X - A_CY z_Y - A_CI z_I (first block row of
 * eq:2D blocks): only row j = n couples to X (North) and column i = n to Y (East);
 * A_CI = 0 for the 5-point stencil.  bC is n x n. */
void orc2_corner_rhs(const orc2d *P, const double *q, const double *z, double *bC)
{
    int n = P->n, m = P->m;
    for (int j = 1; j <= n; j++)
        for (int i = 1; i <= n; i++) {
            size_t p = IX(i, j, m);
            double v = q[p];
            if (j == n) v += P->aN[p] * z[IX(i, n + 1, m)];
            if (i == n) v += P->aE[p] * z[IX(n + 1, j, m)];
            bC[IX(i, j, n)] = v;
        }
}

/* z = M^{-1} q  (eq:2D blocks solved by block back-substitution). */
int orc2_precond(orc2d *P, const double *q, double *z)
{
    int n = P->n, m = P->m;
    memset(z, 0, sizeof(double) * (size_t)m * m);
    orc2_stage_I(P, q, z);
    int st = orc2_stage_Y(P, q, z);
    if (st != ORC_OK) return st;
    st = orc2_stage_X(P, q, z);
    if (st != ORC_OK) return st;
    orc2_corner_rhs(P, q, z, P->bC);
    int cap = 0;
    int cyc = orc2_corner_solve(P, P->bC, P->zC, &cap);
    for (int j = 1; j <= n; j++)
        for (int i = 1; i <= n; i++) z[IX(i, j, m)] = P->zC[IX(i, j, n)];
    if (P->applies < P->cycle_log_cap) P->cycle_log[P->applies] = cyc;
    P->applies++;
    P->mg_cycles_total += cyc;
    if (cyc < P->mg_min) P->mg_min = cyc;
    if (cyc > P->mg_max) P->mg_max = cyc;
    P->mg_cap_hits += cap;
    return ORC_OK;
}

/* ----- context management and solver entry ----- */

void orc2_destroy(orc2d *P)
{
    if (!P) return;
    free(P->aW); free(P->aS); free(P->aE); free(P->aN); free(P->rr); free(P->D);
    for (int l = 0; l < P->L; l++) {
        orc_level *Lv = &P->lev[l];
        free(Lv->aW); free(Lv->aS); free(Lv->aE); free(Lv->aN); free(Lv->rr); free(Lv->D);
        free(Lv->hb); free(Lv->kb); free(Lv->e); free(Lv->rho); free(Lv->b);
        free(Lv->wxl); free(Lv->wxr); free(Lv->wyl); free(Lv->wyr);
    }
    for (int l = 0; l < P->PL; l++) {
        orc_plev *L = &P->pl[l];
        free(L->a); free(L->wW); free(L->wE); free(L->e); free(L->rho); free(L->b);
    }
    free(P->cycle_log); free(P->bC); free(P->zC);
    free(P);
}

/* N even, N/2 a power of two >= 4 (full coarsening). */
orc2d *orc2_create(int N, double eps, const double *x, const double *y, const double *c1,
                   const double *c2, const double *r, double mg_red, int mg_cap, int mg_fixed)
{
    if (N < 8 || (N % 2) || ((N / 2) & (N / 2 - 1)) || !(eps > 0.0)) return NULL;
    orc2d *P = calloc(1, sizeof(orc2d));
    if (!P) return NULL;
    P->N = N; P->n = N / 2; P->m = N - 1; P->eps = eps;
    P->gx = !mesh_is_shishkin(x, N); P->gy = !mesh_is_shishkin(y, N);
    size_t mm = (size_t)P->m * P->m;
    P->aW = calloc(N + 1, sizeof(double)); P->aS = calloc(N + 1, sizeof(double));
    P->aE = malloc(mm * sizeof(double)); P->aN = malloc(mm * sizeof(double));
    P->rr = malloc(mm * sizeof(double)); P->D = malloc(mm * sizeof(double));
    P->bC = malloc(sizeof(double) * (size_t)P->n * P->n); P->zC = malloc(sizeof(double) * (size_t)P->n * P->n);
    P->cycle_log_cap = 4096; P->cycle_log = calloc(P->cycle_log_cap, sizeof(int));
    if (!P->aW || !P->aS || !P->aE || !P->aN || !P->rr || !P->D || !P->bC || !P->zC || !P->cycle_log) {
        orc2_destroy(P); return NULL;
    }
    orc2_coef(P, x, y, c1, c2, r);
    int nl = P->n, L = 1;
    while (nl > 4) { nl /= 2; L++; }          /* coarsest grid: <= 4 points per axis */
    P->L = L;
    for (int l = 0; l < L; l++)
        if (build_level(P, l, x, y, c1, c2, r) != ORC_OK) { P->L = l + 1; orc2_destroy(P); return NULL; }
    /* c2 = 0 everywhere: one parabolic layer along y = 0, semi-coarsening Galerkin
     * multigrid in the corner */
    P->par = 1;
    for (size_t k = 0; k < mm; k++) if (c2[k] != 0.0) { P->par = 0; break; }
    if (P->par && pl_build(P) != ORC_OK) { orc2_destroy(P); return NULL; }
    P->mg_red = mg_red; P->mg_cap = mg_cap; P->mg_fixed = mg_fixed;
    P->mg_min = 1 << 30;
    return P;
}

static void cb2_A(void *c, const double *x, double *y) { orc2_matvec_raw((orc2d *)c, x, y); }
static int cb2_M(void *c, const double *q, double *z) { return orc2_precond((orc2d *)c, q, z); }

/* FGMRES on the 2D system.  out_i: [0]=iters [1]=converged [2]=mg_cycles_total [3]=mg_min
 * [4]=mg_max [5]=mg_cap_hits [6]=applies;  out_d: [0]=res0 [1]=res_final. */
int orc2_solve_r(orc2d *P, const double *f, double *u, int weighted, int stop_abs, double tol,
                 int maxit, int fixed_iters, int restart, double *hist, int hist_cap, int *out_i, double *out_d)
{
    P->mg_cycles_total = 0; P->mg_min = 1 << 30; P->mg_max = 0; P->mg_cap_hits = 0; P->applies = 0;
    orc_sys s = {(size_t)P->m * P->m, P, cb2_A, cb2_M, P->D};
    orc_kstats st;
    int rc = orc_fgmres_r(&s, f, u, weighted, stop_abs, tol, maxit, fixed_iters, restart, hist, hist_cap, &st);
    out_i[0] = st.iters; out_i[1] = st.converged; out_i[2] = (int)P->mg_cycles_total;
    out_i[3] = P->applies ? P->mg_min : 0; out_i[4] = P->mg_max; out_i[5] = P->mg_cap_hits;
    out_i[6] = P->applies;
    out_d[0] = st.res0; out_d[1] = st.res_final;
    return rc;
}

int orc2_solve(orc2d *P, const double *f, double *u, int weighted, int stop_abs, double tol,
               int maxit, int fixed_iters, double *hist, int hist_cap, int *out_i, double *out_d)
{
    return orc2_solve_r(P, f, u, weighted, stop_abs, tol, maxit, fixed_iters, 0, hist, hist_cap, out_i, out_d);
}

/* accessors for tests */
int orc2_levels(const orc2d *P) { return P->L; }
int orc2_level_n(const orc2d *P, int l) { return P->lev[l].nl; }
void orc2_get_coef(const orc2d *P, double *aW, double *aS, double *aE, double *aN, double *D)
{
    size_t mm = (size_t)P->m * P->m;
    memcpy(aW, P->aW, sizeof(double) * (P->N + 1));
    memcpy(aS, P->aS, sizeof(double) * (P->N + 1));
    memcpy(aE, P->aE, sizeof(double) * mm);
    memcpy(aN, P->aN, sizeof(double) * mm);
    memcpy(D, P->D, sizeof(double) * mm);
}
void orc2_get_level_coef(const orc2d *P, int l, double *aW, double *aS, double *aE, double *aN,
                         double *D, double *hb, double *kb)
{
    const orc_level *Lv = &P->lev[l];
    size_t nn = (size_t)Lv->nl * Lv->nl;
    memcpy(aW, Lv->aW, sizeof(double) * (Lv->nl + 2));
    memcpy(aS, Lv->aS, sizeof(double) * (Lv->nl + 2));
    memcpy(aE, Lv->aE, sizeof(double) * nn);
    memcpy(aN, Lv->aN, sizeof(double) * nn);
    memcpy(D, Lv->D, sizeof(double) * nn);
    memcpy(hb, Lv->hb, sizeof(double) * (Lv->nl + 2));
    memcpy(kb, Lv->kb, sizeof(double) * (Lv->nl + 2));
}
void orc2_matvec(const orc2d *P, const double *u, double *y) { orc2_matvec_raw(P, u, y); }
int orc2_cycle_log(const orc2d *P, int *out, int cap)
{
    int k = P->applies < P->cycle_log_cap ? P->applies : P->cycle_log_cap;
    if (k > cap) k = cap;
    memcpy(out, P->cycle_log, sizeof(int) * k);
    return P->applies;
}
void orc2_gs_sweep(orc2d *P, int l, const double *b, double *e) { mg_gs(&P->lev[l], b, e); }
void orc2_vcycle(orc2d *P, int l, const double *b, double *e)
{
    mg_vcycle(P, l, b);
    memcpy(e, P->lev[l].e, sizeof(double) * (size_t)P->lev[l].nl * P->lev[l].nl);
}
void orc2_level_residual(orc2d *P, int l, const double *b, const double *e, double *rho)
{
    mg_residual(&P->lev[l], b, e, rho);
}
void orc2_restrict(orc2d *P, int l, const double *rho, double *bc)
{
    mg_restrict(&P->lev[l], &P->lev[l + 1], rho, bc);
}
void orc2_prolong_add(orc2d *P, int l, const double *ec, double *e)
{
    mg_prolong_add(&P->lev[l], &P->lev[l + 1], ec, e);
}
int orc2_corner_solve_ext(orc2d *P, const double *bC, double *zC, int *cap)
{
    return orc2_corner_solve(P, bC, zC, cap);
}
void orc2_set_mg(orc2d *P, double red, int cap, int fixed)
{
    P->mg_red = red; P->mg_cap = cap; P->mg_fixed = fixed;
}

/* O1 for 2D: banded LU (bandwidth m = N-1, lexicographic order, no pivoting -- A is an
 * M-matrix) followed by difference-form iterative refinement.
 * Memory (2m+1)*m^2 doubles: intended for N <= 256. */
int orc2_direct(const orc2d *P, const double *f, double *u, int refine)
{
    int m = P->m;
    size_t n = (size_t)m * m, bw = (size_t)m, ld = 2 * bw + 1;
    double *B = calloc(n * ld, sizeof(double));       /* B[p*ld + (q - p + bw)] = A[p][q] */
    double *res = malloc(n * sizeof(double)), *cor = malloc(n * sizeof(double));
    if (!B || !res || !cor) { free(B); free(res); free(cor); return ORC_E_NOMEM; }
    for (int j = 1; j <= m; j++)
        for (int i = 1; i <= m; i++) {
            size_t p = IX(i, j, m);
            B[p * ld + bw] = P->D[p];
            if (i > 1) B[p * ld + bw - 1] = -P->aW[i];
            if (i < m) B[p * ld + bw + 1] = -P->aE[p];
            if (j > 1) B[p * ld + bw - bw] = -P->aS[j];
            if (j < m) B[p * ld + bw + bw] = -P->aN[p];
        }
    /* LU in band storage (Doolittle, unit lower) */
    for (size_t k = 0; k < n; k++) {
        double piv = B[k * ld + bw];
        if (!(piv != 0.0)) { free(B); free(res); free(cor); return ORC_E_PIVOT; }
        size_t iend = (k + bw < n - 1) ? k + bw : n - 1;
        for (size_t i = k + 1; i <= iend; i++) {
            double *ai = B + i * ld + bw - i;     /* ai[q] = A[i][q] */
            double l = ai[k] / piv;
            if (l == 0.0) continue;
            ai[k] = l;
            const double *ak = B + k * ld + bw - k;
            for (size_t q = k + 1; q <= iend; q++) ai[q] -= l * ak[q];
        }
    }
    /* solve LU x = rhs; refine in difference form */
    for (int pass = 0; pass <= refine; pass++) {
        if (pass == 0) memcpy(res, f, n * sizeof(double));
        else {
            orc2_matvec_raw(P, u, res);
            for (size_t p = 0; p < n; p++) res[p] = f[p] - res[p];
        }
        for (size_t i = 0; i < n; i++) {
            const double *ai = B + i * ld + bw - i;
            size_t q0 = (i > bw) ? i - bw : 0;
            double s = res[i];
            for (size_t q = q0; q < i; q++) s -= ai[q] * cor[q];
            cor[i] = s;
        }
        for (size_t ii = n; ii-- > 0;) {
            const double *ai = B + ii * ld + bw - ii;
            size_t qe = (ii + bw < n - 1) ? ii + bw : n - 1;
            double s = cor[ii];
            for (size_t q = ii + 1; q <= qe; q++) s -= ai[q] * cor[q];
            cor[ii] = s / ai[ii];
        }
        if (pass == 0) memcpy(u, cor, n * sizeof(double));
        else for (size_t p = 0; p < n; p++) u[p] += cor[p];
    }
    free(B); free(res); free(cor);
    return ORC_OK;
}

/* parabolic-corner accessors for the tests (nine-point levels) */
int orc2_par(const orc2d *P) { return P->par; }
int orc2_plevels(const orc2d *P) { return P->par ? P->PL : 0; }
int orc2_plevel_nx(const orc2d *P, int l) { return P->pl[l].nx; }
void orc2_plevel_stencil(const orc2d *P, int l, double *a)
{
    memcpy(a, P->pl[l].a, sizeof(double) * (size_t)P->pl[l].nx * P->pl[l].ny * 9);
}
void orc2_pgs(orc2d *P, int l, const double *b, double *e) { pl_gs(&P->pl[l], b, e); }
void orc2_pvcycle(orc2d *P, int l, const double *b, double *e)
{
    pl_vcycle(P, l, b);
    memcpy(e, P->pl[l].e, sizeof(double) * (size_t)P->pl[l].nx * P->pl[l].ny);
}
void orc2_presidual(orc2d *P, int l, const double *b, const double *e, double *rho) { pl_residual(&P->pl[l], b, e, rho); }
void orc2_prestrict(orc2d *P, int l, const double *r, double *bc) { pl_restrict(&P->pl[l], &P->pl[l + 1], r, bc); }
void orc2_pprolong_add(orc2d *P, int l, const double *ec, double *e) { pl_prolong_add(&P->pl[l], &P->pl[l + 1], ec, e); }
