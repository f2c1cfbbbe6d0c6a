// capi.cu -- the C ABI (include/spp.h): context management, setup, the FGMRES driver
// (P:1306-1316), the block preconditioner (eq:2D blocks) and the corner
// multigrid driver.  Every arithmetic step runs in the sm_100a kernels of
// k_core.cu / k_sweep.cu / k_lines.cu / k_1d.cu; the host only orchestrates launches and does
// the O(k^2) Givens/Hessenberg bookkeeping of GMRES ("host, k <= a few hundred
// scalars").
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>

#include <nvtx3/nvToolsExt.h>

#include "dist.cuh"
#include "kernels.cuh"

using namespace spp;

static thread_local std::string g_err;

#define FAIL(ctx, code, ...)                                                  \
    do {                                                                      \
        char _b[512];                                                         \
        snprintf(_b, sizeof(_b), __VA_ARGS__);                                \
        if (ctx) ((Ctx *)(ctx))->err = _b;                                    \
        g_err = _b;                                                           \
        return code;                                                          \
    } while (0)

#define CK(ctx, expr)                                                         \
    do {                                                                      \
        cudaError_t _e = (expr);                                              \
        if (_e != cudaSuccess)                                                \
            FAIL(ctx, SPP_E_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
    } while (0)

namespace spp {

// ------------------------------------------------------------------------------------------ profiling
static const char *kProfNames[SPP_PROF_CLASSES] = {"spmv", "sweep_I", "lines_XY", "mg_sweep",
                                                   "mg_resid_restrict", "mg_prolong", "mg_update",
                                                   "krylov_vec", "setup", "other", "mg_coarse", "exchange"};

// NVTX ranges (tracing): SPP_NVTX=1 names every launch class and the setup / solve
// calls on the host timeline of a tracing tool (nvtx3 is header-only and does nothing unless a
// tool is attached).  With the iteration graphs the ranges bracket the capture, not the replay:
// trace with SPP_NO_GRAPH=1 for per-launch ranges.
static bool nvtx_on()
{
    static const bool on = [] { const char *e = getenv("SPP_NVTX"); return e && *e && *e != '0'; }();
    return on;
}
NvtxScope::NvtxScope(const char *name) : on(nvtx_on()) { if (on) nvtxRangePushA(name); }
NvtxScope::~NvtxScope() { if (on) nvtxRangePop(); }

ProfScope::ProfScope(Ctx *c_, int cls_, double bytes_) : c(c_), cls(cls_), bytes(bytes_)
{
    if (nvtx_on() && cls >= 0 && cls < SPP_PROF_CLASSES) { nvtxRangePushA(kProfNames[cls]); nv = true; }
    if (!c || !(c->prof_on & (1 << cls))) { c = nullptr; return; }
    if (c->ev_used + 2 > c->ev_pool.size()) {
        for (int k = 0; k < 64; ++k) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            c->ev_pool.push_back(e);
        }
    }
    a = c->ev_pool[c->ev_used++];
    cudaEventRecord(a, c->st);
}
ProfScope::~ProfScope()
{
    if (nv) nvtxRangePop();
    if (!c) return;
    cudaEvent_t b = c->ev_pool[c->ev_used++];
    cudaEventRecord(b, c->st);
    c->pend.push_back({cls, a, b, bytes});
}

void prof_collect(Ctx *c)
{
    if (c->pend.empty()) { c->ev_used = 0; return; }
    cudaEventSynchronize(c->pend.back().b);
    for (auto &p : c->pend) {
        float ms = 0;
        cudaEventElapsedTime(&ms, p.a, p.b);
        c->prof[p.cls].launches++;
        c->prof[p.cls].ms += ms;
        c->prof[p.cls].bytes += p.bytes;
    }
    c->pend.clear();
    c->ev_used = 0;
}

// ------------------------------------------------------------------------------------------ helpers
static inline int nblk(long work, int tpb = 256, int cap = 148 * 16)
{
    long b = (work + tpb - 1) / tpb;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (int)b;
}

static double host_sum(const double *p, int k)
{
    double s = 0.0;
    for (int i = 0; i < k; ++i) s += p[i];
    return s;
}

// D2H of a partial-sum block and host reduction in fixed order
static cudaError_t fetch_sum(Ctx *c, const double *part, double *out)
{
    cudaError_t e = cudaMemcpyAsync(c->hpin, part, sizeof(double) * kRedBlocks, cudaMemcpyDeviceToHost, c->st);
    if (e != cudaSuccess) return e;
    e = cudaStreamSynchronize(c->st);
    if (e != cudaSuccess) return e;
    *out = host_sum(c->hpin, kRedBlocks);
    return cudaSuccess;
}

static double *part_slot(Ctx *c, int k) { return c->part + (size_t)k * c->nparts * kRedBlocks; }

// ------------------------------------------------------------------------------------------ corner MG
// V(1,1) cycle for A_l e = R, zero initial guess ("standard V(1,1) cycling", one
// downstream GS sweep before and after the coarse-grid correction; coarsest grid: "four sweeps",
// P:1208-1209 / P:1281-1283).  Returns the buffer holding e (lev[l].e or lev[l].q).
// rs: R holds R / D (the z-form V-cycle stores every level's right-hand side divided by D; the
// caller's R may be plain, e.g. the test hooks).
double *vcycle(Ctx *c, int l, const double *R, bool rs)
{
    Level &L = c->lev[l];
    const bool zf = c->mg_zform;
    double *ea = L.e, *eb = L.q;
    if (launch_coarse_vcycle(c, l, R, zf && rs)) return eb;   // levels l..L-1 fused (smem-resident)
    if (l == c->L - 1) {
        launch_gs(c, l, 0, R, nullptr, ea, nullptr, rs);
        launch_gs(c, l, 1, R, ea, eb, nullptr, rs);
        launch_gs(c, l, 1, R, eb, ea, nullptr, rs);
        launch_gs(c, l, 1, R, ea, eb, nullptr, rs);
        return eb;
    }
    Level &C = c->lev[l + 1];
    launch_gs(c, l, 0, R, nullptr, ea, nullptr, rs);          // pre-smoothing from zero
    launch_resid_restrict(c, l, nullptr, ea, false, zf);      // C.b = S^-1 P^T S (R - A_l ea) (/ D_c in z-form),
                                                              // R - A_l ea = aW ea_W + aS ea_S (ea: sweep from 0)
    const double *ec = vcycle(c, l + 1, C.b, zf);
    launch_gs(c, l, 1, R, ea, eb, ec, rs);                    // post-smoothing from ea + P ec
    return eb;
}

// M_CC^{-1} b_C: stationary V-cycle iteration z <- z + V(b_C - A_CC z) from z = 0 until
// ||S_0 rho||_2 <= mg_reduction ||S_0 b_C||_2 (reading R6), cap mg_max_cycles
// (S:496); or exactly mg_fixed_cycles cycles (reading R17).  b0sq = ||S_0 b_C||^2.
// *zout = the buffer holding z (nullptr when no cycle ran: z = 0).  Returns the cycle count.
static int corner_solve(Ctx *c, const double *bc, double b0sq, int *cap_hit, cudaError_t *err,
                        const double **zout)
{
    Level &L0 = c->lev[0];
    *cap_hit = 0;
    *err = cudaSuccess;
    const double b0 = std::sqrt(b0sq);
    double res = b0;
    const double *R = L0.rho;                          // b_C (/ D in z-form), written with b_C
    const double *z = nullptr;
    double *zb[2] = {c->Zc, c->Zc2};
    int cycles = 0;
    const int fixed = c->opt.mg_fixed_cycles;
    for (;;) {
        if (fixed > 0) { if (cycles >= fixed) break; }
        else {
            if (res <= c->opt.mg_reduction * b0) break;
            if (cycles >= c->opt.mg_max_cycles) { *cap_hit = 1; break; }
        }
        const double *e = vcycle(c, 0, R, c->mg_zform);
        double *zn = zb[cycles & 1];
        launch_cycle_update(c, z, e, zn, bc, L0.rho, part_slot(c, 0));   // z += e; rho = b - A z
        z = zn;
        R = L0.rho;
        cycles++;
        if (fixed <= 0) {
            double s = 0;
            cudaError_t e2 = fetch_sum(c, part_slot(c, 0), &s);
            if (e2 != cudaSuccess) { *err = e2; break; }
            res = std::sqrt(s);
        }
    }
    *zout = z;
    return cycles;
}

// ------------------------------------------------------------------------------------------ corner graph
// The stationary iteration of corner_solve as one CUDA graph: an init kernel, then a device-side
// while loop whose body is one V-cycle (every level's launches), the update z' = z + e with
// rho = b_C - A_CC z', and a check kernel that makes exactly corner_solve's decision (same
// partial sums in the same order, same tests) and sets the loop condition.  No host round trip
// per cycle; the cycle count is read back at the FGMRES iteration's own synchronisation.
__device__ __forceinline__ double ordered_sum(const double *p)
{
    double s = 0.0;
    for (int i = 0; i < kRedBlocks; ++i) s += p[i];   // host_sum's order
    return s;
}
__device__ __forceinline__ int mg_continue(MGState *s, double red, int maxc, int fixed)
{
    if (fixed > 0) return s->cycles < fixed;
    if (s->res <= red * s->b0) return 0;
    if (s->cycles >= maxc) { s->cap = 1; return 0; }
    return 1;
}
__global__ void k_mg_init(const double *part_b, MGState *s, double *za, double *zb, double red, int maxc, int fixed,
                          cudaGraphConditionalHandle h)
{
    s->b0 = fixed > 0 ? 0.0 : sqrt(ordered_sum(part_b));
    s->res = s->b0;
    s->cycles = 0; s->cap = 0;
    s->zcur = nullptr; s->za = za; s->zb = zb; s->znext = za;
    cudaGraphSetConditional(h, mg_continue(s, red, maxc, fixed));
}
__global__ void k_mg_check(const double *part_r, MGState *s, double red, int maxc, int fixed,
                           cudaGraphConditionalHandle h)
{
    s->cycles++;
    if (fixed <= 0) s->res = sqrt(ordered_sum(part_r));
    s->zcur = s->znext;
    s->znext = s->znext == s->za ? s->zb : s->za;
    cudaGraphSetConditional(h, mg_continue(s, red, maxc, fixed));
}

// what the captured launches depend on besides fixed buffers: the level plans and MG options
static std::vector<long> corner_signature(const Ctx *c)
{
    std::vector<long> v{c->N, c->L, c->tune.coarse_max, c->opt.mg_fixed_cycles, c->opt.mg_max_cycles,
                        (long)(c->opt.mg_reduction * 1e15)};
    for (int l = 0; l < c->L; ++l) {
        const Level &L = c->lev[l];
        for (long x : {(long)L.n, L.pitch, L.cpitch, (long)L.tile_warps, (long)L.tile_rows, (long)L.tile_cols,
                       (long)L.halo_x, (long)L.halo_y})
            v.push_back(x);
    }
    return v;
}

static void corner_graph_destroy(Ctx *c)
{
    if (c->cg_exec) cudaGraphExecDestroy(c->cg_exec);
    if (c->cg) cudaGraphDestroy(c->cg);
    c->cg_exec = nullptr; c->cg = nullptr; c->cg_sig.clear();
}

// During a capture on c->st into graph g: append a node of type `type` (a conditional with handle
// h) after the captured work, continue the capture after it; *body = its body graph.
static cudaError_t capture_add_conditional(Ctx *c, cudaGraph_t g, cudaGraphConditionalHandle h,
                                           cudaGraphConditionalNodeType type, cudaGraph_t *body)
{
    cudaStreamCaptureStatus cs;
    const cudaGraphNode_t *deps = nullptr;
    size_t nd = 0;
    SPP_CUDA_TRY(cudaStreamGetCaptureInfo(c->st, &cs, nullptr, nullptr, &deps, &nd));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = type;
    cp.conditional.size = 1;
    cudaGraphNode_t wn = nullptr;
    SPP_CUDA_TRY(cudaGraphAddNode(&wn, g, deps, nd, &cp));
    SPP_CUDA_TRY(cudaStreamUpdateCaptureDependencies(c->st, &wn, 1, cudaStreamSetCaptureDependencies));
    *body = cp.conditional.phGraph_out[0];
    return cudaSuccess;
}

// During a capture on c->st into graph g: the corner stationary iteration as k_mg_init + a while
// node (handle *h, created on g); *body receives the (empty) loop body for corner_body.
static cudaError_t capture_corner_loop(Ctx *c, cudaGraph_t g, cudaGraphConditionalHandle *h, cudaGraph_t *body)
{
    SPP_CUDA_TRY(cudaGraphConditionalHandleCreate(h, g, 0, 0));
    k_mg_init<<<1, 1, 0, c->st>>>(part_slot(c, 1), c->mgs, c->Zc, c->Zc2, c->opt.mg_reduction, c->opt.mg_max_cycles,
                                  c->opt.mg_fixed_cycles, *h);
    c->launches++;
    return capture_add_conditional(c, g, *h, cudaGraphCondTypeWhile, body);
}

// the corner loop body (one V-cycle, the update z' = z + e with rho = b_C - A_CC z', the check),
// captured on c->st (no capture active); sets c->cg_body_launches
static cudaError_t corner_body(Ctx *c, cudaGraph_t body, cudaGraphConditionalHandle h)
{
    Level &L0 = c->lev[0];
    SPP_CUDA_TRY(cudaStreamBeginCaptureToGraph(c->st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    const int64_t b0 = c->launches;
    const double *ev = vcycle(c, 0, L0.rho, c->mg_zform);
    launch_cycle_update(c, nullptr, ev, nullptr, c->Bc, L0.rho, part_slot(c, 0), c->mgs);
    k_mg_check<<<1, 1, 0, c->st>>>(part_slot(c, 0), c->mgs, c->opt.mg_reduction, c->opt.mg_max_cycles,
                                   c->opt.mg_fixed_cycles, h);
    c->launches++;
    c->cg_body_launches = c->launches - b0;
    cudaGraph_t tmp = nullptr;
    const cudaError_t e = cudaStreamEndCapture(c->st, &tmp);
    return e != cudaSuccess ? e : cudaGetLastError();
}

static cudaError_t corner_graph_build(Ctx *c)
{
    corner_graph_destroy(c);
    if (!c->cap_st) SPP_CUDA_TRY(cudaStreamCreateWithFlags(&c->cap_st, cudaStreamNonBlocking));
    cudaGraph_t g = nullptr;
    SPP_CUDA_TRY(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle h;
    cudaStream_t user = c->st;
    const int prof = c->prof_on;
    const int64_t l0 = c->launches;
    c->st = c->cap_st; c->prof_on = 0; c->capturing = true;
    cudaError_t e = cudaStreamBeginCaptureToGraph(c->st, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        cudaGraph_t body = nullptr;
        e = capture_corner_loop(c, g, &h, &body);
        cudaGraph_t tmp = nullptr;
        const cudaError_t e2 = cudaStreamEndCapture(c->st, &tmp);
        if (e == cudaSuccess) e = e2;
        if (e == cudaSuccess) e = corner_body(c, body, h);   // the loop body: one cycle
    }
    c->st = user; c->prof_on = prof; c->capturing = false;
    c->launches = l0;
    if (e == cudaSuccess && c->sticky != cudaSuccess) { e = c->sticky; c->sticky = cudaSuccess; }
    if (e == cudaSuccess) e = cudaGraphInstantiate(&c->cg_exec, g, 0);
    if (e != cudaSuccess) { cudaGraphDestroy(g); c->cg_exec = nullptr; return e; }
    c->cg = g;
    c->cg_sig = corner_signature(c);
    if (getenv("SPP_DEBUG_GRAPH")) fprintf(stderr, "[spp] corner graph captured: %lld kernels per cycle\n", (long long)c->cg_body_launches);
    return cudaSuccess;
}

// corner solve through the graph (b_C in c->Bc and L0.rho, ||S0 b_C||^2 partials in part slot 1);
// the result is read through c->mgs (k_corner_out)
static cudaError_t corner_solve_graph(Ctx *c)
{
    if (!c->cg_exec || c->cg_sig != corner_signature(c)) SPP_CUDA_TRY(corner_graph_build(c));
    SPP_CUDA_TRY(cudaGraphLaunch(c->cg_exec, c->st));
    c->launches += 1;                                   // k_mg_init (the body is counted per cycle)
    return cudaSuccess;
}

static bool graph_mode(const Ctx *c) { return c->use_graph && c->prof_on == 0 && !c->par; }

// M_II solve on region I = [n+1, N-1]^2: z = (D - E - N)^{-1} (s v), s = 1/D
// (scaled, unweighted mode) or 1 (Jacobi mode: the input is already D v, reading R11); the exact
// chained row-scan sweep of k_mg.cu with the level origin at (n, n) of the global grid.
static void launch_mii(Ctx *c, const double *v, double *z, bool scaled)
{
    WaveArgs a{};
    a.nl = c->n - 1; a.pv = c->P; a.pc = c->P; a.ioff = c->n; a.joff = c->n;
    a.q = v; a.z = z; a.cd = c->cd;
    if (scaled) { ensure_y0(c); a.ca = c->ya; a.cn = c->yn; }   // D z = v + aE z_E + aN z_N (y-form)
    else { a.ca = c->ca; a.cn = c->cn; }          // z = (D v)/D + ca z_E + cn z_N (z-form)
    const double nn = (double)a.nl * a.nl;
    launch_wave_chain(c, a, c->N + 1, c->N + 1, scaled, 1, nn * (scaled ? 40.0 : 32.0));
}

// z = M^{-1} v (eq:2D blocks by block back-substitution I -> Y -> X -> C).
// v, z: padded global grids.  In Jacobi mode the preconditioner input is D v (reading R11).
// the blocks of M^{-1} before the corner solve: M_II, then M_YY and M_XX, then the corner's
// right-hand side b_C (with ||S0 b_C||^2 partials in part slot 1)
static void precond_head(Ctx *c, const double *v, double *z)
{
    const int N = c->N, n = c->n;
    // M_II: exact downstream triangular solve on region I
    launch_mii(c, v, z, !c->weighted);
    // M_YY and M_XX (one launch, both chains)
    launch_lines(c, v, z);
    Level &L0 = c->lev[0];
    ProfScope ps(c, 9, 40.0 * (double)n * n);
    int nb = 0, nt = 0;
    seg_shape(n, n, &nb, &nt);
    k_corner_rhs<<<nb, nt, 0, c->st>>>(N, c->P, L0.pitch, v, z, c->aE, c->aN, c->rr, c->aW,
                                                        c->aS, L0.hb, L0.kb, c->weighted, c->Bc, part_slot(c, 1),
                                                        L0.rho, c->cd, c->mg_zform, 1, n);
    c->launches++;
}

static int apply_precond(Ctx *c, const double *v, double *z, int *cap_hit, cudaError_t *err)
{
    const int n = c->n;
    precond_head(c, v, z);
    // corner
    Level &L0 = c->lev[0];
    const bool gm = graph_mode(c);
    if (c->par) {                                       // parabolic variant (NEXT-2): host-driven loop
        double b0sq = 0;
        cudaError_t e = fetch_sum(c, part_slot(c, 1), &b0sq);
        if (e != cudaSuccess) { *err = e; return 0; }
        const int cyc = par_corner_solve(c, b0sq, cap_hit, err);
        k_corner_out<<<nblk((long)n * n), 256, 0, c->st>>>(n, L0.pitch, c->Zc, c->P, z, nullptr, 1, n);
        c->launches++;
        return cyc;
    }
    if (gm) {                                           // cycles known after the caller's next sync
        *err = corner_solve_graph(c);
        k_corner_out<<<nblk((long)n * n), 256, 0, c->st>>>(n, L0.pitch, nullptr, c->P, z, c->mgs, 1, n);
        c->launches++;
        return -1;
    }
    double b0sq = 0;
    if (c->opt.mg_fixed_cycles <= 0) {
        cudaError_t e = fetch_sum(c, part_slot(c, 1), &b0sq);
        if (e != cudaSuccess) { *err = e; return 0; }
    }
    const double *zc = nullptr;
    int cyc = corner_solve(c, c->Bc, b0sq, cap_hit, err, &zc);
    if (!zc) {
        *err = cudaMemsetAsync(c->Zc, 0, sizeof(double) * L0.elems, c->st);
        zc = c->Zc;
    }
    k_corner_out<<<nblk((long)n * n), 256, 0, c->st>>>(n, L0.pitch, zc, c->P, z, nullptr, 1, n);
    c->launches++;
    return cyc;
}

// w = W A z_k with <w, v_0>, then modified Gram-Schmidt: h_{j,k} for j = 0..k into
// dscal[0..k], ||w|| into dscal[k+1], v_{k+1} = w / ||w||
static void krylov_tail(Ctx *c, int k)
{
    const int m = c->m;
    const long G = (long)c->G;
    const double mm = (double)m * m;
    {
        ProfScope ps(c, 0, 48.0 * mm);
        k_spmv<<<red_grid((long)m * m), kRedThreads, 0, c->st>>>(m, c->P, c->Z[k], c->aE, c->aN, c->rr, c->aW, c->aS,
                                                                  c->weighted, c->w, c->V[0], part_slot(c, 0), 1, m);
        c->launches++;
    }
    for (int j = 1; j <= k; ++j) {
        ProfScope ps(c, 7, 32.0 * G);
        k_mgs<<<red_grid(G), kRedThreads, 0, c->st>>>(G, c->w, c->V[j - 1], part_slot(c, j - 1), c->dscal + (j - 1),
                                                     c->V[j], part_slot(c, j), 1);
        c->launches++;
    }
    {
        ProfScope ps(c, 7, 24.0 * G + 16.0 * G);
        k_mgs<<<red_grid(G), kRedThreads, 0, c->st>>>(G, c->w, c->V[k], part_slot(c, k), c->dscal + k, c->w,
                                                     part_slot(c, k + 1), 1);
        k_normalize<<<red_grid(G), kRedThreads, 0, c->st>>>(G, c->w, part_slot(c, k + 1), c->dscal + k + 1, c->V[k + 1], 1);
        c->launches += 2;
    }
}

// ------------------------------------------------------------------------------------------ Givens
// The least-squares update of GMRES (Saad 2003, Alg. 6.9 via plane rotations), shared
// by the host loop and the device-side step of the iteration graphs so both make bit-identical
// decisions: explicit fma and a scaled sqrt in place of hypot (whose rounding differs between
// the host and device libraries).
__host__ __device__ inline double rot_norm(double a, double b)
{
    const double m = fmax(fabs(a), fabs(b));
    if (m == 0.0) return 0.0;
    const double x = a / m, y = b / m;
    return m * sqrt(fma(x, x, y * y));
}
// rotate column h (h[0..k+1]) by the previous rotations, form rotation k, update g; returns |g_{k+1}|
__host__ __device__ inline double givens_update(double *h, double *cs, double *sn, double *g, int k, int *brk)
{
    for (int i = 0; i < k; ++i) {
        const double t = fma(cs[i], h[i], sn[i] * h[i + 1]);
        h[i + 1] = fma(-sn[i], h[i], cs[i] * h[i + 1]);
        h[i] = t;
    }
    const double den = rot_norm(h[k], h[k + 1]);
    if (den == 0.0) { cs[k] = 1.0; sn[k] = 0.0; }
    else { cs[k] = h[k] / den; sn[k] = h[k + 1] / den; }
    *brk = h[k + 1] == 0.0;                            // happy breakdown: w in span(V)
    h[k] = den; h[k + 1] = 0.0;
    g[k + 1] = -sn[k] * g[k];
    g[k] = cs[k] * g[k];
    return fabs(g[k + 1]);
}
// the stop test after iteration k (0-based) with residual res; *converged set when stopping
__host__ __device__ inline int fg_stop(int k, double res, int brk, double target, int fixed, int maxit, int *converged)
{
    if (brk) { *converged = res <= target; return 1; }
    if (fixed > 0) {
        if (k + 1 >= fixed) { *converged = res <= target; return 1; }
    } else if (res <= target) { *converged = 1; return 1; }
    return k + 1 >= maxit;
}

// ------------------------------------------------------------------------------------------ iteration graphs
// Small problems are launch- and synchronisation-bound (cfg2: 52 iterations of ~100 launches).
// Iteration k of FGMRES becomes one CUDA graph: a gate kernel sets an IF node from the device
// state (nothing runs once the loop has stopped); its body is the whole iteration (M^{-1} with the
// corner stationary iteration as a nested while node, W A z_k, MGS) followed by k_fg_step, the
// Givens update and stop test on the device.  The host launches the graphs in batches (the first
// as long as the previous solve) and synchronises once per batch.  The kernels and their order
// are the host loop's, so the iterates are bit for bit the same.
__global__ void k_fg_init(FGHead *s, double *g, double *hist, double beta, double target)
{
    s->target = target;
    s->k = 0; s->stop = 0; s->converged = 0; s->nonfinite = 0; s->nf_j = 0; s->capfail = 0;
    s->mg_tot = 0; s->mg_min = 1 << 30; s->mg_max = 0; s->caps = 0;
    s->res = beta;
    g[0] = beta; hist[0] = beta;
}
__global__ void k_fg_gate(const FGHead *s, cudaGraphConditionalHandle h) { cudaGraphSetConditional(h, s->stop ? 0 : 1); }
__global__ void k_fg_step(FGHead *s, double *H, double *cs, double *sn, double *g, double *hist, const double *hsrc,
                          const MGState *ms, int k, int ld, int fixed, int maxit, int strict)
{
    s->k = k + 1;
    if (ms) {
        const int cyc = ms->cycles, cap = ms->cap;
        s->mg_tot += cyc; s->mg_min = min(s->mg_min, cyc); s->mg_max = max(s->mg_max, cyc); s->caps += cap;
        if (cap && strict) { s->capfail = 1; s->stop = 1; return; }
    }
    double *h = H + (size_t)k * ld;
    for (int j = 0; j <= k + 1; ++j) {
        h[j] = hsrc[j];
        if (!isfinite(h[j])) { s->nonfinite = 1; s->nf_j = j; s->stop = 1; return; }
    }
    int brk = 0, conv = 0;
    const double res = givens_update(h, cs, sn, g, k, &brk);
    hist[k + 1] = res;
    s->res = res;
    if (fg_stop(k, res, brk, s->target, fixed, maxit, &conv)) { s->stop = 1; s->converged = conv; }
}

static bool fg_mode(const Ctx *c) { return graph_mode(c) && c->fg_ok && !c->dist; }

static std::vector<long> fg_signature(const Ctx *c)
{
    // everything the captured launches take by value besides fixed buffers: the level plans, the
    // line-chunk plan (it follows the coefficients, so a re-setup may change it), the options
    std::vector<long> v = corner_signature(c);
    v.push_back(c->weighted); v.push_back((long)(size_t)c->d_chunks); v.push_back(c->lines_threads);
    for (const LineChunk &k : c->chunks) { v.push_back(k.chain); v.push_back(k.first); v.push_back(k.last); v.push_back(k.start); }
    v.push_back((long)(c->opt.tol * 1e15)); v.push_back(c->opt.stop); v.push_back(c->opt.fixed_iters);
    v.push_back(c->opt.mg_strict); v.push_back(c->opt.max_iters);
    return v;
}

static void fg_destroy(Ctx *c)
{
    for (auto e : c->itg) if (e) cudaGraphExecDestroy(e);
    c->itg.clear(); c->itg_launches.clear(); c->itg_sig.clear();
}

static cudaError_t fg_alloc(Ctx *c)
{
    if (c->fgh) return cudaSuccess;
    const size_t ld = (size_t)c->opt.max_iters + 1;
    SPP_CUDA_TRY(cudaMalloc(&c->fgh, sizeof(FGHead)));
    SPP_CUDA_TRY(cudaMallocHost(&c->hfgh, sizeof(FGHead)));
    SPP_CUDA_TRY(cudaMalloc(&c->fgd, sizeof(double) * (ld * ld + 4 * (ld + 1))));
    return cudaMemsetAsync(c->fgd, 0, sizeof(double) * (ld * ld + 4 * (ld + 1)), c->st);
}

// device arrays of the FGMRES state: H (column k at k * ld), cs, sn, g, hist
static double *fg_H(Ctx *c) { return c->fgd; }
static double *fg_arr(Ctx *c, int a)
{
    const size_t ld = (size_t)c->opt.max_iters + 1;
    return c->fgd + ld * ld + (size_t)a * (ld + 1);
}

// capture graph k (V[k+1], Z[k] allocated)
static cudaError_t fg_build(Ctx *c, int k, cudaGraphExec_t *out)
{
    if (!c->cap_st) SPP_CUDA_TRY(cudaStreamCreateWithFlags(&c->cap_st, cudaStreamNonBlocking));
    const int ld = c->opt.max_iters + 1;
    cudaGraph_t g = nullptr;
    SPP_CUDA_TRY(cudaGraphCreate(&g, 0));
    cudaStream_t user = c->st;
    const int prof = c->prof_on;
    const int64_t l0 = c->launches;
    c->st = c->cap_st; c->prof_on = 0; c->capturing = true;
    int64_t body_launches = 0;
    cudaGraph_t ifb = nullptr, wb = nullptr;
    cudaGraphConditionalHandle hif, hw;
    cudaError_t e = cudaGraphConditionalHandleCreate(&hif, g, 0, 0);
    if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(c->st, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        k_fg_gate<<<1, 1, 0, c->st>>>(c->fgh, hif);
        e = capture_add_conditional(c, g, hif, cudaGraphCondTypeIf, &ifb);
        cudaGraph_t tmp = nullptr;
        const cudaError_t e2 = cudaStreamEndCapture(c->st, &tmp);
        if (e == cudaSuccess) e = e2;
    }
    if (e == cudaSuccess) e = cudaStreamBeginCaptureToGraph(c->st, ifb, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        const int64_t b0 = c->launches;
        const int n = c->n;
        Level &L0 = c->lev[0];
        precond_head(c, c->V[k], c->Z[k]);
        e = capture_corner_loop(c, ifb, &hw, &wb);
        if (e == cudaSuccess) {
            k_corner_out<<<nblk((long)n * n), 256, 0, c->st>>>(n, L0.pitch, nullptr, c->P, c->Z[k], c->mgs, 1, n);
            c->launches++;
            krylov_tail(c, k);
            k_fg_step<<<1, 1, 0, c->st>>>(c->fgh, fg_H(c), fg_arr(c, 0), fg_arr(c, 1), fg_arr(c, 2), fg_arr(c, 3),
                                          c->dscal, c->mgs, k, ld, c->opt.fixed_iters, c->opt.max_iters,
                                          c->opt.mg_strict);
            c->launches++;
        }
        body_launches = c->launches - b0;
        cudaGraph_t tmp = nullptr;
        const cudaError_t e2 = cudaStreamEndCapture(c->st, &tmp);
        if (e == cudaSuccess) e = e2;
    }
    if (e == cudaSuccess) e = corner_body(c, wb, hw);
    c->st = user; c->prof_on = prof; c->capturing = false;
    c->launches = l0;
    if (e == cudaSuccess && c->sticky != cudaSuccess) { e = c->sticky; c->sticky = cudaSuccess; }
    if (e == cudaSuccess) e = cudaGraphInstantiate(out, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) { *out = nullptr; return e; }
    if ((int)c->itg_launches.size() <= k) c->itg_launches.resize(k + 1, 0);
    c->itg_launches[k] = body_launches;
    return cudaSuccess;
}

}  // namespace spp

// =========================================================================================== ABI
extern "C" {

#ifdef SPP_STRESS
const char *spp_version(void) { return "spp-b200 0.1 (sm_100a, fp64) +stress"; }   // race-check build
#else
const char *spp_version(void) { return "spp-b200 0.1 (sm_100a, fp64)"; }
#endif

const char *spp_last_error(const spp_ctx *c)
{
    if (c) return ((const Ctx *)c)->err.c_str();
    return g_err.c_str();
}

const char *spp_profile_name(int32_t k) { return (k >= 0 && k < SPP_PROF_CLASSES) ? kProfNames[k] : "?"; }

void spp_default_options(int32_t dim, spp_options *o)
{
    if (!o) return;
    memset(o, 0, sizeof(*o));
    o->side = SPP_RIGHT_FLEXIBLE;
    o->stop = SPP_STOP_REL_JACOBI;
    o->tol = dim == 1 ? 1e-10 : 1e-8;
    o->max_iters = 200;
    o->restart = 0;
    o->mg_reduction = 1e-3;
    o->mg_max_cycles = 20;
    o->mg_fixed_cycles = 0;
    o->mg_coarsest = 4;
    o->fixed_iters = 0;
    o->mg_strict = 0;
}

spp_status spp_shishkin_mesh(int32_t n, double eps, double sigma, double beta, double *x)
{
    if (!x || n < 4 || (n % 2) != 0 || !(eps > 0.0) || eps > 1.0 || !(sigma > 0.0) || !(beta > 0.0))
        FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_shishkin_mesh: bad arguments (n=%d eps=%g sigma=%g beta=%g)",
             n, eps, sigma, beta);
    // eq:tau 1D / eq:tau exponential
    double tau = sigma * eps * std::log((double)n) / beta;
    if (tau > 0.5) tau = 0.5;
    const int h = n / 2;
    const double w = tau / h, W = (1.0 - tau) / h;
    for (int i = 0; i < h; ++i) x[i] = i * w;
    x[h] = tau;
    for (int i = h + 1; i < n; ++i) x[i] = tau + (i - h) * W;
    x[n] = 1.0;
    return SPP_OK;
}

// SPP_TUNE="gs_tile_rows=128,gs_tile_cols=256,..." overrides kernel tunables (experiments only;
// every setting computes the same result to rounding).
static void parse_tune(Ctx *c)
{
    const char *env = getenv("SPP_TUNE");
    if (!env) return;
    std::string s(env);
    size_t pos = 0;
    while (pos < s.size()) {
        size_t end = s.find(',', pos);
        if (end == std::string::npos) end = s.size();
        const std::string kv = s.substr(pos, end - pos);
        const size_t eq = kv.find('=');
        if (eq != std::string::npos) {
            const std::string k = kv.substr(0, eq);
            const int v = atoi(kv.c_str() + eq + 1);
            if (k == "gs_warps") c->tune.gs_warps = v;
            else if (k == "gs_tile_cols") c->tune.gs_tile_cols = v;
            else if (k == "gs_max_halo") c->tune.gs_max_halo = v;
            else if (k == "sweep_warps") c->tune.sweep_warps = v;
            else if (k == "coarse_max") c->tune.coarse_max = v;
            else if (k == "gs_lag") c->tune.gs_lag = v;
            else if (k == "dist_levels") c->tune.dist_levels = v;
            else if (k == "rho_halo") c->tune.rho_halo = v;
        }
        pos = end + 1;
    }
}

// spp.h "Option validation": the combinations a dim does not implement are rejected, never
// silently replaced by other stopping semantics.
static spp_status check_options(const spp_options *o, int dim, Ctx *c)
{
    if (o->restart < 0) FAIL(c, SPP_E_ARG, "restart = %d must be >= 0", o->restart);
    if (o->restart > 0 && dim != 2) FAIL(c, SPP_E_ARG, "restart > 0 (FGMRES(m)) is implemented for 2D solves only");
    if (o->restart > 0 && o->fixed_iters > 0) FAIL(c, SPP_E_ARG, "restart > 0 with fixed_iters > 0 is not implemented");
    if (!(o->tol > 0.0) || !std::isfinite(o->tol)) FAIL(c, SPP_E_ARG, "tol must be finite and > 0");
    if (o->side != SPP_RIGHT_FLEXIBLE && o->side != SPP_LEFT) FAIL(c, SPP_E_ARG, "unknown side %d", (int)o->side);
    if ((int)o->stop < 0 || (int)o->stop > 3) FAIL(c, SPP_E_ARG, "unknown stop %d", (int)o->stop);
    if (dim == 2 && (o->side == SPP_LEFT || o->stop == SPP_STOP_ABS_MAX))
        FAIL(c, SPP_E_ARG, "2D solves are right/flexible FGMRES with a recurrence stop (SPP_LEFT / SPP_STOP_ABS_MAX are 1D only)");
    if (dim == 1 && ((o->side == SPP_LEFT) != (o->stop == SPP_STOP_ABS_MAX)))
        FAIL(c, SPP_E_ARG, "1D: side = SPP_LEFT goes with stop = SPP_STOP_ABS_MAX and only with it (P:828-833)");
    return SPP_OK;
}

// A mesh the library solves on: x[0] = 0, x[N] = 1, 0 < x[N/2] <= 1/2.  Either the piecewise-
// uniform Shishkin mesh broken at N/2 (*graded = 0: widths from the formula, R12), or
// -- when `allow_graded` (2D) -- any strictly increasing mesh with its transition point at index
// N/2 (a graded layer-adapted mesh such as Bakhvalov-Shishkin; *graded = 1:
// widths are coordinate differences, R21).
static spp_status check_mesh(const double *x, int N, double *tau, Ctx *c, bool allow_graded = false, int *graded = nullptr)
{
    if (!x) FAIL(c, SPP_E_ARG, "mesh coordinates are NULL");
    const int n = N / 2;
    const double t = x[n];
    if (graded) *graded = 0;
    if (x[0] != 0.0 || x[N] != 1.0 || !(t > 0.0) || !(t <= 0.5))
        FAIL(c, SPP_E_MESH, "mesh: need x[0]=0, x[N]=1, 0 < x[N/2] <= 1/2");
    const double h = t / n, H = (1.0 - t) / n;
    for (int i = 0; i <= N; ++i) {
        const double want = i <= n ? i * h : t + (i - n) * H;
        if (std::fabs(x[i] - want) > 1e-12 * (std::fabs(want) + h)) {
            if (!allow_graded)
                FAIL(c, SPP_E_MESH, "mesh: node %d = %.17g is not on the piecewise-uniform Shishkin mesh (want %.17g)",
                     i, x[i], want);
            for (int k = 1; k <= N; ++k)
                if (!(x[k] > x[k - 1]) || !std::isfinite(x[k]))
                    FAIL(c, SPP_E_MESH, "mesh: nodes must increase strictly (node %d = %.17g after %.17g)", k, x[k], x[k - 1]);
            if (graded) *graded = 1;
            break;
        }
    }
    *tau = t;
    return SPP_OK;
}

// bakhvalov-shishkin mesh on the host (spp.h)
spp_status spp_bakhvalov_mesh(int32_t n, double eps, double sigma, double beta, double *x)
{
    if (!x || n < 4 || (n % 2) != 0 || !(eps > 0.0) || eps > 1.0 || !(sigma > 0.0) || !(beta > 0.0))
        FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_bakhvalov_mesh: bad arguments (n=%d eps=%g sigma=%g beta=%g)", n, eps,
             sigma, beta);
    const double sc = sigma * eps / beta, tau = sc * std::log((double)n);
    if (tau > 0.5) {
        for (int i = 0; i <= n; ++i) x[i] = (double)i / n;
        x[n] = 1.0;
        return SPP_OK;
    }
    const int h = n / 2;
    x[0] = 0.0;
    for (int i = 1; i < h; ++i) x[i] = -sc * std::log(1.0 - 2.0 * (1.0 - 1.0 / n) * i / n);
    x[h] = tau;
    const double H = (1.0 - tau) / h;
    for (int i = h + 1; i < n; ++i) x[i] = tau + (i - h) * H;
    x[n] = 1.0;
    return SPP_OK;
}

// The mesh-only device arrays (once per context): the widths h_i, k_j of the 2D operator and,
// per corner level, the widths of its 1D meshes and the geometric interpolation weights from the
// next coarser level.  On a Shishkin mesh every value is the formula's (R8, R12: widths tau/n,
// (1-tau)/n, 2^l tau/n; weights 1/2 exactly), so the kernels compute what they computed from the
// scalar widths; on a graded mesh they are coordinate differences (R21), as in the oracle.
static spp_status set_mesh_arrays(Ctx *c)
{
    const int N = c->N, n = c->n;
    std::vector<double> wx(N + 2, 0.0), wy(N + 2, 0.0);
    for (int i = 1; i <= N; ++i) {
        wx[i] = c->gx ? c->xh[i] - c->xh[i - 1] : (i <= n ? c->hx : c->Hx);
        wy[i] = c->gy ? c->yh[i] - c->yh[i - 1] : (i <= n ? c->hy : c->Hy);
    }
    CK(c, cudaMemcpy(c->wxd, wx.data(), sizeof(double) * (N + 2), cudaMemcpyHostToDevice));
    CK(c, cudaMemcpy(c->wyd, wy.data(), sizeof(double) * (N + 2), cudaMemcpyHostToDevice));
    for (int l = 0; l < c->L; ++l) {
        Level &Lv = c->lev[l];
        const int nl = Lv.n, step = 1 << l;
        std::vector<double> lw[2] = {std::vector<double>(nl + 2, 0.0), std::vector<double>(nl + 2, 0.0)};
        std::vector<double> wt(4 * (size_t)(nl + 2), 0.0);
        for (int a = 0; a < 2; ++a) {
            const bool g = a == 0 ? c->gx : c->gy;
            const std::vector<double> &X = a == 0 ? c->xh : c->yh;
            const double h = a == 0 ? c->hx : c->hy, H = a == 0 ? c->Hx : c->Hy;
            for (int q = 1; q <= nl; ++q) lw[a][q] = g ? X[q * step] - X[(q - 1) * step] : h * step;
            lw[a][nl + 1] = g ? X[n + 1] - X[n] : H;
            double *wl = wt.data() + (size_t)(2 * a) * (nl + 2), *wr = wl + (nl + 2);
            for (int q = 1; q < nl; q += 2) {          // odd node q between q-1 and q+1
                const double u = lw[a][q], v = lw[a][q + 1];
                wl[q] = u == v ? 0.5 : v / (u + v);
                wr[q] = u == v ? 0.5 : u / (u + v);
            }
        }
        CK(c, cudaMemcpy(Lv.lwx, lw[0].data(), sizeof(double) * (nl + 2), cudaMemcpyHostToDevice));
        CK(c, cudaMemcpy(Lv.lwy, lw[1].data(), sizeof(double) * (nl + 2), cudaMemcpyHostToDevice));
        CK(c, cudaMemcpy((double *)Lv.w.xl, wt.data(), sizeof(double) * 4 * (nl + 2), cudaMemcpyHostToDevice));
        bool uni = true;                               // all 1/2: the kernels skip the loads
        for (int a = 0; a < 4; ++a)
            for (int q = 1; q < nl; q += 2) uni = uni && wt[(size_t)a * (nl + 2) + q] == 0.5;
        Lv.w.uni = uni ? 1 : 0;
    }
    return SPP_OK;
}

static spp_status alloc_all(Ctx *c)
{
    const int N = c->N;
    if (c->dim == 1) return SPP_OK;   // 1D allocates in k_1d.cu's setup
    const int n = c->n, m = c->m;
    c->P = round_up(N + 1, 16);
    c->G = (size_t)(N + 1) * c->P;
    const size_t G = c->G;
    // kTmaSlack: the sheared TMA boxes of k_wave may read a few dozen elements past the last row
    CK(c, cudaMalloc(&c->coef_block, sizeof(double) * (8 * G + 2 * (N + 1) + 2 * (N + 2) + kTmaSlack)));
    CK(c, cudaMemsetAsync(c->coef_block, 0, sizeof(double) * (8 * G + 2 * (N + 1) + 2 * (N + 2) + kTmaSlack), c->st));
    c->aE = c->coef_block; c->aN = c->aE + G; c->rr = c->aN + G;
    c->ca = c->rr + G; c->cn = c->ca + G; c->cd = c->cn + G;
    c->ya = c->cd + G; c->yn = c->ya + G;
    c->aW = c->yn + G; c->aS = c->aW + (N + 1);
    c->wxd = c->aS + (N + 1); c->wyd = c->wxd + (N + 2);
    const size_t per = (size_t)(n - 1) * n;
    CK(c, cudaMalloc(&c->fac, sizeof(double) * (8 * per + 4 * (size_t)n)));
    c->tX = c->fac + 8 * per; c->tY = c->tX + n; c->kapX = c->tY + n; c->kapY = c->kapX + n;
    const size_t cb = std::max<size_t>(3 * (size_t)m * m, 2 * per);
    CK(c, cudaMalloc(&c->cbuf, sizeof(double) * cb));
    // Krylov work vectors
    CK(c, cudaMalloc(&c->w, sizeof(double) * (4 * G + kTmaSlack)));
    CK(c, cudaMemsetAsync(c->w, 0, sizeof(double) * (4 * G + kTmaSlack), c->st));
    c->F = c->w + G; c->U = c->F + G; c->T1 = c->U + G;
    const int maxit = c->opt.max_iters;
    // reduction partials: one kRedBlocks segment per strip (nparts) in every slot
    CK(c, cudaMalloc(&c->part, sizeof(double) * (size_t)(std::max(maxit, 3 * kMaxLevels) + 8) * kRedBlocks * c->nparts));
    CK(c, cudaMalloc(&c->dscal, sizeof(double) * (size_t)(3 * maxit + 64)));
    CK(c, cudaMallocHost(&c->hpin, sizeof(double) * std::max<size_t>(8 * (size_t)kRedBlocks * c->nparts + 4 * (size_t)maxit + 64,
                                                                      (size_t)kMaxLevels * kRedBlocks)));
    CK(c, cudaMalloc(&c->flags, sizeof(int) * 256));
    CK(c, cudaMemsetAsync(c->flags, 0, sizeof(int) * 256, c->st));
    CK(c, cudaMalloc(&c->mgs, sizeof(MGState)));
    CK(c, cudaMallocHost(&c->hmgs, sizeof(MGState)));
    {
        const char *ng = getenv("SPP_NO_GRAPH");
        c->use_graph = !(ng && ng[0] == '1');
        const char *nig = getenv("SPP_NO_ITER_GRAPH");
        c->fg_ok = (nig && nig[0] == '1') ? 0 : 1;
        const char *nl = getenv("SPP_NO_LINES_TMA");
        c->no_lines_tma = (nl && nl[0] == '1') ? 1 : 0;
        const char *yf = getenv("SPP_MG_YFORM");
        c->mg_zform = (yf && yf[0] == '1') ? 0 : 1;
    }
    {   // exact chained sweep: one progress flag and one inflow row per CTA (the launch's CTA
        // count, wave_chain_ctas), plus the inflow slot of a row strip's chain
        const long ncta = wave_chain_ctas(c, n) + 2;
        c->chain_ld = n + 32;
        CK(c, cudaMalloc(&c->chain, sizeof(double) * (size_t)(ncta * c->chain_ld)));
        CK(c, cudaMalloc(&c->chain_flags, sizeof(int) * (size_t)(ncta + 1)));
    }
    // corner MG levels (levels until <= mg_coarsest per axis)
    int nl = n, L = 1;
    const int coarsest = c->opt.mg_coarsest > 0 ? c->opt.mg_coarsest : 4;
    while (nl > coarsest && L < kMaxLevels) { nl /= 2; L++; }
    c->L = L;
    size_t tot = 0;
    for (int l = 0; l < L; ++l) {
        Level &Lv = c->lev[l];
        Lv.n = n >> l;
        Lv.slo = 1; Lv.shi = Lv.n; Lv.shalo = 0; Lv.sdist = false;
        Lv.pitch = round_up(Lv.n + 2, 16);
        Lv.elems = (size_t)(Lv.n + 2) * Lv.pitch;
        tot += 5 * Lv.elems + 10 * (size_t)(Lv.n + 2) + (l > 0 ? 6 * Lv.elems : 0);
    }
    tot += 3 * c->lev[0].elems;   // Zc, Zc2, Bc
    tot += kTmaSlack;
    CK(c, cudaMalloc(&c->mg_block, sizeof(double) * tot));
    CK(c, cudaMemsetAsync(c->mg_block, 0, sizeof(double) * tot, c->st));
    double *p = c->mg_block;
    for (int l = 0; l < L; ++l) {
        Level &Lv = c->lev[l];
        Lv.b = p; p += Lv.elems; Lv.e = p; p += Lv.elems; Lv.q = p; p += Lv.elems; Lv.rho = p; p += Lv.elems;
        Lv.g = p; p += Lv.elems;
        Lv.aW = p; p += Lv.n + 2; Lv.aS = p; p += Lv.n + 2; Lv.hb = p; p += Lv.n + 2; Lv.kb = p; p += Lv.n + 2;
        Lv.lwx = p; p += Lv.n + 2; Lv.lwy = p; p += Lv.n + 2;
        {
            double *w4 = p; p += 4 * (size_t)(Lv.n + 2);
            Lv.w = Wts{w4, w4 + (Lv.n + 2), w4 + 2 * (Lv.n + 2), w4 + 3 * (Lv.n + 2), 1};
        }
        if (l > 0) {
            Lv.own = p;
            double *aE = p; p += Lv.elems; double *aN = p; p += Lv.elems; double *rr = p; p += Lv.elems;
            double *ya = p; p += Lv.elems; double *yn = p; p += Lv.elems; double *cd = p; p += Lv.elems;
            Lv.aE = aE; Lv.aN = aN; Lv.rr = rr; Lv.ya = ya; Lv.yn = yn; Lv.cd = cd;
            Lv.cpitch = Lv.pitch;
        } else {
            Lv.aE = c->aE; Lv.aN = c->aN; Lv.rr = c->rr; Lv.ya = c->ya; Lv.yn = c->yn; Lv.cd = c->cd;
            Lv.cpitch = c->P;
        }
    }
    c->Zc = p; p += c->lev[0].elems;
    c->Zc2 = p; p += c->lev[0].elems;
    c->Bc = p; p += c->lev[0].elems;
    return set_mesh_arrays(c);
}

}  // extern "C"
namespace spp {
cudaError_t ensure_vectors(Ctx *c, int k)
{
    // V[0..k], Z[0..k-1]
    while ((int)c->V.size() <= k) {
        double *p = nullptr;
        cudaError_t e = cudaMalloc(&p, sizeof(double) * (c->G + kTmaSlack));
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(p, 0, sizeof(double) * (c->G + kTmaSlack), c->st);
        if (e != cudaSuccess) return e;
        c->V.push_back(p);
    }
    while ((int)c->Z.size() < k) {
        double *p = nullptr;
        cudaError_t e = cudaMalloc(&p, sizeof(double) * (c->G + kTmaSlack));
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(p, 0, sizeof(double) * (c->G + kTmaSlack), c->st);
        if (e != cudaSuccess) return e;
        c->Z.push_back(p);
    }
    return cudaSuccess;
}

spp_status setup_2d_ctx(Ctx *c, const double *c1, const double *c2, const double *r, spp_mem mem)
{
    const int N = c->N, m = c->m;
    const size_t mm = (size_t)m * m;
    const double *d1 = c1, *d2 = c2, *d3 = r;
    cudaEvent_t e0, e1;
    CK(c, cudaEventCreate(&e0));
    CK(c, cudaEventCreate(&e1));
    CK(c, cudaEventRecord(e0, c->st));
    if (mem == SPP_HOST) {
        CK(c, cudaMemcpyAsync(c->cbuf, c1, sizeof(double) * mm, cudaMemcpyHostToDevice, c->st));
        CK(c, cudaMemcpyAsync(c->cbuf + mm, c2, sizeof(double) * mm, cudaMemcpyHostToDevice, c->st));
        CK(c, cudaMemcpyAsync(c->cbuf + 2 * mm, r, sizeof(double) * mm, cudaMemcpyHostToDevice, c->st));
        d1 = c->cbuf; d2 = c->cbuf + mm; d3 = c->cbuf + 2 * mm;
    }
    int *bad = c->flags + 200;
    CK(c, cudaMemsetAsync(bad, 0, sizeof(int), c->st));
    k_coef_1d<<<nblk(N + 1), 256, 0, c->st>>>(N, c->eps, c->wxd, c->wyd, c->aW, c->aS);
    const int want_y = (!c->mg_zform || !c->weighted) ? 1 : 0;
    c->y0_ok = want_y;
    k_coef_2d<<<nblk((long)mm), 256, 0, c->st>>>(N, c->P, c->eps, c->wxd, c->wyd, d1, d2, d3, c->aW,
                                                c->aS, c->aE, c->aN, c->rr, c->ca, c->cn, c->cd, c->ya, c->yn, want_y, bad);
    Level &L0 = c->lev[0];
    k_level0_1d<<<1, 256, 0, c->st>>>(N, c->wxd, c->wyd, c->aW, c->aS, L0.aW, L0.aS, L0.hb, L0.kb);
    c->launches += 3;
    for (int l = 1; l < c->L; ++l) {
        Level &Lv = c->lev[l];
        // (k_coef_level writes aE/D, aN/D into ya, yn; launch_ycoef then replaces them by the
        // y-form couplings aE/D_E, aN/D_N once the whole cd of the level exists)
        k_coef_level<<<nblk((long)Lv.n * Lv.n), 256, 0, c->st>>>(N, Lv.n, 1 << l, Lv.pitch, c->eps, Lv.lwx, Lv.lwy,
            d1, d2, d3, Lv.aW, Lv.aS, Lv.hb, Lv.kb, (double *)Lv.aE, (double *)Lv.aN,
            (double *)Lv.rr, (double *)Lv.ya, (double *)Lv.yn, (double *)Lv.cd);
        c->launches++;
        if (!c->mg_zform) launch_ycoef(c, Lv.n, Lv.pitch, Lv.aE, Lv.aN, Lv.cd, (double *)Lv.ya, (double *)Lv.yn);
    }
    int hbad = 0;
    CK(c, cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c->st));
    // one host synchronisation for the validation flags, the line chains' contraction factors and
    // the MG levels' (their kernels run on whatever coefficients arrived; a rejected set is
    // reported before anything is planned from them)
    CK(c, setup_lines_launch(c));
    CK(c, setup_mg_tiles_launch(c));
    CK(c, cudaStreamSynchronize(c->st));
    if (hbad & 1) FAIL(c, SPP_E_COEF, "coefficients violate c1 > 0, c2 >= 0, r >= 0 or are not finite (P:208-212, P:907)");
    if ((hbad & 6) == 6)
        FAIL(c, SPP_E_COEF, "c2 must be > 0 everywhere (two exponential layers) or = 0 everywhere (a parabolic layer, "
                            "P:872-878)");
    c->par = (hbad & 4) ? 1 : 0;
    if (c->par && c->dist) FAIL(c, SPP_E_ARG, "row strips: the parabolic-layer corner (c2 = 0) runs on one GPU only");
    if (c->par) {                                       // NEXT-2: semi-coarsening Galerkin corner MG
        if (!c->par_block) CK(c, par_alloc(c));
        CK(c, setup_lines_plan(c));
        CK(c, par_setup(c));
        CK(c, cudaEventRecord(e1, c->st));
        CK(c, cudaEventSynchronize(e1));
        cudaEventElapsedTime(&c->setup_ms, e0, e1);
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        CK(c, cudaGetLastError());
        return SPP_OK;
    }
    CK(c, setup_lines_plan(c));
    CK(c, setup_mg_tiles_plan(c));
    CK(c, cudaEventRecord(e1, c->st));
    CK(c, cudaEventSynchronize(e1));
    cudaEventElapsedTime(&c->setup_ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CK(c, cudaGetLastError());
    return SPP_OK;
}

}  // namespace spp
extern "C" {

spp_status spp_setup(spp_ctx *cx, const double *c1, const double *c2, const double *r, spp_mem mem)
{
    Ctx *c = (Ctx *)cx;
    NvtxScope nvs("spp_setup");
    if (!c) FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_setup: NULL context");
    if (!c1 || !r || (c->dim == 2 && !c2)) FAIL(c, SPP_E_ARG, "spp_setup: NULL coefficient array");
    if (c->dim == 1) return (spp_status)setup_1d(c, c1, r, mem);
    if (c->dist) return setup_dist(c, c1, c2, r, mem);
    return setup_2d_ctx(c, c1, c2, r, mem);
}

// Host-side validation of a problem + options and a fresh (unallocated) context with the mesh
// widths set.  Everything here runs without a device, so argument errors are reported the same
// way with or without a GPU.
static spp_status ctx_new(const spp_problem *p, const spp_options *o, void *stream, Ctx **out)
{
    *out = nullptr;
    const int N = p->n;
    if (p->dim != 1 && p->dim != 2) FAIL((Ctx *)nullptr, SPP_E_ARG, "dim must be 1 or 2");
    if (N < 4 || (N % 2)) FAIL((Ctx *)nullptr, SPP_E_ARG, "N must be even and >= 4 (got %d)", N);
    if (p->dim == 2 && (N < 8 || ((N / 2) & (N / 2 - 1))))
        FAIL((Ctx *)nullptr, SPP_E_ARG, "2D needs N >= 8 with N/2 a power of two (got %d)", N);
    if (!(p->eps > 0.0) || p->eps > 1.0) FAIL((Ctx *)nullptr, SPP_E_ARG, "eps must be in (0,1]");
    spp_options opt;
    if (o) opt = *o; else spp_default_options(p->dim, &opt);
    spp_status s = check_options(&opt, p->dim, nullptr);
    if (s != SPP_OK) return s;
    double tx = 0, ty = 0;
    int gx = 0, gy = 0;
    if ((s = check_mesh(p->x, N, &tx, nullptr, p->dim == 2, &gx)) != SPP_OK) return s;
    if (p->dim == 2 && (s = check_mesh(p->y, N, &ty, nullptr, true, &gy)) != SPP_OK) return s;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        FAIL((Ctx *)nullptr, SPP_E_CUDA, "spp_create: no CUDA device (this library has no CPU path)");
    Ctx *c = new (std::nothrow) Ctx();
    if (!c) FAIL((Ctx *)nullptr, SPP_E_NOMEM, "host allocation failed");
    c->dim = p->dim; c->N = N; c->n = N / 2; c->m = N - 1; c->eps = p->eps;
    c->st = (cudaStream_t)stream;
    c->opt = opt;
    if (c->opt.max_iters < 1) c->opt.max_iters = 1;
    if (c->opt.mg_max_cycles < 1) c->opt.mg_max_cycles = 20;
    if (!(c->opt.mg_reduction > 0.0)) c->opt.mg_reduction = 1e-3;
    c->weighted = c->opt.stop == SPP_STOP_REL_JACOBI ? 1 : 0;
    parse_tune(c);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (wave_init() != cudaSuccess || lines_init() != cudaSuccess) { delete c; FAIL((Ctx *)nullptr, SPP_E_CUDA, "kernel attribute setup failed"); }
    c->tx = tx; c->ty = ty;
    c->hx = tx / c->n; c->Hx = (1.0 - tx) / c->n;
    c->hy = ty / c->n; c->Hy = (1.0 - ty) / c->n;
    c->xh.assign(p->x, p->x + N + 1);
    if (p->dim == 2) c->yh.assign(p->y, p->y + N + 1);
    c->gx = gx; c->gy = gy;
    *out = c;
    return SPP_OK;
}

spp_status spp_create(const spp_problem *p, const spp_options *o, void *stream, spp_ctx **out)
{
    if (!p || !out) FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_create: NULL argument");
    *out = nullptr;
    Ctx *c = nullptr;
    spp_status s = ctx_new(p, o, stream, &c);
    if (s != SPP_OK) return s;
    if ((s = alloc_all(c)) != SPP_OK) { g_err = c->err; spp_destroy((spp_ctx *)c); return s; }
    if ((s = spp_setup((spp_ctx *)c, p->c1, p->c2, p->r, p->mem)) != SPP_OK) {
        g_err = c->err;
        spp_destroy((spp_ctx *)c);
        return s;
    }
    *out = (spp_ctx *)c;
    return SPP_OK;
}

static void ctx_free(Ctx *c);
void spp_destroy(spp_ctx *cx)
{
    Ctx *c = (Ctx *)cx;
    if (!c) return;
    if (c->dist) {                                      // row strips: every local strip, then the decomposition
        Dist *d = c->dist;
        std::vector<Ctx *> all = d->cx;
        if (d->st) cudaStreamSynchronize(d->st);
        destroy_dist(c);
        for (Ctx *x : all) { x->dist = nullptr; ctx_free(x); }
        return;
    }
    ctx_free(c);
}

static void ctx_free(Ctx *c)
{
    if (c->st) cudaStreamSynchronize(c->st); else cudaDeviceSynchronize();
    for (double *p : c->V) cudaFree(p);
    for (double *p : c->Z) cudaFree(p);
    cudaFree(c->coef_block); cudaFree(c->fac); cudaFree(c->cbuf); cudaFree(c->w);
    cudaFree(c->part); cudaFree(c->dscal); cudaFree(c->flags); cudaFree(c->mg_block);
    cudaFree(c->chain); cudaFree(c->chain_flags); cudaFree(c->par_block);
    cudaFree(c->d_chunks); cudaFree(c->d1);
    if (c->hpin) cudaFreeHost(c->hpin);
    corner_graph_destroy(c);
    fg_destroy(c);
    cudaFree(c->fgh); cudaFree(c->fgd);
    if (c->hfgh) cudaFreeHost(c->hfgh);
    if (c->cap_st) cudaStreamDestroy(c->cap_st);
    cudaFree(c->mgs);
    if (c->hmgs) cudaFreeHost(c->hmgs);
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    delete c;
}

int64_t spp_kernel_launches(const spp_ctx *cx) { return cx ? ((const Ctx *)cx)->launches : 0; }

int32_t spp_mg_levels(const spp_ctx *cx) { return cx ? ((const Ctx *)cx)->L : 0; }
int32_t spp_mg_level_n(const spp_ctx *cx, int32_t l)
{
    const Ctx *c = (const Ctx *)cx;
    return (c && l >= 0 && l < c->L) ? c->lev[l].n : 0;
}

spp_status spp_profile_enable(spp_ctx *cx, int32_t en)
{
    Ctx *c = (Ctx *)cx;
    if (!c) return SPP_E_ARG;
    c->prof_on = en ? (en == 1 ? 0xfff : en) : 0;
    return SPP_OK;
}
spp_status spp_profile_reset(spp_ctx *cx)
{
    Ctx *c = (Ctx *)cx;
    if (!c) return SPP_E_ARG;
    for (auto &r : c->prof) r = ProfRec();
    return SPP_OK;
}
spp_status spp_profile_get(const spp_ctx *cx, int32_t k, int64_t *launches, double *ms, double *bytes)
{
    const Ctx *c = (const Ctx *)cx;
    if (!c || k < 0 || k >= SPP_PROF_CLASSES) return SPP_E_ARG;
    if (launches) *launches = c->prof[k].launches;
    if (ms) *ms = c->prof[k].ms;
    if (bytes) *bytes = c->prof[k].bytes;
    return SPP_OK;
}

// ------------------------------------------------------------------------------------------ solve (2D)
static spp_status solve_2d(Ctx *c, const double *f, double *u, spp_mem mem, double *hist, int hcap,
                           spp_stats *st)
{
    const int m = c->m, maxit = c->opt.max_iters;
    const long G = (long)c->G;
    const size_t mm = (size_t)m * m;
    const int64_t launches0 = c->launches;
    cudaEvent_t e0, e1;
    CK(c, cudaEventCreate(&e0));
    CK(c, cudaEventCreate(&e1));
    CK(c, cudaEventRecord(e0, c->st));
    // f -> padded F
    const double *fd = f;
    if (mem == SPP_HOST) {
        CK(c, cudaMemcpyAsync(c->cbuf, f, sizeof(double) * mm, cudaMemcpyHostToDevice, c->st));
        fd = c->cbuf;
    }
    k_pack<<<nblk((long)mm), 256, 0, c->st>>>(m, c->P, fd, c->F, 1, m);
    c->launches++;
    CK(c, ensure_vectors(c, 1));
    const int weighted = c->weighted;
    const int stop = c->opt.stop;
    // v0 = W f / beta
    {
        ProfScope ps(c, 7, 48.0 * mm);
        k_rhs<<<red_grid((long)m * m), kRedThreads, 0, c->st>>>(m, c->P, c->F, c->aE, c->aN, c->rr, c->aW, c->aS, weighted,
                                                     c->V[0], part_slot(c, 0), 1, m);
        c->launches++;
    }
    double bsq = 0;
    CK(c, fetch_sum(c, part_slot(c, 0), &bsq));
    const double beta = std::sqrt(bsq);
    if (!std::isfinite(beta)) FAIL(c, SPP_E_NONFINITE, "||W f|| is not finite (NaN/Inf in the right-hand side)");
    std::vector<double> H((size_t)(maxit + 1) * (maxit + 1), 0.0), cs(maxit + 1), sn(maxit + 1),
        g(maxit + 2, 0.0), yv(maxit + 1);
    if (hist && hcap > 0) hist[0] = beta;
    int iters = 0, converged = 0, mg_tot = 0, mg_min = 1 << 30, mg_max = 0, caps = 0;
    double resf = beta;
    const double target = (stop == SPP_STOP_ABS_L2) ? c->opt.tol : c->opt.tol * beta;
    CK(c, cudaMemsetAsync(c->U, 0, sizeof(double) * G, c->st));
    // FGMRES (restart = 0, the paper) or FGMRES(m) (reading R23): cycles of at most mr Arnoldi
    // steps; after a cycle without convergence x += sum_j y_j z_j and the next cycle starts from
    // the true residual W (f - A x), the stopping target staying the initial one
    const int mr = (c->opt.restart > 0 && c->opt.restart < maxit) ? c->opt.restart : maxit;
    double bc = beta;                                   // the cycle's initial residual
    int stopped = 0;
    if (beta == 0.0) converged = 1;
    for (int cycle = 0; !converged && !stopped && iters < maxit; ++cycle) {
        if (cycle > 0) {                                // restart vector v0 = W (f - A x) / ||.||
            k_spmv<<<red_grid((long)m * m), kRedThreads, 0, c->st>>>(m, c->P, c->U, c->aE, c->aN, c->rr, c->aW, c->aS,
                                                                      0, c->w, nullptr, nullptr, 1, m);
            k_rhs<<<red_grid((long)m * m), kRedThreads, 0, c->st>>>(m, c->P, c->F, c->aE, c->aN, c->rr, c->aW, c->aS,
                                                                     weighted, c->V[0], part_slot(c, 0), 1, m, c->w);
            c->launches += 2;
            double s2 = 0;
            CK(c, fetch_sum(c, part_slot(c, 0), &s2));
            bc = std::sqrt(s2);
            if (!std::isfinite(bc)) FAIL(c, SPP_E_NONFINITE, "restart residual is not finite after %d iterations", iters);
            if (bc == 0.0) { converged = 1; break; }
        }
        const int steps = std::min(mr, maxit - iters);  // Arnoldi steps of this cycle at most
        int kk = 0;                                     // steps taken in this cycle
        k_scale<<<nblk(G / 2), 256, 0, c->st>>>(G, c->V[0], 1.0 / bc);
        c->launches++;
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = bc;
        const int ld = maxit + 1;
        if (fg_mode(c)) {                               // iteration graphs, one sync per batch
            CK(c, fg_alloc(c));
            const std::vector<long> sig = fg_signature(c);
            if (c->itg_sig != sig) { fg_destroy(c); c->itg_sig = sig; }
            k_fg_init<<<1, 1, 0, c->st>>>(c->fgh, fg_arr(c, 2), fg_arr(c, 3), bc, target);
            c->launches++;
            int launched = 0;
            int batch = std::max(1, std::min(steps, c->last_iters > 0 ? c->last_iters : 4));
            for (;;) {
                for (int b = 0; b < batch && launched < steps; ++b, ++launched) {
                    const int k = launched;
                    CK(c, ensure_vectors(c, k + 1));
                    if ((int)c->itg.size() <= k) c->itg.resize(k + 1, nullptr);
                    if (!c->itg[k]) CK(c, fg_build(c, k, &c->itg[k]));
                    CK(c, cudaGraphLaunch(c->itg[k], c->st));
                    c->launches++;                      // the gate
                }
                CK(c, cudaMemcpyAsync(c->hfgh, c->fgh, sizeof(FGHead), cudaMemcpyDeviceToHost, c->st));
                CK(c, cudaStreamSynchronize(c->st));
                if (c->hfgh->stop || launched >= steps) break;
                batch = 8;
            }
            const FGHead fs = *c->hfgh;
            if (fs.nonfinite)
                FAIL(c, SPP_E_NONFINITE, "Hessenberg entry h(%d,%d) is not finite at iteration %d", fs.nf_j, fs.k - 1, iters + fs.k);
            if (fs.capfail) FAIL(c, SPP_E_MG_CAP, "corner multigrid hit the cycle cap (%d)", c->opt.mg_max_cycles);
            kk = fs.k; converged = fs.converged; stopped = fs.stop; resf = fs.res;
            mg_tot += fs.mg_tot; mg_min = std::min(mg_min, fs.mg_min); mg_max = std::max(mg_max, fs.mg_max); caps += fs.caps;
            for (int k = 0; k < kk; ++k) c->launches += c->itg_launches[k];
            c->launches += (int64_t)fs.mg_tot * c->cg_body_launches;
            CK(c, cudaMemcpyAsync(H.data(), fg_H(c), sizeof(double) * (size_t)kk * ld, cudaMemcpyDeviceToHost, c->st));
            CK(c, cudaMemcpyAsync(g.data(), fg_arr(c, 2), sizeof(double) * (kk + 1), cudaMemcpyDeviceToHost, c->st));
            if (hist && hcap > iters + 1)
                CK(c, cudaMemcpyAsync(hist + iters + 1, fg_arr(c, 3) + 1, sizeof(double) * std::min(kk, hcap - 1 - iters),
                                      cudaMemcpyDeviceToHost, c->st));
            CK(c, cudaStreamSynchronize(c->st));
        } else
        for (int k = 0; k < steps; ++k) {
            CK(c, ensure_vectors(c, k + 1));
            int cap = 0;
            cudaError_t err = cudaSuccess;
            int cyc = apply_precond(c, c->V[k], c->Z[k], &cap, &err);
            CK(c, err);
            if (cyc >= 0) {
                if (cap && c->opt.mg_strict) FAIL(c, SPP_E_MG_CAP, "corner multigrid hit the cycle cap (%d)", c->opt.mg_max_cycles);
                mg_tot += cyc; mg_min = std::min(mg_min, cyc); mg_max = std::max(mg_max, cyc); caps += cap;
            }
            krylov_tail(c, k);
            if (cyc < 0) CK(c, cudaMemcpyAsync(c->hmgs, c->mgs, sizeof(MGState), cudaMemcpyDeviceToHost, c->st));
            CK(c, cudaMemcpyAsync(c->hpin, c->dscal, sizeof(double) * (k + 2), cudaMemcpyDeviceToHost, c->st));
            CK(c, cudaStreamSynchronize(c->st));
            if (cyc < 0) {                              // corner graph: this apply's cycle count
                cyc = c->hmgs->cycles; cap = c->hmgs->cap;
                c->launches += (int64_t)cyc * c->cg_body_launches;
                if (cap && c->opt.mg_strict) FAIL(c, SPP_E_MG_CAP, "corner multigrid hit the cycle cap (%d)", c->opt.mg_max_cycles);
                mg_tot += cyc; mg_min = std::min(mg_min, cyc); mg_max = std::max(mg_max, cyc); caps += cap;
            }
            double *h = &H[(size_t)k * ld];
            for (int j = 0; j <= k + 1; ++j) {
                h[j] = c->hpin[j];
                // SURVEY 5 "NaN/Inf guard on h_{k+1,k}": a non-finite Hessenberg entry is a
                // failure (non-finite data or a preconditioner blow-up), never a breakdown
                if (!std::isfinite(h[j]))
                    FAIL(c, SPP_E_NONFINITE, "Hessenberg entry h(%d,%d) is not finite at iteration %d", j, k, iters + k + 1);
            }
            int brk = 0;
            const double res = givens_update(h, cs.data(), sn.data(), g.data(), k, &brk);
            kk = k + 1;
            resf = res;
            if (hist && iters + k + 1 < hcap) hist[iters + k + 1] = res;
            // the cycle's last step ends it without a verdict (maxit = steps); a stop before it is final
            const int fin = fg_stop(k, res, brk, target, c->opt.fixed_iters, steps, &converged);
            if (fin && (converged || brk || c->opt.fixed_iters > 0 || k + 1 < steps)) stopped = 1;
            if (fin) break;
        }
        // y = R^{-1} g;  x (+)= sum_j y_j z_j
        for (int i = kk - 1; i >= 0; --i) {
            double t = g[i];
            for (int j = i + 1; j < kk; ++j) t -= H[(size_t)j * (maxit + 1) + i] * yv[j];
            yv[i] = t / H[(size_t)i * (maxit + 1) + i];
        }
        // device copies of the Z pointers and y (pinned staging, pre-allocated device slots)
        const double **hz = (const double **)(c->hpin + 4 * kRedBlocks);
        double *hy = c->hpin + 4 * kRedBlocks + maxit + 8;
        if (cycle > 0) CK(c, cudaStreamSynchronize(c->st));   // staging of the last cycle's copies
        for (int j = 0; j < kk; ++j) { hz[j] = c->Z[j]; hy[j] = yv[j]; }
        const double **dptr = (const double **)(c->dscal + maxit + 8);
        double *dy = c->dscal + 2 * maxit + 16;
        CK(c, cudaMemcpyAsync(dptr, hz, sizeof(double *) * kk, cudaMemcpyHostToDevice, c->st));
        CK(c, cudaMemcpyAsync(dy, hy, sizeof(double) * kk, cudaMemcpyHostToDevice, c->st));
        {
            ProfScope ps(c, 7, 8.0 * G * (kk + 1));
            k_update_x<<<nblk(G / 2), 256, 0, c->st>>>(G, kk, dptr, dy, c->U, cycle > 0 ? 1 : 0);
            c->launches++;
        }
        iters += kk;
    }
    c->last_iters = std::min(iters, mr);
    if (c->sticky != cudaSuccess) { const cudaError_t se = c->sticky; c->sticky = cudaSuccess; CK(c, se); }
    CK(c, cudaEventRecord(e1, c->st));
    // output
    if (u) {
        if (mem == SPP_HOST) {
            k_unpack<<<nblk((long)mm), 256, 0, c->st>>>(m, c->P, c->U, c->cbuf, 1, m);
            CK(c, cudaMemcpyAsync(u, c->cbuf, sizeof(double) * mm, cudaMemcpyDeviceToHost, c->st));
        } else {
            k_unpack<<<nblk((long)mm), 256, 0, c->st>>>(m, c->P, c->U, u, 1, m);
        }
        c->launches++;
    }
    CK(c, cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    // statistics: true residuals (after the timed region)
    if (st) {
        memset(st, 0, sizeof(*st));
        k_spmv<<<kRedBlocks, kRedThreads, 0, c->st>>>(m, c->P, c->U, c->aE, c->aN, c->rr, c->aW, c->aS, 0, c->w,
                                                      nullptr, nullptr, 1, m);
        k_resid_stats<<<kRedBlocks, kRedThreads, 0, c->st>>>(m, c->P, c->F, c->w, c->aE, c->aN, c->rr, c->aW, c->aS,
                                                             c->part, kRedBlocks, 1, m);
        CK(c, cudaMemcpyAsync(c->hpin, c->part, sizeof(double) * 4 * kRedBlocks, cudaMemcpyDeviceToHost, c->st));
        CK(c, cudaStreamSynchronize(c->st));
        const double s0 = host_sum(c->hpin, kRedBlocks), s1 = host_sum(c->hpin + kRedBlocks, kRedBlocks);
        const double s2 = host_sum(c->hpin + 2 * kRedBlocks, kRedBlocks), s3 = host_sum(c->hpin + 3 * kRedBlocks, kRedBlocks);
        st->true_res_l2_rel = s2 > 0 ? std::sqrt(s0 / s2) : 0.0;
        st->true_res_jacobi_rel = s3 > 0 ? std::sqrt(s1 / s3) : 0.0;
        st->iters = iters; st->converged = converged;
        st->mg_cycles_total = mg_tot; st->mg_cycles_min = iters ? mg_min : 0; st->mg_cycles_max = mg_max;
        st->mg_cap_hits = caps; st->applies = iters;
        st->kernel_launches = (int32_t)(c->launches - launches0);
        st->res0 = beta; st->res_final = resf;
        st->setup_s = c->setup_ms * 1e-3; st->solve_s = ms * 1e-3;
    }
    prof_collect(c);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    CK(c, cudaGetLastError());
    return converged ? SPP_OK : SPP_NOT_CONVERGED;
}

spp_status spp_solve(spp_ctx *cx, const double *f, double *u, spp_mem mem, double *hist, int32_t hcap,
                     spp_stats *st)
{
    Ctx *c = (Ctx *)cx;
    NvtxScope nvs("spp_solve");
    if (!c) FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_solve: NULL context");
    if (!f) FAIL(c, SPP_E_ARG, "spp_solve: NULL rhs");
    if (c->dim == 1) return (spp_status)solve_1d_abi(c, f, u, mem, hist, hcap, st);
    if (c->dist) return solve_dist(c, f, u, mem, hist, hcap, st);
    return solve_2d(c, f, u, mem, hist, hcap, st);
}

// ------------------------------------------------------------------------------------------ test hooks
spp_status spp_apply_stage(spp_ctx *cx, spp_stage s, int32_t l, const double *in, double *out, int32_t *cyc)
{
    Ctx *c = (Ctx *)cx;
    if (!c || !in || !out) FAIL(c, SPP_E_ARG, "spp_apply_stage: NULL argument");
    if (c->dim != 2) FAIL(c, SPP_E_STATE, "spp_apply_stage: 2D contexts only");
    if (c->dist) FAIL(c, SPP_E_STATE, "spp_apply_stage: single-GPU contexts only (not row strips)");
    const int m = c->m, n = c->n;
    const long mm = (long)m * m;
    const long G = (long)c->G;
    CK(c, ensure_vectors(c, 1));
    double *A = c->V[0], *B = c->Z[0];
    auto pk = [&](const double *src, double *dst) { k_pack<<<nblk(mm), 256, 0, c->st>>>(m, c->P, src, dst, 1, m); };
    auto up = [&](const double *src, double *dst) { k_unpack<<<nblk(mm), 256, 0, c->st>>>(m, c->P, src, dst, 1, m); };
    if (s == SPP_STAGE_MII_JACOBI) {
        pk(in, A);
        pk(out, B);
        launch_mii(c, A, B, false);                     // the solve's Jacobi-mode call (z-form)
        up(B, out);
    } else if (s == SPP_STAGE_MATVEC) {
        pk(in, A);
        k_spmv<<<kRedBlocks, kRedThreads, 0, c->st>>>(m, c->P, A, c->aE, c->aN, c->rr, c->aW, c->aS, 0, B, nullptr, nullptr, 1, m);
        up(B, out);
    } else if (s == SPP_STAGE_PRECOND) {
        pk(in, A);
        int cap = 0; cudaError_t err = cudaSuccess;
        // the hook applies the plain M^{-1} (unweighted input) regardless of the stop mode
        const int w = c->weighted;
        c->weighted = 0;
        if (w) { c->weighted = 0; CK(c, setup_lines(c)); }
        int k = apply_precond(c, A, B, &cap, &err);
        c->weighted = w;
        if (w) CK(c, setup_lines(c));
        CK(c, err);
        if (k < 0) {                                    // corner graph: read the cycle count
            CK(c, cudaMemcpyAsync(c->hmgs, c->mgs, sizeof(MGState), cudaMemcpyDeviceToHost, c->st));
            CK(c, cudaStreamSynchronize(c->st));
            k = c->hmgs->cycles;
            c->launches += (int64_t)k * c->cg_body_launches;
        }
        if (cyc) *cyc = k;
        up(B, out);
    } else if (s == SPP_STAGE_MII || s == SPP_STAGE_MYY || s == SPP_STAGE_MXX) {
        pk(in, A);
        // out holds the current z (compact): load it into B
        pk(out, B);
        const int w = c->weighted;
        if (w) { c->weighted = 0; CK(c, setup_lines(c)); }
        if (s == SPP_STAGE_MII) {
            launch_mii(c, A, B, true);
        } else {
            // run only the requested chain: temporarily restrict chunks
            std::vector<LineChunk> keep = c->chunks, sel;
            for (auto &ck : keep) if (ck.chain == (s == SPP_STAGE_MXX ? 0 : 1)) sel.push_back(ck);
            CK(c, cudaMemcpyAsync(c->d_chunks, sel.data(), sizeof(LineChunk) * sel.size(), cudaMemcpyHostToDevice, c->st));
            c->chunks = sel;
            launch_lines(c, A, B);
            c->chunks = keep;
            CK(c, cudaMemcpyAsync(c->d_chunks, keep.data(), sizeof(LineChunk) * keep.size(), cudaMemcpyHostToDevice, c->st));
        }
        c->weighted = w;
        if (w) CK(c, setup_lines(c));
        up(B, out);
    } else if (s == SPP_STAGE_CORNER_RHS) {
        pk(in, A);
        pk(in + mm, B);
        Level &L0 = c->lev[0];
        k_corner_rhs<<<kRedBlocks, kRedThreads, 0, c->st>>>(c->N, c->P, L0.pitch, A, B, c->aE, c->aN, c->rr, c->aW,
                                                            c->aS, L0.hb, L0.kb, 0, c->Bc, part_slot(c, 0), nullptr, c->cd, 0, 1, n);
        k_unpack_level<<<nblk((long)n * n), 256, 0, c->st>>>(n, L0.pitch, c->Bc, out);
    } else if (s == SPP_STAGE_CORNER_SOLVE) {
        Level &L0 = c->lev[0];
        CK(c, cudaMemsetAsync(c->Bc, 0, sizeof(double) * L0.elems, c->st));
        k_pack_level<<<nblk((long)n * n), 256, 0, c->st>>>(n, L0.pitch, in, c->Bc);
        // ||S_0 b||^2 via the residual kernel with z = 0
        CK(c, cudaMemsetAsync(c->Zc, 0, sizeof(double) * L0.elems, c->st));
        k_mg_resid<<<kRedBlocks, kRedThreads, 0, c->st>>>(n, L0.pitch, L0.cpitch, c->Zc, nullptr, c->Bc, L0.aE, L0.aN,
                                                          L0.rr, L0.aW, L0.aS, L0.hb, L0.kb, L0.rho, part_slot(c, 1));
        double b0sq = 0;
        CK(c, fetch_sum(c, part_slot(c, 1), &b0sq));
        if (c->par) {                                   // parabolic variant: the Galerkin corner MG
            int cap = 0; cudaError_t err = cudaSuccess;
            const int k = par_corner_solve(c, b0sq, &cap, &err);
            CK(c, err);
            if (cyc) *cyc = k;
            k_unpack_level<<<nblk((long)n * n), 256, 0, c->st>>>(n, L0.pitch, c->Zc, out);
            CK(c, cudaStreamSynchronize(c->st));
            return SPP_OK;
        }
        // the first cycle's V-cycle input: b_C (/ D in z-form)
        if (c->mg_zform) launch_scale_cd(c, 0, c->Bc, L0.rho);
        else CK(c, cudaMemcpyAsync(L0.rho, c->Bc, sizeof(double) * L0.elems, cudaMemcpyDeviceToDevice, c->st));
        int cap = 0; cudaError_t err = cudaSuccess;
        const double *zc = nullptr;
        int k = corner_solve(c, c->Bc, b0sq, &cap, &err, &zc);
        CK(c, err);
        if (!zc) { CK(c, cudaMemsetAsync(c->Zc, 0, sizeof(double) * L0.elems, c->st)); zc = c->Zc; }
        if (cyc) *cyc = k;
        k_unpack_level<<<nblk((long)n * n), 256, 0, c->st>>>(n, L0.pitch, zc, out);
    } else {
        if (l < 0 || l >= c->L) FAIL(c, SPP_E_ARG, "level %d out of range", l);
        Level &Lv = c->lev[l];
        const int nl = Lv.n;
        const long nn = (long)nl * nl;
        double *b = Lv.b, *e = Lv.e;
        if (s == SPP_STAGE_GS_SWEEP) {
            // one downstream GS sweep from e0 = out for rhs in (out-of-place kernel, e -> q)
            double *rhs = c->T1;
            CK(c, cudaMemsetAsync(rhs, 0, sizeof(double) * Lv.elems, c->st));
            k_pack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, in, rhs);
            k_pack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, out, e);
            launch_gs(c, l, 1, rhs, e, Lv.q, nullptr);
            k_unpack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, Lv.q, out);
        } else if (s == SPP_STAGE_VCYCLE) {
            double *tmp = c->T1;   // level-l rhs must not alias the level buffers used by vcycle
            CK(c, cudaMemsetAsync(tmp, 0, sizeof(double) * Lv.elems, c->st));
            k_pack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, in, tmp);
            const double *res = vcycle(c, l, tmp, false);
            k_unpack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, res, out);
        } else if (s == SPP_STAGE_RESTRICT) {
            // the fused residual-restriction kernel with e = 0 restricts R = in
            if (l + 1 >= c->L) FAIL(c, SPP_E_ARG, "no coarser level");
            Level &C = c->lev[l + 1];
            CK(c, cudaMemsetAsync(e, 0, sizeof(double) * Lv.elems, c->st));
            k_pack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, in, Lv.rho);
            launch_resid_restrict(c, l, Lv.rho, e);
            k_unpack_level<<<nblk((long)C.n * C.n), 256, 0, c->st>>>(C.n, C.pitch, C.b, out);
        } else if (s == SPP_STAGE_PROLONG_ADD) {
            if (l + 1 >= c->L) FAIL(c, SPP_E_ARG, "no coarser level");
            Level &C = c->lev[l + 1];
            k_pack_level<<<nblk((long)C.n * C.n), 256, 0, c->st>>>(C.n, C.pitch, in, C.e);
            k_pack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, out, e);
            k_prolong_add<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, e, C.e, C.pitch, Lv.w);
            k_unpack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, e, out);
        } else if (s == SPP_STAGE_POST_SMOOTH) {
            // the V-cycle's post-smoothing call: b stored as b/D, e, e_c in the level buffers the
            // product uses (lev[l].e, lev[l+1].q), prolongation fused into the sweep's rhs kernel
            if (l + 1 >= c->L) FAIL(c, SPP_E_ARG, "no coarser level");
            if (!c->mg_zform) FAIL(c, SPP_E_STATE, "POST_SMOOTH drives the z-form path");
            Level &C = c->lev[l + 1];
            double *bq = c->T1;
            CK(c, cudaMemsetAsync(bq, 0, sizeof(double) * Lv.elems, c->st));
            k_pack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, in, bq);
            k_pack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, in + nn, e);
            k_pack_level<<<nblk((long)C.n * C.n), 256, 0, c->st>>>(C.n, C.pitch, in + 2 * nn, C.q);
            launch_scale_cd(c, l, bq, bq);                  // b -> b/D (in place, element-wise)
            launch_gs(c, l, 1, bq, e, Lv.q, C.q, true);
            k_unpack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, Lv.q, out);
        } else if (s == SPP_STAGE_RESID_RESTRICT) {
            // the V-cycle's call: R read as R/D, b_c written divided by D_c (z-form)
            if (l + 1 >= c->L) FAIL(c, SPP_E_ARG, "no coarser level");
            if (!c->mg_zform) FAIL(c, SPP_E_STATE, "RESID_RESTRICT drives the z-form path");
            Level &C = c->lev[l + 1];
            double *Rq = c->T1;
            CK(c, cudaMemsetAsync(Rq, 0, sizeof(double) * Lv.elems, c->st));
            k_pack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, in, Rq);
            k_pack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, in + nn, e);
            launch_scale_cd(c, l, Rq, Rq);
            launch_resid_restrict(c, l, Rq, e, true, true);
            k_unpack_level<<<nblk((long)C.n * C.n), 256, 0, c->st>>>(C.n, C.pitch, C.b, out);
        } else if (s == SPP_STAGE_PRE_RESTRICT) {
            // the V-cycle's pre-smoothing from zero + residual-restriction (z-form, as in vcycle)
            if (l + 1 >= c->L) FAIL(c, SPP_E_ARG, "no coarser level");
            if (!c->mg_zform) FAIL(c, SPP_E_STATE, "PRE_RESTRICT drives the z-form path");
            Level &C = c->lev[l + 1];
            double *Rq = c->T1;
            CK(c, cudaMemsetAsync(Rq, 0, sizeof(double) * Lv.elems, c->st));
            CK(c, cudaMemsetAsync(e, 0, sizeof(double) * Lv.elems, c->st));
            k_pack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, in, Rq);
            launch_scale_cd(c, l, Rq, Rq);
            launch_gs(c, l, 0, Rq, nullptr, e, nullptr, true);
            launch_resid_restrict(c, l, nullptr, e, false, true);
            k_unpack_level<<<nblk((long)C.n * C.n), 256, 0, c->st>>>(C.n, C.pitch, C.b, out);
        } else if (s == SPP_STAGE_LEVEL_RESIDUAL) {
            k_pack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, in, b);
            k_pack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, in + nn, e);
            k_mg_resid<<<kRedBlocks, kRedThreads, 0, c->st>>>(nl, Lv.pitch, Lv.cpitch, e, nullptr, b, Lv.aE, Lv.aN,
                                                              Lv.rr, Lv.aW, Lv.aS, Lv.hb, Lv.kb, Lv.rho, nullptr);
            k_unpack_level<<<nblk(nn), 256, 0, c->st>>>(nl, Lv.pitch, Lv.rho, out);
        } else {
            FAIL(c, SPP_E_ARG, "unknown stage %d", (int)s);
        }
    }
    CK(c, cudaStreamSynchronize(c->st));
    CK(c, cudaGetLastError());
    if (c->sticky != cudaSuccess) { const cudaError_t se = c->sticky; c->sticky = cudaSuccess; CK(c, se); }
    (void)G;
    return SPP_OK;
}

// ------------------------------------------------------------------ batched 1D (NEXT-3)
#define BFAIL(bp, code, ...)                                                  \
    do {                                                                      \
        char _b[512];                                                         \
        snprintf(_b, sizeof(_b), __VA_ARGS__);                                \
        if (bp) (bp)->err = _b;                                               \
        g_err = _b;                                                           \
        return code;                                                          \
    } while (0)
#define BCK(bp, expr)                                                         \
    do {                                                                      \
        cudaError_t _e = (expr);                                              \
        if (_e != cudaSuccess)                                                \
            BFAIL(bp, SPP_E_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(_e), __FILE__, __LINE__); \
    } while (0)

static void batch1d_free(Batch1 *b)
{
    if (!b) return;
    if (b->st) cudaStreamSynchronize(b->st); else cudaDeviceSynchronize();
    cudaFree(b->scratch); cudaFree(b->dpar); cudaFree(b->doff); cudaFree(b->dint); cudaFree(b->stage);
    delete b;
}

spp_status spp_batch1d_setup(spp_batch1d *bx, const double *c, const double *r, spp_mem mem)
{
    Batch1 *b = (Batch1 *)bx;
    if (!b) FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_batch1d_setup: NULL batch");
    if (!c || !r) BFAIL(b, SPP_E_ARG, "spp_batch1d_setup: NULL coefficient array");
    const int nprob = b->nprob;
    const size_t bytes = sizeof(double) * (size_t)b->total;
    const double *dc = c, *dr = r;
    if (mem == SPP_HOST) {
        if (!b->stage) BCK(b, cudaMalloc(&b->stage, 2 * bytes));
        BCK(b, cudaMemcpyAsync(b->stage, c, bytes, cudaMemcpyHostToDevice, b->st));
        BCK(b, cudaMemcpyAsync(b->stage + b->total, r, bytes, cudaMemcpyHostToDevice, b->st));
        dc = b->stage; dr = b->stage + b->total;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, b->st);
    cudaError_t ce = batch1d_setup(b, dc, dr);
    cudaEventRecord(e1, b->st);
    std::vector<int> bad(nprob);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(bad.data(), b->dint + 4 * nprob, sizeof(int) * nprob, cudaMemcpyDeviceToHost, b->st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(b->st);
    cudaEventElapsedTime(&b->setup_ms, e0, e1);
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    if (ce != cudaSuccess) BFAIL(b, SPP_E_CUDA, "1D batch setup: %s", cudaGetErrorString(ce));
    for (int p = 0; p < nprob; ++p)
        if (bad[p]) BFAIL(b, SPP_E_COEF, "problem %d: coefficients violate c > 0, r >= 0 (P:208-212)", p);
    return SPP_OK;
}

spp_status spp_batch1d_create(int32_t nprob, const int32_t *n, const double *eps, const double *x,
                              const double *c, const double *r, spp_mem mem, const spp_options *o,
                              void *stream, spp_batch1d **out)
{
    if (!out || !n || !eps || !x || !c || !r || nprob < 1) FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_batch1d_create: bad argument");
    *out = nullptr;
    {
        spp_options oc;
        if (o) oc = *o; else spp_default_options(1, &oc);
        const spp_status so = check_options(&oc, 1, nullptr);
        if (so != SPP_OK) return so;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        FAIL((Ctx *)nullptr, SPP_E_CUDA, "spp_batch1d_create: no CUDA device (this library has no CPU path)");
    Batch1 *b = new (std::nothrow) Batch1();
    if (!b) FAIL((Ctx *)nullptr, SPP_E_NOMEM, "host allocation failed");
    b->st = (cudaStream_t)stream;
    if (o) b->opt = *o; else spp_default_options(1, &b->opt);
    if (b->opt.max_iters < 1) b->opt.max_iters = 1;
    b->nprob = nprob; b->maxit = b->opt.max_iters;
    if (b->maxit > 512) { delete b; FAIL((Ctx *)nullptr, SPP_E_ARG, "1D batch: max_iters <= 512 (single-CTA solver)"); }
    b->n.assign(n, n + nprob);
    b->eps.assign(eps, eps + nprob);
    b->h.resize(nprob); b->H.resize(nprob);
    long long xoff = 0;
    for (int p = 0; p < nprob; ++p) {
        const int N = n[p];
        if (N < 4 || (N % 2) || N - 1 > 8191) { delete b; FAIL((Ctx *)nullptr, SPP_E_ARG, "problem %d: N must be even, 4 <= N <= 8192 (got %d)", p, N); }
        if (!(eps[p] > 0.0) || eps[p] > 1.0) { delete b; FAIL((Ctx *)nullptr, SPP_E_ARG, "problem %d: eps must be in (0,1]", p); }
        double tau = 0.0;
        const spp_status s = check_mesh(x + xoff, N, &tau, nullptr);
        if (s != SPP_OK) { const std::string m = g_err; delete b; FAIL((Ctx *)nullptr, s, "problem %d: %s", p, m.c_str()); }
        b->h[p] = tau / (N / 2); b->H[p] = (1.0 - tau) / (N / 2);
        xoff += N + 1;
    }
    if (batch1d_alloc(b) != cudaSuccess) { batch1d_free(b); FAIL((Ctx *)nullptr, SPP_E_NOMEM, "1D batch: device allocation failed"); }
    const spp_status s = spp_batch1d_setup((spp_batch1d *)b, c, r, mem);
    if (s != SPP_OK) { batch1d_free(b); return s; }
    *out = (spp_batch1d *)b;
    return SPP_OK;
}

spp_status spp_batch1d_solve(spp_batch1d *bx, const double *f, double *u, spp_mem mem, int32_t *iters,
                             int32_t *converged, double *res, spp_stats *st)
{
    Batch1 *b = (Batch1 *)bx;
    if (!b) FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_batch1d_solve: NULL batch");
    if (!f || !u) BFAIL(b, SPP_E_ARG, "spp_batch1d_solve: NULL f or u");
    const int P = b->nprob;
    const size_t bytes = sizeof(double) * (size_t)b->total;
    if (mem == SPP_HOST && !b->stage) BCK(b, cudaMalloc(&b->stage, 2 * bytes));
    const int64_t l0 = b->launches;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, b->st);
    const double *df = f;
    double *du = u;
    if (mem == SPP_HOST) {
        BCK(b, cudaMemcpyAsync(b->stage, f, bytes, cudaMemcpyHostToDevice, b->st));
        df = b->stage; du = b->stage + b->total;
    }
    BCK(b, batch1d_solve(b, df, du));
    if (mem == SPP_HOST) BCK(b, cudaMemcpyAsync(u, du, bytes, cudaMemcpyDeviceToHost, b->st));
    cudaEventRecord(e1, b->st);
    std::vector<int> io(2 * (size_t)P);
    std::vector<double> rr(2 * (size_t)P);
    BCK(b, cudaMemcpyAsync(io.data(), b->dint + 2 * P, sizeof(int) * 2 * P, cudaMemcpyDeviceToHost, b->st));
    BCK(b, cudaMemcpyAsync(rr.data(), b->dpar + 3 * P, sizeof(double) * 2 * P, cudaMemcpyDeviceToHost, b->st));
    BCK(b, cudaStreamSynchronize(b->st));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    int all = 1, itmax = 0, itsum = 0;
    for (int p = 0; p < P; ++p) {
        if (iters) iters[p] = io[p];
        if (converged) converged[p] = io[P + p];
        if (res) res[p] = rr[P + p];
        all &= io[P + p] ? 1 : 0;
        itmax = std::max(itmax, io[p]); itsum += io[p];
    }
    if (st) {
        memset(st, 0, sizeof(*st));
        st->iters = itmax; st->converged = all; st->applies = itsum;
        st->kernel_launches = (int32_t)(b->launches - l0);
        st->setup_s = b->setup_ms * 1e-3; st->solve_s = ms * 1e-3;
        st->res0 = -1.0; st->res_final = -1.0; st->true_res_l2_rel = -1.0; st->true_res_jacobi_rel = -1.0;
    }
    return all ? SPP_OK : SPP_NOT_CONVERGED;
}

int32_t spp_batch1d_nprob(const spp_batch1d *b) { return b ? ((const Batch1 *)b)->nprob : 0; }
int64_t spp_batch1d_launches(const spp_batch1d *b) { return b ? ((const Batch1 *)b)->launches : 0; }
const char *spp_batch1d_last_error(const spp_batch1d *b) { return b ? ((const Batch1 *)b)->err.c_str() : g_err.c_str(); }
void spp_batch1d_destroy(spp_batch1d *b) { batch1d_free((Batch1 *)b); }

}  // extern "C"

// =========================================================================== row strips
extern "C" {

spp_status spp_strip_partition(int32_t n, int32_t nranks, int32_t *j)
{
    if (!j || nranks < 1 || n < 8 || (n % 2)) FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_strip_partition: bad arguments");
    std::vector<int> J;
    if (!strip_partition(n, nranks, J)) FAIL((Ctx *)nullptr, SPP_E_ARG, "%d strips do not fit N = %d", nranks, n);
    for (int r = 0; r <= nranks; ++r) j[r] = J[r];
    return SPP_OK;
}

// strip contexts share the problem's validation and setup; the decomposition is finished by the
// first spp_setup (setup_dist)
static spp_status strip_ctx(const spp_problem *p, const spp_options *o, void *stream, int rank, int nranks,
                            const std::vector<int> &J, int Pb, Ctx **out)
{
    Ctx *c = nullptr;
    spp_status s = ctx_new(p, o, stream, &c);
    if (s != SPP_OK) return s;
    if (p->dim != 2) { delete c; FAIL((Ctx *)nullptr, SPP_E_ARG, "row strips are a 2D decomposition"); }
    c->rank = rank; c->nparts = nranks;
    c->use_graph = 0;
    const int N = c->N;
    if (rank >= Pb) { c->line_lo[0] = N - J[rank + 1]; c->line_hi[0] = N - 1 - J[rank]; c->line_lo[1] = 0; c->line_hi[1] = -1; }
    else {
        const int nl = c->n - 1;
        c->line_lo[0] = 0; c->line_hi[0] = -1;
        c->line_lo[1] = (int)((long)nl * rank / Pb); c->line_hi[1] = (int)((long)nl * (rank + 1) / Pb) - 1;
    }
    if ((s = alloc_all(c)) != SPP_OK) { g_err = c->err; ctx_free(c); return s; }
    *out = c;
    return SPP_OK;
}

spp_status spp_create_strips(const spp_problem *p, int32_t nstrips, const spp_options *o, void *stream, spp_ctx **out)
{
    if (!p || !out) FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_create_strips: NULL argument");
    *out = nullptr;
    if (nstrips == 1) return spp_create(p, o, stream, out);
    if (o && o->restart != 0) FAIL((Ctx *)nullptr, SPP_E_ARG, "row strips run FGMRES without restarts (restart = 0)");
    std::vector<int> J;
    if (nstrips < 1 || p->dim != 2 || !strip_partition(p->n, nstrips, J))
        FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_create_strips: %d strips of a %s N = %d problem", nstrips,
             p->dim == 2 ? "2D" : "1D", p->n);
    int Pb = 0;
    std::string why;
    if (!check_partition(p->n, J, &Pb, &why)) FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_create_strips: %s", why.c_str());
    Dist *d = new (std::nothrow) Dist();
    if (!d) FAIL((Ctx *)nullptr, SPP_E_NOMEM, "host allocation failed");
    d->me = -1; d->st = (cudaStream_t)stream;
    d->g.P = nstrips; d->g.Pb = Pb; d->g.J = J;
    for (int r = 0; r < nstrips; ++r) {
        Ctx *c = nullptr;
        const spp_status s = strip_ctx(p, o, stream, r, nstrips, J, Pb, &c);
        if (s != SPP_OK) {
            const std::string m = g_err;
            for (Ctx *x : d->cx) ctx_free(x);
            delete d;
            g_err = m;
            return s;
        }
        c->dist = d;
        d->cx.push_back(c);
    }
    const spp_status s = spp_setup((spp_ctx *)d->cx[0], p->c1, p->c2, p->r, p->mem);
    if (s != SPP_OK) { g_err = d->cx[0]->err; spp_destroy((spp_ctx *)d->cx[0]); return s; }
    *out = (spp_ctx *)d->cx[0];
    return SPP_OK;
}

spp_status spp_create_dist(const spp_problem *local, int32_t j0, int32_t j1, void *nccl_comm, int32_t rank,
                           int32_t nranks, const spp_options *o, void *stream, spp_ctx **out)
{
    if (!local || !out) FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_create_dist: NULL argument");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_create_dist: rank %d of %d", rank, nranks);
    if (nranks == 1) {
        if (j0 != 1 || j1 != local->n) FAIL((Ctx *)nullptr, SPP_E_ARG, "one rank owns rows 1..N-1");
        return spp_create(local, o, stream, out);
    }
    if (!nccl_comm) FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_create_dist: NULL NCCL communicator");
    if (o && o->restart != 0) FAIL((Ctx *)nullptr, SPP_E_ARG, "row strips run FGMRES without restarts (restart = 0)");
    // gather every rank's [j0, j1) through a provisional strip context (its partial-sum buffer)
    std::vector<int> J0(nranks + 1, 0);
    Ctx *c = nullptr;
    {   // validate the problem and options before any communication
        spp_status s = ctx_new(local, o, stream, &c);
        if (s != SPP_OK) return s;
        delete c;
        c = nullptr;
        if (local->dim != 2) FAIL((Ctx *)nullptr, SPP_E_ARG, "row strips are a 2D decomposition");
    }
    Dist *d = new (std::nothrow) Dist();
    if (!d) FAIL((Ctx *)nullptr, SPP_E_NOMEM, "host allocation failed");
    d->me = rank; d->comm = nccl_comm; d->st = (cudaStream_t)stream; d->g.P = nranks;
    {
        double *buf = nullptr, hb[2] = {(double)j0, (double)j1};
        std::vector<double> all(2 * (size_t)nranks);
        if (cudaMalloc(&buf, sizeof(double) * 2 * nranks) != cudaSuccess) { delete d; FAIL((Ctx *)nullptr, SPP_E_NOMEM, "device allocation"); }
        cudaMemcpyAsync(buf + 2 * rank, hb, sizeof(hb), cudaMemcpyHostToDevice, d->st);
        // a throw-away context whose part buffer is `buf`: the exchange addresses buffers by role
        Ctx tmp;
        tmp.part = buf; tmp.st = d->st;
        d->cx.push_back(&tmp);
        std::vector<Xfer> xs;
        for (int s = 0; s < nranks; ++s)
            for (int t = 0; t < nranks; ++t)
                if (s != t) xs.push_back({s, t, R_PART, 0, 2L * s, 2L * s, 2, 1, 2});
        const spp_status s = exchange_rows(d, xs);
        d->cx.clear();
        tmp.part = nullptr;
        if (s == SPP_OK) cudaMemcpyAsync(all.data(), buf, sizeof(double) * 2 * nranks, cudaMemcpyDeviceToHost, d->st);
        cudaStreamSynchronize(d->st);
        cudaFree(buf);
        if (s != SPP_OK) { delete d; FAIL((Ctx *)nullptr, s, "spp_create_dist: gathering the strips failed (%s)", g_err.c_str()); }
        for (int r = 0; r < nranks; ++r) {
            J0[r] = (int)all[2 * r];
            if (r + 1 < nranks && (int)all[2 * r + 1] != (int)all[2 * r + 2]) {
                delete d;
                FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_create_dist: strip %d ends at %d but strip %d starts at %d", r,
                     (int)all[2 * r + 1], r + 1, (int)all[2 * r + 2]);
            }
        }
        J0[nranks] = (int)all[2 * nranks - 1];
    }
    int Pb = 0;
    std::string why;
    if (!check_partition(local->n, J0, &Pb, &why)) { delete d; FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_create_dist: %s", why.c_str()); }
    d->g.Pb = Pb; d->g.J = J0;
    spp_status s = strip_ctx(local, o, stream, rank, nranks, J0, Pb, &c);
    if (s != SPP_OK) { delete d; return s; }
    c->dist = d;
    d->cx.push_back(c);
    s = spp_setup((spp_ctx *)c, local->c1, local->c2, local->r, local->mem);
    if (s != SPP_OK) { g_err = c->err; spp_destroy((spp_ctx *)c); return s; }
    *out = (spp_ctx *)c;
    return SPP_OK;
}

spp_status spp_dist_info(const spp_ctx *cx, int32_t *nranks, int32_t *strip_levels, int64_t *xfers, double *bytes,
                         int64_t *exchanges)
{
    const Ctx *c = (const Ctx *)cx;
    if (!c) FAIL((Ctx *)nullptr, SPP_E_ARG, "spp_dist_info: NULL context");
    const Dist *d = c->dist;
    if (nranks) *nranks = d ? d->g.P : 1;
    if (strip_levels) *strip_levels = d ? d->g.D : 0;
    if (xfers) *xfers = d ? d->nxfer : 0;
    if (bytes) *bytes = d ? d->xbytes : 0.0;
    if (exchanges) *exchanges = d ? d->nexch : 0;
    return SPP_OK;
}

}  // extern "C"
