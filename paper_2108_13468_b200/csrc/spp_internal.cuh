// spp_internal.cuh -- device layout, context and kernel declarations of the B200 solver.
//
// Layout: every 2D grid function lives in a padded array
// with a zero ghost ring: node (i, j) at [j * pitch + i], i, j = 0 .. n+1 where 1..n are the
// unknowns of that grid and 0 / n+1 the (homogeneous Dirichlet) ghosts; pitch is a multiple
// of 16 doubles so 16-column blocks are 128-byte aligned.  Ghosts and padding hold zeros and
// every kernel preserves that, so vector kernels run over the flat array.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cuda.h>

#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "spp.h"

namespace spp {

struct Dist;                             // row-strip decomposition (dist.cuh)
constexpr int kMaxLevels = 24;
constexpr int kWarp = 32;
constexpr int kRedBlocks = 592;      // 4 x 148 SMs: fixed grid for deterministic reductions
// reduction grid for `work` elements: kRedBlocks for large grids; fewer for small ones (the
// producers zero the unused partial slots, so every consumer still sums kRedBlocks partials)
inline int red_grid(long work)
{
    const long b = (work + 511) / 512;                 // ~2 elements per thread
    return (int)(b < 1 ? 1 : (b > kRedBlocks ? kRedBlocks : b));
}
// the unused tail of a partials array (blocks >= gridDim.x of a shortened reduction grid)
__device__ __forceinline__ void zero_tail(double *part)
{
    if (blockIdx.x == 0)
        for (int b = gridDim.x + threadIdx.x; b < kRedBlocks; b += blockDim.x) part[b] = 0.0;
}
constexpr int kRedThreads = 256;
// Launch shape of the row-segment reduction kernels (k_cycle_update, k_corner_rhs): a thread per
// column pair of a row of n + 2 columns (ghosts included), at most kRedThreads threads per block,
// a warp multiple; one block-iteration per row segment, at most kRedBlocks blocks.
inline void seg_shape(int n, long rows, int *blocks, int *threads)
{
    // the row's column pairs spread evenly over its segments (n = 2048: 1025 pairs = 5 segments of
    // 224 threads; 256-thread blocks would leave the fifth segment with one pair)
    const int pairs = (n + 3) / 2;
    const int ns = (pairs + kRedThreads - 1) / kRedThreads;
    int t = ((pairs + ns - 1) / ns + 31) / 32 * 32;
    t = t < 32 ? 32 : (t > kRedThreads ? kRedThreads : t);
    const long nseg = (n + 2 + 2L * t - 1) / (2L * t);
    const long b = rows * nseg;
    *threads = t;
    *blocks = (int)(b < 1 ? 1 : (b > kRedBlocks ? kRedBlocks : b));
}

// Grid-stride walk over level nodes (i, j), i = 1..m, j = j0.. in the order p = (j - j0) m + (i - 1):
// one division at the start, then (i, j) advance incrementally (a 64-bit division per element was
// a visible share of the memory-bound kernels' issue slots).  Same visiting order as p / m, p % m.
struct GridWalk {
    long p, tot, stride;
    int i, j, m, si, sj;
    __device__ __forceinline__ GridWalk(long tot_, int m_, int j0)
        : p(blockIdx.x * (long)blockDim.x + threadIdx.x), tot(tot_), stride((long)gridDim.x * blockDim.x), m(m_)
    {
        j = (int)(p / m) + j0; i = (int)(p % m) + 1;
        sj = (int)(stride / m); si = (int)(stride % m);
    }
    __device__ __forceinline__ bool ok() const { return p < tot; }
    __device__ __forceinline__ void next()
    {
        p += stride; i += si; j += sj;
        if (i > m) { i -= m; ++j; }
    }
};
constexpr long kTmaSlack = 1L << 16;     // doubles appended to grid allocations (TMA over-read)

inline long round_up(long a, long b) { return (a + b - 1) / b * b; }

// line-chain solve (M_XX / M_YY): see k_lines.cu
struct LineChain {
    int nlines, len;        // lines in the chain, unknowns per line
    long vstride;           // address step along a line in the value grid
    long vline;             // address step from line l to line l+1 (the next line processed)
    long v0;                // value-grid address of element 0 of line 0
    long istep;             // value-grid address offset of the I-neighbour of the last element
    const double *p, *e, *al, *be;  // factors, line-major [l * len + k]
    const double *t;        // per-line coupling factor to I at the last element
};
struct LineChunk { int chain, first, last, start; };   // lines [first,last] owned, processing from `start`

// Geometric interpolation weights of the odd nodes of a corner level from the next coarser
// level (R21): node q between the coarser nodes at its left / right (x) and below /
// above (y); 1/2 on a uniform (Shishkin) corner.  Device arrays indexed 1..n.
struct Wts { const double *xl, *xr, *yl, *yr; int uni; };   // uni: every weight is 1/2 (no loads)

struct Level {
    int n = 0;                           // unknowns per axis
    long pitch = 0;                      // value pitch
    size_t elems = 0;
    const double *aE = nullptr, *aN = nullptr, *rr = nullptr;   // coefficients (coef pitch cpitch)
    const double *ya = nullptr, *yn = nullptr, *cd = nullptr;   // aE/D_E, aN/D_N, 1/D
    long cpitch = 0;
    double *aW = nullptr, *aS = nullptr, *hb = nullptr, *kb = nullptr;   // 1D [n+2]
    double *lwx = nullptr, *lwy = nullptr;   // the level's 1D mesh widths, index 1..n+1 [n+2]
    Wts w{};                             // interpolation weights from level l+1 [n+2 each]
    double *own = nullptr;               // owned coefficient block (levels >= 1)
    double *b = nullptr, *e = nullptr, *q = nullptr, *rho = nullptr;     // work (value layout)
    double *g = nullptr;                 // GS right-hand side (k_gs_prep)
    // GS tiling (k_mg.cu): tile_rows <= 0 -> one CTA sweeps the level; halo = certified rows /
    // columns recomputed above / right of each tile (-1: none certifiable -> exact chained sweep)
    int tile_rows = 0, tile_cols = 0, tile_warps = 0, halo_x = 0, halo_y = 0;
    double contraction = 0.0;            // max (aE + aN) / D over the level
    int halo_cert = -1, halo_certx = -1; // certified halo rows / columns of the level (-1: none)
    // row strip of a distributed solve: this rank owns rows slo..shi of the level
    // (1..n on one GPU).  sdist: the level's GS sweeps run on the strip (own rows plus shalo
    // halo rows above, whose right-hand side comes from the strip above) with the tile plan
    // above; otherwise the level runs whole on every rank.
    int slo = 1, shi = 0, shalo = 0;
    bool sdist = false;
};

// one level of the parabolic-variant corner multigrid (k_par.cu; c2 = 0)
struct ParLevel {
    int nx = 0; long pv = 0;             // unknowns in x (ny = n), value pitch
    double *a = nullptr;                 // nine-point stencil, 9 compact arrays of n*nx
    double *wW = nullptr, *wE = nullptr; // interpolation weights of the odd-x nodes [n*nx]
    double *e = nullptr, *rho = nullptr, *b = nullptr;   // padded value layout
};

// corner GS sweep arguments (k_mg.cu)
// downstream sweep on [1, nl]^2 (k_mg.cu): y = q + ca y_E + cn y_N, z = cd y (y-form) or z = y
struct WaveArgs {
    int nl; long pv, pc;                 // nl: columns 1..nl of the swept block
    int ioff, joff;                      // node (i, j) lives at array index (i+ioff, j+joff)
    const double *q, *ca, *cn, *cd;
    double *z;
    int rows_out, cols_out, halo_y, halo_x;
    int *chain_flags; double *chain_buf; long chain_ld;   // exact chained mode
    long long *prof;                     // SPP_WAVE_PROF builds only
    // rows of the block: 1..nr_out are output rows, nr_out+1..nr the halo rows above them that a
    // row strip of a distributed solve recomputes from the strip above's right-hand side
    // (DESIGN.md §9); nr = nr_out = nl for a whole level (0 = that default)
    int nr, nr_out;
    // exact chained mode across row strips: the first CTA strip's North inflow (the bottom row of
    // the strip above, in the chain buffer's order; nullptr = zero inflow) and whether the last
    // CTA strip publishes its bottom row into chain slot gridDim.y - 1
    const double *ext_in;
    int chain_last;
};

// tunables (defaults in spp_create; overridable through SPP_TUNE="key=val,..." for experiments)
struct Tune {
    int gs_warps = 5;          // max warps (32-row strips) per GS tile (4 in y-form)
    int gs_tile_cols = 0;      // output columns per GS tile (0: one wave of CTAs per level)
    int gs_max_halo = 128;     // no certified halo below this -> exact chained sweep
    int sweep_warps = 2;       // warps per CTA of the exact chained sweep (M_II; 2 measured best)
    int gs_lag = 5;            // tiling model: chunk-times each extra warp adds
    int coarse_max = 32;       // levels with n <= this run as one fused single-CTA V-cycle (<= kCoarseMaxN = 32)
    int dist_levels = 2;       // row strips: corner levels whose sweeps run on the strips
    int rho_halo = 0;          // 1: certify halos by rho = max (ca + cn) (round 1) instead of gamma_y, gamma_x
};

struct ProfRec { int64_t launches = 0; double ms = 0, bytes = 0; };

// device-resident state of the corner stationary iteration when it runs as a CUDA graph with a
// device-side while loop (capi.cu "corner graph")
struct MGState {
    const double *zcur;     // current iterate z (nullptr: z = 0, no cycle ran yet)
    double *znext;          // buffer the next cycle writes
    double *za, *zb;        // the two iterate buffers
    double b0, res;         // ||S0 b_C||, ||S0 rho||
    int cycles, cap;        // cycles run, cycle cap hit
};

// device-resident FGMRES state of the iteration graphs (capi.cu "iteration graphs"): the
// Givens/Hessenberg bookkeeping and the stop test run on the device, so a batch of iterations
// needs no host round trip
struct FGHead {
    int k;                  // iterations done
    int stop;               // the loop has ended (the gates of later graphs skip their iteration)
    int converged, nonfinite, nf_j, capfail;
    int mg_tot, mg_min, mg_max, caps;
    double res;             // |g_k|
    double target;          // the stop test's threshold (tol, or tol * beta in the relative modes)
};

struct Ctx {
    int dim = 0, N = 0, n = 0, m = 0;    // N intervals, n = N/2, m = N-1
    double eps = 0;
    spp_options opt{};
    cudaStream_t st = nullptr;
    int weighted = 1;
    std::string err;
    // mesh (widths from the piecewise-uniform formula with tau = x[N/2])
    double tx = 0, ty = 0, hx = 0, Hx = 0, hy = 0, Hy = 0;
    std::vector<double> xh, yh;
    int gx = 0, gy = 0;                  // graded (not piecewise-uniform) mesh in x / y (R21)
    double *wxd = nullptr, *wyd = nullptr;   // device widths h_i, k_j (i = 1..N) [N+2]
    // global padded grid
    long P = 0; size_t G = 0;
    double *aE = nullptr, *aN = nullptr, *rr = nullptr;         // coefficients
    double *ca = nullptr, *cn = nullptr, *cd = nullptr;         // aE/D, aN/D, 1/D
    double *ya = nullptr, *yn = nullptr;                        // aE/D_E, aN/D_N (y-form sweeps)
    double *aW = nullptr, *aS = nullptr;                        // [N+1]
    double *coef_block = nullptr;
    // line factors
    double *fac = nullptr;                 // X then Y: 4 arrays each of (n-1)*n
    double *tX = nullptr, *tY = nullptr, *kapX = nullptr, *kapY = nullptr;
    LineChain chX{}, chY{};
    std::vector<LineChunk> chunks; LineChunk *d_chunks = nullptr; int nchunks_alloc = 0;
    std::vector<double> kx, ky;            // per-line chain contractions kappa_l (host copies)
    int line_lo[2] = {-1, -1}, line_hi[2] = {-2, -2};   // owned lines per chain (-1: all, one GPU)
    int lines_threads = 256;
    // Krylov
    std::vector<double *> V, Z;
    double *w = nullptr, *F = nullptr, *U = nullptr, *T1 = nullptr;
    double *part = nullptr;                // reduction partials [kMaxParts][kRedBlocks]
    double *dscal = nullptr;               // device scalars
    double *hpin = nullptr;                // pinned host mirror of scalars
    int vec_alloc = 0;
    // corner MG
    int L = 0;
    Level lev[kMaxLevels];
    double *Zc = nullptr, *Bc = nullptr;   // corner iterate / rhs (level-0 value layout)
    double *Zc2 = nullptr;                 // ping-pong partner of Zc
    double *chain = nullptr; long chain_ld = 0;   // inflow buffer of the exact chained sweep
    int *chain_flags = nullptr;
    Tune tune;
    std::map<std::tuple<const void *, long, long>, CUtensorMap> tmaps;   // sheared TMA maps (k_mg.cu)
    std::map<std::tuple<const void *, unsigned long long, unsigned long long, unsigned long long, unsigned, unsigned, bool>,
             CUtensorMap> tmaps2;          // generic 2D maps (tmap2d)
    cudaError_t sticky = cudaSuccess;      // first launch-configuration error of a solve
    double *mg_block = nullptr;
    int *flags = nullptr; int epoch = 0;
    // 1D
    double *d1 = nullptr;
    // compact staging buffers
    double *cbuf = nullptr;
    // statistics / profiling
    int64_t launches = 0;
    int prof_on = 0;
    ProfRec prof[SPP_PROF_CLASSES];
    std::vector<cudaEvent_t> ev_pool; size_t ev_used = 0;
    struct PendingProf { int cls; cudaEvent_t a, b; double bytes; };
    std::vector<PendingProf> pend;
    float setup_ms = 0;
    int sm_count = 148;
    // corner graph: the stationary V-cycle iteration as one CUDA graph with a while node
    MGState *mgs = nullptr;                // device state
    MGState *hmgs = nullptr;               // pinned host copy
    cudaStream_t cap_st = nullptr;         // private capture stream
    cudaGraph_t cg = nullptr; cudaGraphExec_t cg_exec = nullptr;
    std::vector<long> cg_sig;              // plan signature the graph was captured for
    int64_t cg_body_launches = 0;          // kernels per loop iteration
    bool capturing = false;
    int use_graph = 1;
    // iteration graphs: graph k = [gate] -> IF { FGMRES iteration k (the corner loop a nested
    // while node) }, built on first use and kept while the plan (fg_signature) is unchanged
    FGHead *fgh = nullptr, *hfgh = nullptr;   // device state / pinned host copy
    double *fgd = nullptr;                 // device H [(maxit+1)^2], cs, sn, g, hist [maxit+2 each]
    std::vector<cudaGraphExec_t> itg;
    std::vector<int64_t> itg_launches;     // kernels of iteration k's body (the corner cycles apart)
    std::vector<long> itg_sig;
    int fg_ok = 1;                         // 0: graphs unavailable on this device -> host loop
    int last_iters = 0;                    // the previous solve's iterations (first batch size)
    int no_lines_tma = 0;                  // SPP_NO_LINES_TMA=1: LSU-loaded line kernel
    int mg_zform = 1;                      // corner GS sweeps in z-form (SPP_MG_YFORM=1: y-form)
    int y0_ok = 0;                         // ya, yn of the global grid are current (ensure_y0)
    std::vector<double> rho_h;             // setup: the levels' contraction partials (host copy)
    // parabolic-layer variant (c2 = 0 everywhere; NEXT-2): semi-coarsening Galerkin corner MG
    int par = 0, PL = 0;
    ParLevel plev[kMaxLevels];
    double *par_block = nullptr, *par_sb = nullptr, *par_rho = nullptr;
    // row strips: the decomposition this context is one strip of (nullptr: one
    // GPU), the strip's rank, and the partial-sum segments per reduction slot (one per strip)
    Dist *dist = nullptr;
    int rank = 0, nparts = 1;
};

// kernels / launchers (defined in the .cu files)
cudaError_t setup_global(Ctx *c, const double *c1, const double *c2, const double *r);
spp_status setup_2d_ctx(Ctx *c, const double *c1, const double *c2, const double *r, spp_mem mem);
cudaError_t ensure_vectors(Ctx *c, int k);
bool strip_partition(int N, int P, std::vector<int> &J);
bool check_partition(int N, const std::vector<int> &J, int *Pb, std::string *why);
cudaError_t setup_levels(Ctx *c, const double *c1, const double *c2, const double *r);
cudaError_t setup_lines(Ctx *c);
cudaError_t setup_lines_launch(Ctx *c);
cudaError_t setup_lines_plan(Ctx *c);
void plan_chunks(Ctx *c, const std::vector<double> &kx, const std::vector<double> &ky, const int lo[2],
                 const int hi[2], int budget);
std::vector<LineChunk> plan_chain_chunks(int chain, const std::vector<double> &k, int l0, int l1, int budget);
// corner multigrid (k_mg.cu)
void launch_gs(Ctx *c, int l, int mode, const double *b, const double *eold, double *enew, const double *ec,
               bool bscaled = false);
void launch_gs_prep(Ctx *c, int l, const double *b, const double *eold, const double *ec, bool bscaled);
void launch_gs_sweep(Ctx *c, int l, const double *q, double *enew);
double *vcycle(Ctx *c, int l, const double *R, bool rs);
void launch_wave_chain(Ctx *c, WaveArgs a, long rows_v, long rows_c, bool yform, int cls, double bytes);
long wave_chain_ctas(const Ctx *c, long rows);
void launch_ycoef(Ctx *c, int nl, long pc, const double *aE, const double *aN, const double *cd, double *ya, double *yn);
void ensure_y0(Ctx *c);
cudaError_t wave_init();
cudaError_t lines_init();
const CUtensorMap *tmap2d(Ctx *c, const void *base, unsigned long long d0, unsigned long long d1,
                          unsigned long long stride_bytes, unsigned b0, unsigned b1, bool swz128);
void launch_resid_restrict(Ctx *c, int l, const double *R, const double *e, bool rs_in = false, bool scale_out = false);
void launch_cycle_update(Ctx *c, const double *z, const double *e, double *znew, const double *b, double *rho,
                         double *part, const MGState *ms = nullptr);
void launch_lines(Ctx *c, const double *v, double *z);
cudaError_t setup_mg_tiles(Ctx *c);
cudaError_t setup_mg_tiles_launch(Ctx *c);
cudaError_t setup_mg_tiles_plan(Ctx *c);
cudaError_t par_alloc(Ctx *c);
cudaError_t par_setup(Ctx *c);
int par_corner_solve(Ctx *c, double b0sq, int *cap_hit, cudaError_t *err);
bool plan_tiles(const Ctx *c, int n, int rows, int halo, int halox, bool whole, Level &L);
void launch_scale_cd(Ctx *c, int l, const double *b, double *q);
bool launch_coarse_vcycle(Ctx *c, int lc, const double *R, bool rs = false);

// linear interpolation of the coarse correction at fine node (i, j): an even node
// 2I is the coarse node I; an odd node 2I+1 lies between I and I+1 (the ghost 0 at I = 0), with
// the level's geometric weights (1/2 on a Shishkin corner: then bit for bit the classical
// 0.5 (a + b) / 0.25 ((a + b) + (c + d)), every product by 1/2 being exact).
template <bool UNI = false>
__device__ __forceinline__ double interp_w(const double *ec, long Pc, int i, int j, const Wts &W)
{
    const int I0 = i >> 1, J0 = j >> 1;
    const bool oi = i & 1, oj = j & 1;
    const double *r0 = ec + (long)J0 * Pc + I0;
    if (!oi && !oj) return r0[0];
    if (UNI) {                                   // the classical weights of a uniform corner
        if (oi && !oj) return 0.5 * (r0[0] + r0[1]);
        if (!oi && oj) return 0.5 * (r0[0] + r0[Pc]);
        return 0.25 * ((r0[0] + r0[1]) + (r0[Pc] + r0[Pc + 1]));
    }
    const double xl = W.xl[i], xr = W.xr[i], yl = W.yl[j], yr = W.yr[j];
    if (oi && !oj) return xl * r0[0] + xr * r0[1];
    if (!oi && oj) return yl * r0[0] + yr * r0[Pc];
    return yl * (xl * r0[0] + xr * r0[1]) + yr * (xl * r0[Pc] + xr * r0[Pc + 1]);
}

// interp_w with the parity of i known at compile time (a thread that owns a column pair (i0,
// i0+1), i0 even, knows it; the parity of j is uniform over a row): the same expressions, so the
// same bits, without the lane-alternating branch on i.
template <bool UNI, bool OI>
__device__ __forceinline__ double interp_p(const double *ec, long Pc, int i, int j, const Wts &W)
{
    const int I0 = i >> 1, J0 = j >> 1;
    const bool oj = j & 1;
    const double *r0 = ec + (long)J0 * Pc + I0;
    if (!OI && !oj) return r0[0];
    if (UNI) {
        if (OI && !oj) return 0.5 * (r0[0] + r0[1]);
        if (!OI && oj) return 0.5 * (r0[0] + r0[Pc]);
        return 0.25 * ((r0[0] + r0[1]) + (r0[Pc] + r0[Pc + 1]));
    }
    const double xl = W.xl[i], xr = W.xr[i], yl = W.yl[j], yr = W.yr[j];
    if (OI && !oj) return xl * r0[0] + xr * r0[1];
    if (!OI && oj) return yl * r0[0] + yr * r0[Pc];
    return yl * (xl * r0[0] + xr * r0[1]) + yr * (xl * r0[Pc] + xr * r0[Pc + 1]);
}

// profiling helpers
void prof_collect(Ctx *c);
struct ProfScope {
    Ctx *c; int cls; double bytes; cudaEvent_t a = nullptr; bool nv = false;
    ProfScope(Ctx *c_, int cls_, double bytes_);
    ~ProfScope();
};
// NVTX range for a host-side phase (SPP_NVTX=1; no cost otherwise): spp_setup, spp_solve, and one
// range per launch class from ProfScope (tracing)
struct NvtxScope {
    bool on;
    explicit NvtxScope(const char *name);
    ~NvtxScope();
};

}  // namespace spp

#define SPP_CUDA_TRY(expr)                                                   \
    do {                                                                     \
        cudaError_t _e = (expr);                                             \
        if (_e != cudaSuccess) return _e;                                    \
    } while (0)
