// k_par.cu -- the corner multigrid of the parabolic-layer variant (c2 = 0, SURVEY
// 8(f) NEXT-2), sm_100a, fp64.
//
// Semi-coarsening in x only (ny = n rows on every level, nx halved per level down to <= 4).  The
// finest operator is A_CC with row (i,j) scaled by hbar_i kbar_j (FE scaling);
// interpolation to an odd-x fine node from the coarse nodes at x_{i-1}, x_{i+1} with minus the W /
// E column sums over the centre column sum of its stencil (the North-South collapse);
// restriction = interpolation^T; coarse operators by the Galerkin product R A P:
// nine-point.  Downstream point Gauss-Seidel (top-right to bottom-left), V(1,1), four
// sweeps on the coarsest level; the corner iteration stops at a 10^2 reduction of the FE-scaled
// residual (reading R22).
//
// Layout: a level's stencil is nine compact arrays a[k][(j-1) nx + (i-1)], k = (dj+1)*3 + (di+1),
// entries to nodes outside the block are 0; its vectors use the padded value layout (zero ghost
// ring, pitch pv), so neighbour reads need no bounds checks.
#include <algorithm>
#include <cmath>

#include "kernels.cuh"

namespace spp {

struct ParLev {
    int nx, ny;
    long pv;                       // value pitch (padded layout, rows 0 .. ny+1)
    const double *a;               // [9][ny*nx]
    const double *wW, *wE;         // [ny*nx] interpolation weights of odd-x nodes
};

__device__ __forceinline__ double st9(const ParLev &L, int k, int i, int j)
{
    return L.a[(size_t)k * L.ny * L.nx + (size_t)(j - 1) * L.nx + (i - 1)];
}

// level 0: S A_CC from the global coefficients (corner block), S = hbar_i kbar_j
__global__ void k_par_level0(int n, long P, const double *__restrict__ aE, const double *__restrict__ aN,
                             const double *__restrict__ rr, const double *__restrict__ aW, const double *__restrict__ aS,
                             const double *__restrict__ hb, const double *__restrict__ kb, double *a)
{
    const long tot = (long)n * n;
    for (GridWalk gw(tot, n, 1); gw.ok(); gw.next()) {
        const long p = gw.p; const int j = gw.j, i = gw.i;
        const long g = (long)j * P + i;
        const double S = hb[i] * kb[j];
        const double D = ((aW[i] + aE[g]) + (aS[j] + aN[g])) + rr[g];
        double v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        v[4] = S * D;
        if (i > 1) v[3] = -S * aW[i];
        if (i < n) v[5] = -S * aE[g];
        if (j > 1) v[1] = -S * aS[j];
        if (j < n) v[7] = -S * aN[g];
#pragma unroll
        for (int k = 0; k < 9; ++k) a[(size_t)k * tot + p] = v[k];
    }
}

// interpolation weights of the odd-x nodes of level L (from its collapsed stencil)
__global__ void k_par_weights(ParLev L, double *wW, double *wE)
{
    const long tot = (long)L.nx * L.ny;
    for (GridWalk gw(tot, L.nx, 1); gw.ok(); gw.next()) {
        const long p = gw.p; const int j = gw.j, i = gw.i;
        double w = 0.0, e = 0.0;
        if (i & 1) {
            const double den = (st9(L, 1, i, j) + st9(L, 4, i, j)) + st9(L, 7, i, j);
            w = -((st9(L, 0, i, j) + st9(L, 3, i, j)) + st9(L, 6, i, j)) / den;
            e = -((st9(L, 2, i, j) + st9(L, 5, i, j)) + st9(L, 8, i, j)) / den;
        }
        wW[p] = w; wE[p] = e;
    }
}

// P_{(i,j),(I,j)}: weight of coarse node I in fine node i of row j (0 if not a parent)
__device__ __forceinline__ double par_P(const ParLev &F, int i, int j, int I)
{
    if (i < 1 || i > F.nx) return 0.0;
    const size_t p = (size_t)(j - 1) * F.nx + (i - 1);
    if ((i & 1) == 0) return I == i / 2 ? 1.0 : 0.0;
    if (I == (i - 1) / 2) return I >= 1 ? F.wW[p] : 0.0;
    if (I == (i + 1) / 2) return F.wE[p];
    return 0.0;
}

// C = P^T F P: every coarse row (I, j) gathers its fine rows i = 2I-1, 2I, 2I+1 in the oracle's
// accumulation order (fine i ascending, then dj, di, coarse column)
__global__ void k_par_galerkin(ParLev F, int ncx, double *ac)
{
    const long tot = (long)ncx * F.ny;
    for (GridWalk gw(tot, ncx, 1); gw.ok(); gw.next()) {
        const long p = gw.p; const int j = gw.j, I = gw.i;
        double v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int i = 2 * I - 1; i <= 2 * I + 1; ++i) {
            if (i > F.nx) continue;
            const double wi = par_P(F, i, j, I);
            if (wi == 0.0) continue;
            for (int dj = -1; dj <= 1; ++dj)
                for (int di = -1; di <= 1; ++di) {
                    const double a = st9(F, (dj + 1) * 3 + (di + 1), i, j);
                    if (a == 0.0) continue;
                    const int i2 = i + di, j2 = j + dj;
                    for (int I2 = (i2 - 1) / 2; I2 <= (i2 + 1) / 2; ++I2) {
                        if (I2 < 1 || I2 > ncx || i2 < 1 || i2 > F.nx) continue;
                        const double w2 = par_P(F, i2, j2, I2);
                        if (w2 == 0.0) continue;
                        v[(dj + 1) * 3 + (I2 - I + 1)] += wi * a * w2;
                    }
                }
        }
#pragma unroll
        for (int k = 0; k < 9; ++k) ac[(size_t)k * tot + p] = v[k];
    }
}

// rho = b - A e (nine-point); optional partial ||rho||^2 (kRedBlocks grid)
__global__ void __launch_bounds__(kRedThreads) k_par_resid(ParLev L, const double *__restrict__ b,
                                                           const double *__restrict__ e, double *rho, double *part)
{
    __shared__ double sm[32];
    double acc = 0.0;
    const long tot = (long)L.nx * L.ny;
    for (GridWalk gw(tot, L.nx, 1); gw.ok(); gw.next()) {
        const int j = gw.j, i = gw.i;
        const long g = (long)j * L.pv + i;
        double s = 0.0;
#pragma unroll
        for (int dj = -1; dj <= 1; ++dj)
#pragma unroll
            for (int di = -1; di <= 1; ++di) s += st9(L, (dj + 1) * 3 + (di + 1), i, j) * e[g + dj * L.pv + di];
        const double r = b[g] - s;
        rho[g] = r;
        acc += r * r;
    }
    if (part) {
        double v = acc;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
        if (lane == 0) sm[wid] = v;
        __syncthreads();
        if (threadIdx.x == 0) {
            double s2 = 0.0;
            for (int k = 0; k < nw; ++k) s2 += sm[k];
            part[blockIdx.x] = s2;
        }
        zero_tail(part);
    }
}

// S b (level 0 of the corner: the FE-scaled right-hand side)
__global__ void k_par_scale(int n, long pv, const double *__restrict__ b, const double *__restrict__ hb,
                            const double *__restrict__ kb, double *sb)
{
    const long tot = (long)n * n;
    for (GridWalk gw(tot, n, 1); gw.ok(); gw.next()) {
        const int j = gw.j, i = gw.i;
        sb[(long)j * pv + i] = (hb[i] * kb[j]) * b[(long)j * pv + i];
    }
}

// bc = P^T r
__global__ void k_par_restrict(ParLev F, int ncx, long pvc, const double *__restrict__ r, double *bc)
{
    const long tot = (long)ncx * F.ny;
    for (GridWalk gw(tot, ncx, 1); gw.ok(); gw.next()) {
        const int j = gw.j, I = gw.i;
        double s = 0.0;
        for (int i = 2 * I - 1; i <= 2 * I + 1; ++i)
            if (i <= F.nx) s += par_P(F, i, j, I) * r[(long)j * F.pv + i];
        bc[(long)j * pvc + I] = s;
    }
}

// e += P ec
__global__ void k_par_prolong(ParLev F, int ncx, long pvc, const double *__restrict__ ec, double *e)
{
    const long tot = (long)F.nx * F.ny;
    for (GridWalk gw(tot, F.nx, 1); gw.ok(); gw.next()) {
        const int j = gw.j, i = gw.i;
        double s = 0.0;
        for (int I = (i - 1) / 2; I <= (i + 1) / 2; ++I)
            if (I >= 1 && I <= ncx) s += par_P(F, i, j, I) * ec[(long)j * pvc + I];
        e[(long)j * F.pv + i] += s;
    }
}

// z += e on the n x n corner (padded layout)
__global__ void k_par_add(int n, long pv, double *z, const double *__restrict__ e)
{
    const long tot = (long)n * n;
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < tot; p += (long)gridDim.x * blockDim.x) {
        const long g = (long)(p / n + 1) * pv + (p % n + 1);
        z[g] += e[g];
    }
}

// One downstream point GS sweep (rows descending, columns descending) of the nine-point level L,
// in place on e (e = 0 first when `zero`).  Node (i,j) needs E and the row above (NW, N, NE) new,
// W, SW, S, SE old: with the schedule t = (nx - i) + 2 (ny - j) its new inputs have smaller t and
// its old inputs larger t, so every t is one parallel step (one node per row).  One CTA; thread k
// owns rows j with (ny - j) % T == k.
__global__ void __launch_bounds__(1024) k_par_gs(ParLev L, const double *__restrict__ b, double *e, int zero)
{
    const int nx = L.nx, ny = L.ny, T = blockDim.x;
    if (zero)
        for (long p = threadIdx.x; p < (long)(ny + 2) * L.pv; p += T) e[p] = 0.0;
    __syncthreads();
    const int steps = nx + 2 * (ny - 1);
    for (int t = 0; t < steps; ++t) {
        for (int r = threadIdx.x; r < ny; r += T) {        // r = ny - j
            const int j = ny - r, i = nx - (t - 2 * r);
            if (i < 1 || i > nx) continue;
            const long g = (long)j * L.pv + i;
            double s = b[g];
#pragma unroll
            for (int dj = -1; dj <= 1; ++dj)
#pragma unroll
                for (int di = -1; di <= 1; ++di)
                    if (di || dj) s -= st9(L, (dj + 1) * 3 + (di + 1), i, j) * e[g + dj * L.pv + di];
            e[g] = s / st9(L, 4, i, j);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------ host
static inline int pblocks(long work) { long b = (work + 255) / 256; return (int)std::max(1L, std::min(b, 148L * 16)); }

static ParLev parlev(const Ctx *c, int l)
{
    const ParLevel &P = c->plev[l];
    return ParLev{P.nx, c->n, P.pv, P.a, P.wW, P.wE};
}

cudaError_t par_alloc(Ctx *c)
{
    const int n = c->n;
    int nx = n, L = 0;
    size_t tot = 0;
    for (;;) {
        const long pv = round_up(nx + 2, 16);
        tot += 9 * (size_t)nx * n + 2 * (size_t)nx * n + 3 * (size_t)(n + 2) * pv;
        ++L;
        if (nx <= 4 || L >= kMaxLevels) break;
        nx /= 2;
    }
    tot += 2 * (size_t)(n + 2) * round_up(n + 2, 16);   // sb, rho0
    SPP_CUDA_TRY(cudaMalloc(&c->par_block, sizeof(double) * tot));
    SPP_CUDA_TRY(cudaMemsetAsync(c->par_block, 0, sizeof(double) * tot, c->st));
    double *p = c->par_block;
    nx = n;
    for (int l = 0; l < L; ++l) {
        ParLevel &P = c->plev[l];
        P.nx = nx; P.pv = round_up(nx + 2, 16);
        P.a = p; p += 9 * (size_t)nx * n;
        P.wW = p; p += (size_t)nx * n; P.wE = p; p += (size_t)nx * n;
        P.e = p; p += (size_t)(n + 2) * P.pv; P.rho = p; p += (size_t)(n + 2) * P.pv; P.b = p; p += (size_t)(n + 2) * P.pv;
        nx /= 2;
    }
    c->PL = L;
    const long pv0 = round_up(n + 2, 16);
    c->par_sb = p; p += (size_t)(n + 2) * pv0;
    c->par_rho = p;
    return cudaSuccess;
}

// the hierarchy from the (already set up) global coefficients and the level-0 FE weights
cudaError_t par_setup(Ctx *c)
{
    const int n = c->n;
    const Level &L0 = c->lev[0];
    k_par_level0<<<pblocks((long)n * n), 256, 0, c->st>>>(n, c->P, c->aE, c->aN, c->rr, c->aW, c->aS, L0.hb, L0.kb,
                                                          c->plev[0].a);
    c->launches++;
    for (int l = 0; l + 1 < c->PL; ++l) {
        const ParLev F = parlev(c, l);
        k_par_weights<<<pblocks((long)F.nx * n), 256, 0, c->st>>>(F, c->plev[l].wW, c->plev[l].wE);
        k_par_galerkin<<<pblocks((long)c->plev[l + 1].nx * n), 256, 0, c->st>>>(F, c->plev[l + 1].nx, c->plev[l + 1].a);
        c->launches += 2;
    }
    return cudaGetLastError();
}

static void par_gs(Ctx *c, int l, const double *b, double *e, bool zero)
{
    const ParLev L = parlev(c, l);
    const int threads = std::min(1024, (c->n + 31) / 32 * 32);
    ProfScope ps(c, 3, (double)L.nx * L.ny * 88.0);   // b, e, 9 coefficients read; e written
    k_par_gs<<<1, threads, 0, c->st>>>(L, b, e, zero ? 1 : 0);
    c->launches++;
}

// V(1,1) on level l for rhs b (padded layout of level l); result in plev[l].e
static void par_vcycle(Ctx *c, int l, const double *b)
{
    ParLevel &P = c->plev[l];
    const ParLev L = parlev(c, l);
    if (l == c->PL - 1) {
        par_gs(c, l, b, P.e, true);
        for (int s = 1; s < 4; ++s) par_gs(c, l, b, P.e, false);
        return;
    }
    ParLevel &C = c->plev[l + 1];
    par_gs(c, l, b, P.e, true);
    {
        ProfScope ps(c, 4, (double)L.nx * L.ny * 104.0);
        k_par_resid<<<pblocks((long)L.nx * L.ny), 256, 0, c->st>>>(L, b, P.e, P.rho, nullptr);
        k_par_restrict<<<pblocks((long)C.nx * L.ny), 256, 0, c->st>>>(L, C.nx, C.pv, P.rho, C.b);
        c->launches += 2;
    }
    par_vcycle(c, l + 1, C.b);
    {
        ProfScope ps(c, 5, (double)L.nx * L.ny * 32.0);
        k_par_prolong<<<pblocks((long)L.nx * L.ny), 256, 0, c->st>>>(L, C.nx, C.pv, C.e, P.e);
        c->launches++;
    }
    par_gs(c, l, b, P.e, false);
}

// M_CC^{-1} b_C (b_C in c->Bc, level-0 layout): z += V(S b - S A_CC z) from z = 0 until the
// FE-scaled residual has dropped by mg_reduction (R22); b0sq = ||S b_C||^2.  The result
// is left in c->Zc; returns the cycle count.
int par_corner_solve(Ctx *c, double b0sq, int *cap_hit, cudaError_t *err)
{
    const int n = c->n;
    const ParLev L = parlev(c, 0);
    const Level &L0 = c->lev[0];
    *cap_hit = 0; *err = cudaSuccess;
    cudaMemsetAsync(c->Zc, 0, sizeof(double) * L0.elems, c->st);
    k_par_scale<<<pblocks((long)n * n), 256, 0, c->st>>>(n, L.pv, c->Bc, L0.hb, L0.kb, c->par_sb);
    c->launches++;
    const double b0 = std::sqrt(b0sq);
    int cycles = 0;
    const int fixed = c->opt.mg_fixed_cycles;
    for (;;) {
        double *part = c->part;
        {
            ProfScope ps(c, 6, (double)n * n * 96.0);
            k_par_resid<<<kRedBlocks, kRedThreads, 0, c->st>>>(L, c->par_sb, c->Zc, c->par_rho, part);
            c->launches++;
        }
        double s = 0.0;
        if (fixed <= 0) {
            cudaError_t e = cudaMemcpyAsync(c->hpin, part, sizeof(double) * kRedBlocks, cudaMemcpyDeviceToHost, c->st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(c->st);
            if (e != cudaSuccess) { *err = e; break; }
            for (int k = 0; k < kRedBlocks; ++k) s += c->hpin[k];
        }
        if (fixed > 0) { if (cycles >= fixed) break; }
        else {
            if (std::sqrt(s) <= c->opt.mg_reduction * b0) break;
            if (cycles >= c->opt.mg_max_cycles) { *cap_hit = 1; break; }
        }
        par_vcycle(c, 0, c->par_rho);
        k_par_add<<<pblocks((long)n * n), 256, 0, c->st>>>(n, L.pv, c->Zc, c->plev[0].e);
        c->launches++;
        ++cycles;
    }
    return cycles;
}

}  // namespace spp
