// k_lines.cu -- the edge-layer line solves M_YY and M_XX.
//
// M_YY: block downstream Gauss-Seidel over lines of constant x, right-to-left; each line is
// the tridiagonal (-aS, D, -aN) along y with the West coupling dropped, the East (already
// solved) line and, on the top row, the North neighbour in I on the right-hand side.
// M_XX: lines of constant y, top-to-bottom, tridiagonal (-aW, D, -aE) along x, South dropped.
// Both are a chain  T_l z_l = s.v_l + C_l z_{l-1} (+ I coupling)  over the lines l.
//
// Setup (k_line_factor): the Thomas factorisation of every line ("performing the
// forward sweep of the Thomas algorithm to factor these systems" is part of the setup), stored
// as affine-recurrence coefficients
//     y_k = p_k v_k + e_k zprev_k + al_k y_{k-1}      (forward)
//     z_k = y_k + be_k z_{k+1}                        (backward)
// and a certified contraction bound of the chain, kappa_l = || T_l^{-1} C_l ||_inf
// = max_k (T_l^{-1} c_l)_k < 1 (T_l an M-matrix with T_l 1 >= c_l).
//
// Apply (k_lines): the chain is cut into chunks processed concurrently, one CTA per chunk;
// a chunk starts `warm-up` lines upstream of its first owned line from zero inflow, where the
// warm-up length L makes prod kappa < 1e-20 (so the result equals the sequential chain to
// rounding).  Each line is solved by the CTA with two
// block-wide affine scans (warp shuffles + one shared-memory level).
#include <algorithm>
#include <cmath>

#include "spp_internal.cuh"
#include "scan.cuh"

namespace spp {

// ------------------------------------------------------------------------------ setup
// One lane per line, 32 lines per warp (one warp per CTA), both chains in one launch
// (blockIdx.y = chain): chain 0 = X (lines of constant y, j = N-1-l; element k -> i = k+1),
// chain 1 = Y (lines of constant x, i = N-1-l; element k -> j = k+1).  The Thomas forward sweep
// (a dependent chain of reciprocals) runs 8 elements per block with the coefficient loads of the
// next block in flight; the outputs of 32 consecutive elements are staged in shared memory and
// stored as coalesced line segments (the factor arrays are line-major, as the apply reads them).
// The certified contraction kappa_l = max_k (T_l^{-1} c_l)_k is formed in the same kernel:
// forward part y = al y + e alongside the factorisation, backward part over the staged blocks of
// the scratch copy of y, last block first.
struct LineFactorOut { double *p, *e, *al, *be, *t, *kap, *scratch; };

constexpr int LFB = 32;   // elements per staged block

__global__ void __launch_bounds__(32) k_line_factor(int N, long P, const double *__restrict__ aE,
    const double *__restrict__ aN, const double *__restrict__ rr, const double *__restrict__ aW,
    const double *__restrict__ aS, int weighted, LineFactorOut ox, LineFactorOut oy)
{
    __shared__ double buf[5][32][LFB + 1];
    const int chain = blockIdx.y;
    const LineFactorOut &o = chain == 0 ? ox : oy;
    const int n = N / 2, nl = n - 1;
    const int lane = threadIdx.x, l0 = blockIdx.x * 32;
    const int l = min(l0 + lane, nl - 1);               // idle lanes redo the last line (not stored)
    const int line = N - 1 - l;
    // element k of this lane's line: coefficient address g0 + k*gs, 1D indices
    const long g0 = chain == 0 ? (long)line * P + 1 : P + line, gs = chain == 0 ? 1 : P;
    const double wsub = chain == 0 ? 0.0 : __ldg(aW + line);   // per-line 1D coefficients
    const double ssub = chain == 0 ? __ldg(aS + line) : 0.0;
    double gprev = 0.0, supprev = 0.0, y = 0.0;
    struct Raw { double E[8], Nn[8], R[8], w[8], s[8]; };
    auto load = [&](int k0, Raw &r) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = min(k0 + u, n - 1);
            const long g = g0 + (long)k * gs;
            r.E[u] = __ldg(aE + g); r.Nn[u] = __ldg(aN + g); r.R[u] = __ldg(rr + g);
            r.w[u] = chain == 0 ? __ldg(aW + k + 1) : wsub;
            r.s[u] = chain == 0 ? ssub : __ldg(aS + k + 1);
        }
    };
    auto factor8 = [&](int k0, const Raw &r) {          // elements k0..k0+7 (k0 % LFB + 8 <= LFB)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = k0 + u;
            if (k < n) {
                const double vE = r.E[u], vN = r.Nn[u], vw = r.w[u], vs = r.s[u];
                const double D = ((vw + vE) + (vs + vN)) + r.R[u];
                const double sub = chain == 0 ? vw : vs, sup = chain == 0 ? vE : vN, cE = chain == 0 ? vN : vE;
                const double den = (k == 0) ? D : D - sub * (supprev * gprev);
                const double gk = 1.0 / den;
                const double alk = (k == 0) ? 0.0 : sub * gk, ek = cE * gk;
                const int kk = k % LFB;
                buf[0][lane][kk] = (weighted ? D : 1.0) * gk;
                buf[1][lane][kk] = ek;
                buf[2][lane][kk] = alk;
                buf[3][lane][kk] = (k == n - 1) ? 0.0 : sup * gk;
                y = alk * y + ek;                       // forward part of T^{-1} c
                buf[4][lane][kk] = y;
                if (k == n - 1 && l0 + lane < nl) o.t[l] = sup * gk;   // coupling to the I neighbour
                gprev = gk; supprev = sup;
            }
        }
    };
    auto flush = [&](int kb) {                          // block kb..kb+LFB-1 of the 32 lines
        __syncwarp();
        const int k = kb + lane;
        for (int r = 0; r < 32 && l0 + r < nl; ++r) {
            if (k < n) {
                const long q = (long)(l0 + r) * n + k;
                o.p[q] = buf[0][r][lane]; o.e[q] = buf[1][r][lane]; o.al[q] = buf[2][r][lane];
                o.be[q] = buf[3][r][lane]; o.scratch[q] = buf[4][r][lane];
            }
        }
        __syncwarp();
    };
    Raw ra, rb;
    load(0, ra);
    for (int k0 = 0; k0 < n; k0 += 16) {                // two blocks of 8 per iteration (static buffers)
        load(k0 + 8, rb);
        factor8(k0, ra);
        if ((k0 + 8) % LFB == 0) flush(k0 + 8 - LFB);
        load(k0 + 16, ra);
        factor8(k0 + 8, rb);
        if ((k0 + 16) % LFB == 0 || k0 + 16 >= n) flush((k0 + 16 - 1) / LFB * LFB);
    }
    // backward part of T^{-1} c: z_k = y_k + be_k z_{k+1}; kappa = max z (blocks staged in buf)
    double z = 0.0, mx = 0.0;
    for (int kb = (n - 1) / LFB * LFB; kb >= 0; kb -= LFB) {
        __syncwarp();
        const int k = kb + lane;
#pragma unroll
        for (int r0 = 0; r0 < 32; r0 += 16) {           // 32 loads in flight per round
            double vb[16], vy[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const bool ok = k < n && l0 + r0 + r < nl;
                const long q = (long)(l0 + r0 + r) * n + k;
                vb[r] = ok ? o.be[q] : 0.0; vy[r] = ok ? o.scratch[q] : 0.0;
            }
#pragma unroll
            for (int r = 0; r < 16; ++r) { buf[3][r0 + r][lane] = vb[r]; buf[4][r0 + r][lane] = vy[r]; }
        }
        __syncwarp();
        for (int kk = min(LFB, n - kb) - 1; kk >= 0; --kk) {
            z = buf[4][lane][kk] + buf[3][lane][kk] * z;
            mx = fmax(mx, z);
        }
    }
    if (l0 + lane < nl) o.kap[l] = mx;
}

// ------------------------------------------------------------------------------ apply
template <int K>
struct LineRaw { double v[K], p[K], e[K], al[K], be[K], tI; };

// raw operands of line l for this thread's K elements (loads only; nothing depends on the chain)
template <int K>
__device__ __forceinline__ void line_load(const LineChain &ch, int l, int k0, const double *__restrict__ v,
                                          const double *z, LineRaw<K> &r)
{
    const int len = ch.len;
    const long base = ch.v0 + (long)l * ch.vline, fo = (long)l * len;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int kk = k0 + k;
        const bool ok = kk < len;
        r.v[k] = ok ? __ldg(v + base + (long)kk * ch.vstride) : 0.0;
        r.p[k] = ok ? __ldg(ch.p + fo + kk) : 0.0;
        r.e[k] = ok ? __ldg(ch.e + fo + kk) : 0.0;
        r.al[k] = ok ? __ldg(ch.al + fo + kk) : 0.0;
        r.be[k] = ok ? __ldg(ch.be + fo + kk) : 0.0;
    }
    // coupling to the I neighbour of the last element (written by the M_II sweep)
    r.tI = (k0 <= len - 1 && len - 1 < k0 + K) ? ch.t[l] * z[base + (long)(len - 1) * ch.vstride + ch.istep] : 0.0;
}

// Line solves of one chunk: lines start..last in order, each T_l z_l = s v_l + C_l z_{l-1} (+ I
// coupling) by two block-wide affine scans.  The raw operands of line l+1 are loaded while line l
// is scanned (register double buffer; the loop is unrolled by two so the buffers are static).
template <int K>
__global__ void __launch_bounds__(256) k_lines(LineChain cx, LineChain cy, const LineChunk *chunks,
                                               const double *__restrict__ v, double *z)
{
    __shared__ double sA[32], sB[64];
    const LineChunk ck = chunks[blockIdx.x];
    const LineChain &ch = ck.chain == 0 ? cx : cy;
    const int len = ch.len;
    const int k0 = threadIdx.x * K;
    double zp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) zp[k] = 0.0;
    auto solve = [&](int l, const LineRaw<K> &r) {
        double al[K], be[K], b[K], y[K], zz[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double bb = r.p[k] * r.v[k] + r.e[k] * zp[k];
            if (k0 + k == len - 1) bb += r.tI;
            b[k] = bb; al[k] = r.al[k]; be[k] = r.be[k];
        }
        fwd_scan<K>(al, b, y, sA, sB);
        bwd_scan<K>(be, y, zz, sA, sB);
        const long base = ch.v0 + (long)l * ch.vline;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            zp[k] = zz[k];
            const int kk = k0 + k;
            if (l >= ck.first && kk < len) z[base + (long)kk * ch.vstride] = zz[k];
        }
    };
    if (K <= 8) {
        LineRaw<K> ra, rb;
        line_load<K>(ch, ck.start, k0, v, z, ra);
        for (int l = ck.start; l <= ck.last; l += 2) {
            if (l + 1 <= ck.last) line_load<K>(ch, l + 1, k0, v, z, rb);
            solve(l, ra);
            if (l + 1 > ck.last) break;
            if (l + 2 <= ck.last) line_load<K>(ch, l + 2, k0, v, z, ra);
            solve(l + 1, rb);
        }
    } else {                                           // large K: no double buffer (registers)
        for (int l = ck.start; l <= ck.last; ++l) {
            LineRaw<K> r;
            line_load<K>(ch, l, k0, v, z, r);
            solve(l, r);
        }
    }
}

// ------------------------------------------------------------------------------ host
void plan_chunks(Ctx *c, const std::vector<double> &kx, const std::vector<double> &ky)
{
    c->chunks.clear();
    const int nl = c->n - 1;
    const double target = std::log(1e-20);
    const int budget = std::max(1, c->sm_count / 2);      // CTAs per chain: one resident CTA per SM
    for (int chain = 0; chain < 2; ++chain) {
        const std::vector<double> &k = chain == 0 ? kx : ky;
        std::vector<double> lg(nl + 1, 0.0);                 // prefix sums of log kappa
        for (int l = 0; l < nl; ++l) lg[l + 1] = lg[l] + std::log(std::max(k[l], 1e-300));
        auto warm = [&](int first) {                          // warm-up start for a chunk
            int st = first;
            while (st > 0 && lg[first] - lg[st] > target) --st;
            return st;
        };
        int bestG = nl; long bestCost = nl;
        for (int G = 1; G <= nl; G = (G < 8 ? G + 1 : G + G / 4)) {
            const int P = (nl + G - 1) / G;
            if (P > budget) continue;
            long worst = 0;
            for (int f = 0; f < nl; f += G) {
                const int last = std::min(nl - 1, f + G - 1);
                worst = std::max<long>(worst, last - warm(f) + 1);
            }
            if (worst < bestCost) { bestCost = worst; bestG = G; }
        }
        for (int f = 0; f < nl; f += bestG)
            c->chunks.push_back({chain, f, std::min(nl - 1, f + bestG - 1), warm(f)});
    }
}

cudaError_t setup_lines(Ctx *c)
{
    const int n = c->n, nl = n - 1, N = c->N;
    const long per = (long)nl * n;
    double *base = c->fac;
    double *xp = base, *xe = base + per, *xa = base + 2 * per, *xb = base + 3 * per;
    double *yp = base + 4 * per, *ye = base + 5 * per, *ya = base + 6 * per, *yb = base + 7 * per;
    const int nb = (nl + 31) / 32;
    const LineFactorOut ox{xp, xe, xa, xb, c->tX, c->kapX, c->cbuf};
    const LineFactorOut oy{yp, ye, ya, yb, c->tY, c->kapY, c->cbuf + per};
    k_line_factor<<<dim3(nb, 2), 32, 0, c->st>>>(N, c->P, c->aE, c->aN, c->rr, c->aW, c->aS, c->weighted, ox, oy);
    c->launches++;
    SPP_CUDA_TRY(cudaGetLastError());
    std::vector<double> kx(nl), ky(nl);
    SPP_CUDA_TRY(cudaMemcpyAsync(kx.data(), c->kapX, sizeof(double) * nl, cudaMemcpyDeviceToHost, c->st));
    SPP_CUDA_TRY(cudaMemcpyAsync(ky.data(), c->kapY, sizeof(double) * nl, cudaMemcpyDeviceToHost, c->st));
    SPP_CUDA_TRY(cudaStreamSynchronize(c->st));
    plan_chunks(c, kx, ky);
    // chains
    const long P = c->P;
    c->chX = LineChain{nl, n, 1, -P, (long)(N - 1) * P + 1, 1, xp, xe, xa, xb, c->tX};
    c->chY = LineChain{nl, n, P, -1, (long)1 * P + (N - 1), P, yp, ye, ya, yb, c->tY};
    if ((int)c->chunks.size() > c->nchunks_alloc) {
        if (c->d_chunks) cudaFree(c->d_chunks);
        SPP_CUDA_TRY(cudaMalloc(&c->d_chunks, sizeof(LineChunk) * c->chunks.size()));
        c->nchunks_alloc = (int)c->chunks.size();
    }
    SPP_CUDA_TRY(cudaMemcpyAsync(c->d_chunks, c->chunks.data(), sizeof(LineChunk) * c->chunks.size(),
                                 cudaMemcpyHostToDevice, c->st));
    int T = n / 8;
    if (T < 32) T = 32;
    if (T > 256) T = 256;
    c->lines_threads = T;
    return cudaStreamSynchronize(c->st);
}

void launch_lines(Ctx *c, const double *v, double *z)
{
    const int T = c->lines_threads, K = (c->n + T - 1) / T;
    const int nb = (int)c->chunks.size();
    double bytes = 0;   // algorithmic: v + 4 factors read, z written, per node of X and Y
    bytes = 2.0 * (c->n - 1) * c->n * 48.0;
    ProfScope ps(c, 2, bytes);
    if (K <= 1) k_lines<1><<<nb, T, 0, c->st>>>(c->chX, c->chY, c->d_chunks, v, z);
    else if (K <= 2) k_lines<2><<<nb, T, 0, c->st>>>(c->chX, c->chY, c->d_chunks, v, z);
    else if (K <= 4) k_lines<4><<<nb, T, 0, c->st>>>(c->chX, c->chY, c->d_chunks, v, z);
    else if (K <= 8) k_lines<8><<<nb, T, 0, c->st>>>(c->chX, c->chY, c->d_chunks, v, z);
    else k_lines<16><<<nb, T, 0, c->st>>>(c->chX, c->chY, c->d_chunks, v, z);
    c->launches++;
}

}  // namespace spp
