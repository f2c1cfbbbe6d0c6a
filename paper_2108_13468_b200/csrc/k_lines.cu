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
// One thread per line.  chain 0 = X (lines of constant y, j = N-1-l; element k -> i = k+1),
// chain 1 = Y (lines of constant x, i = N-1-l; element k -> j = k+1).
__global__ void k_line_factor(int chain, int N, long P, const double *aE, const double *aN,
                              const double *rr, const double *aW, const double *aS, int weighted,
                              double *p, double *e, double *al, double *be, double *t)
{
    const int n = N / 2, nl = n - 1;
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= nl) return;
    const int line = N - 1 - l;
    double gprev = 0.0, supprev = 0.0;
    for (int k = 0; k < n; ++k) {
        int i, j;
        double sub, sup, cE;
        if (chain == 0) { i = k + 1; j = line; } else { i = line; j = k + 1; }
        const long g = (long)j * P + i;
        const double vE = aE[g], vN = aN[g];
        const double D = ((aW[i] + vE) + (aS[j] + vN)) + rr[g];
        if (chain == 0) { sub = aW[i]; sup = vE; cE = vN; } else { sub = aS[j]; sup = vN; cE = vE; }
        const double den = (k == 0) ? D : D - sub * (supprev * gprev);
        const double gk = 1.0 / den;
        const long o = (long)l * n + k;
        p[o] = (weighted ? D : 1.0) * gk;
        e[o] = cE * gk;
        al[o] = (k == 0) ? 0.0 : sub * gk;
        const double bek = (k == n - 1) ? 0.0 : sup * gk;
        be[o] = bek;
        if (k == n - 1) t[l] = sup * gk;     // coupling to the I neighbour of the last element
        gprev = gk; supprev = sup;
    }
}

// kappa_l = max_k (T_l^{-1} c_l)_k from the stored factors: forward y = al*y + e, backward.
__global__ void k_line_kappa(int n, int nl, const double *e, const double *al, const double *be,
                             double *scratch, double *kap)
{
    const int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= nl) return;
    const long o = (long)l * n;
    double y = 0.0;
    for (int k = 0; k < n; ++k) { y = al[o + k] * y + e[o + k]; scratch[o + k] = y; }
    double z = 0.0, mx = 0.0;
    for (int k = n - 1; k >= 0; --k) { z = scratch[o + k] + be[o + k] * z; mx = fmax(mx, z); }
    kap[l] = mx;
}

// ------------------------------------------------------------------------------ apply
template <int K>
__global__ void __launch_bounds__(512) k_lines(LineChain cx, LineChain cy, const LineChunk *chunks,
                                               const double *__restrict__ v, double *z)
{
    __shared__ double sA[32], sB[64];
    const LineChunk ck = chunks[blockIdx.x];
    const LineChain &ch = ck.chain == 0 ? cx : cy;
    const int len = ch.len;
    const int k0 = threadIdx.x * K;
    double zp[K], al[K], be[K], b[K], y[K], zz[K];
#pragma unroll
    for (int k = 0; k < K; ++k) zp[k] = 0.0;
    for (int l = ck.start; l <= ck.last; ++l) {
        const long base = ch.v0 + (long)l * ch.vline;
        const long fo = (long)l * len;
        // prefetch the next line's factors into L2
        if (l < ck.last && k0 < len) {
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ch.p + fo + len + k0));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ch.e + fo + len + k0));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ch.al + fo + len + k0));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ch.be + fo + len + k0));
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const int kk = k0 + k;
            if (kk < len) {
                const double vv = v[base + (long)kk * ch.vstride];
                double bb = ch.p[fo + kk] * vv + ch.e[fo + kk] * zp[k];
                if (kk == len - 1) bb += ch.t[l] * z[base + (long)kk * ch.vstride + ch.istep];
                b[k] = bb; al[k] = ch.al[fo + kk]; be[k] = ch.be[fo + kk];
            } else {
                b[k] = 0.0; al[k] = 0.0; be[k] = 0.0;
            }
        }
        fwd_scan<K>(al, b, y, sA, sB);
        bwd_scan<K>(be, y, zz, sA, sB);
#pragma unroll
        for (int k = 0; k < K; ++k) {
            zp[k] = zz[k];
            const int kk = k0 + k;
            if (l >= ck.first && kk < len) z[base + (long)kk * ch.vstride] = zz[k];
        }
    }
}

// ------------------------------------------------------------------------------ host
void plan_chunks(Ctx *c, const std::vector<double> &kx, const std::vector<double> &ky)
{
    c->chunks.clear();
    const int nl = c->n - 1;
    const double target = std::log(1e-20);
    const int budget = std::max(1, c->sm_count);          // CTAs per chain
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
    const int tpb = 64, nb = (nl + tpb - 1) / tpb;
    k_line_factor<<<nb, tpb, 0, c->st>>>(0, N, c->P, c->aE, c->aN, c->rr, c->aW, c->aS, c->weighted,
                                         xp, xe, xa, xb, c->tX);
    k_line_factor<<<nb, tpb, 0, c->st>>>(1, N, c->P, c->aE, c->aN, c->rr, c->aW, c->aS, c->weighted,
                                         yp, ye, ya, yb, c->tY);
    k_line_kappa<<<nb, tpb, 0, c->st>>>(n, nl, xe, xa, xb, c->cbuf, c->kapX);
    k_line_kappa<<<nb, tpb, 0, c->st>>>(n, nl, ye, ya, yb, c->cbuf + per, c->kapY);
    c->launches += 4;
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
    if (T > 512) T = 512;
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
    else k_lines<8><<<nb, T, 0, c->st>>>(c->chX, c->chY, c->d_chunks, v, z);
    c->launches++;
}

}  // namespace spp
