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
// warm-up length L makes prod kappa < 1e-17 (so the result equals the sequential chain to
// rounding).  Each line is solved by the CTA with two
// block-wide affine scans (warp shuffles + one shared-memory level).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cmath>

#include "spp_internal.cuh"
#include "scan.cuh"
#include "tma.cuh"

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

// Block-parallel factorisation: one CTA per line, thread t owns K consecutive elements.  The
// pivots of the Thomas sweep obey den_k = D_k - s_k / den_{k-1} (s_k = sub_k sup_{k-1}), a
// continued fraction: den_k = p_k / q_k with (p_k, q_k)^T = M_k (p_{k-1}, q_{k-1})^T,
// M_k = [[D_k, -s_k], [1, 0]], (p_{-1}, q_{-1}) = (1, 0).  The prefix products of the M_k come from
// one block-wide scan of 2x2 matrices (each partial product rescaled by a power of two, which is
// exact and leaves the ratio unchanged), so a line costs O(log n) dependent steps instead of n
// reciprocals.  The contraction kappa_l = max_k (T_l^{-1} c_l)_k follows from two affine scans.
struct M2 { double a, b, c, d; };
__device__ __forceinline__ M2 m2mul(const M2 &x, const M2 &y)      // x * y, rescaled
{
    M2 r{fma(x.a, y.a, x.b * y.c), fma(x.a, y.b, x.b * y.d), fma(x.c, y.a, x.d * y.c), fma(x.c, y.b, x.d * y.d)};
    const double m = fmax(fmax(fabs(r.a), fabs(r.b)), fmax(fabs(r.c), fabs(r.d)));
    if (m > 0.0) {
        const double sc = ldexp(1.0, -ilogb(m));
        r.a *= sc; r.b *= sc; r.c *= sc; r.d *= sc;
    }
    return r;
}
__device__ __forceinline__ M2 m2shfl_up(const M2 &x, int d)
{
    return M2{__shfl_up_sync(0xffffffffu, x.a, d), __shfl_up_sync(0xffffffffu, x.b, d),
              __shfl_up_sync(0xffffffffu, x.c, d), __shfl_up_sync(0xffffffffu, x.d, d)};
}

template <int K>
__global__ void __launch_bounds__(256) k_line_factor_scan(int N, long P, const double *__restrict__ aE,
    const double *__restrict__ aN, const double *__restrict__ rr, const double *__restrict__ aW,
    const double *__restrict__ aS, int weighted, LineFactorOut ox, LineFactorOut oy)
{
    __shared__ double sA[32], sB[64];
    __shared__ M2 wtot[32];
    __shared__ double smax[32];
    const int chain = blockIdx.y;
    const LineFactorOut &o = chain == 0 ? ox : oy;
    const int n = N / 2;
    const int l = blockIdx.x;                           // line
    const int line = N - 1 - l;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int k0 = threadIdx.x * K;
    const long g0 = chain == 0 ? (long)line * P + 1 : P + line, gs = chain == 0 ? 1 : P;
    const double w1 = chain == 0 ? 0.0 : __ldg(aW + line), s1 = chain == 0 ? __ldg(aS + line) : 0.0;
    double D[K], sub[K], sup[K], cE[K], sv[K];
    double supprev = 0.0;
#pragma unroll
    for (int u = -1; u < K; ++u) {
        const int k = k0 + u;
        if (k < 0 || k >= n) { if (u >= 0) { D[u] = 1.0; sub[u] = sup[u] = cE[u] = sv[u] = 0.0; } continue; }
        const long g = g0 + (long)k * gs;
        const double vE = __ldg(aE + g), vN = __ldg(aN + g);
        const double vw = chain == 0 ? __ldg(aW + k + 1) : w1, vs = chain == 0 ? s1 : __ldg(aS + k + 1);
        const double su = chain == 0 ? vE : vN;
        if (u < 0) { supprev = su; continue; }
        D[u] = ((vw + vE) + (vs + vN)) + __ldg(rr + g);
        sub[u] = chain == 0 ? vw : vs;
        sup[u] = su;
        cE[u] = chain == 0 ? vN : vE;
        sv[u] = k == 0 ? 0.0 : sub[u] * supprev;        // s_k = sub_k sup_{k-1}
        supprev = su;
    }
    // thread aggregate M_{k0+K-1} ... M_{k0}
    M2 agg{1.0, 0.0, 0.0, 1.0};
#pragma unroll
    for (int u = 0; u < K; ++u) agg = m2mul(M2{D[u], -sv[u], 1.0, 0.0}, agg);
    // inclusive warp scan (later * earlier)
    M2 inc = agg;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const M2 up = m2shfl_up(inc, d);
        if (lane >= d) inc = m2mul(inc, up);
    }
    if (lane == 31) wtot[wid] = inc;
    __syncthreads();
    if (wid == 0) {                                     // exclusive prefix over warps
        M2 x = lane < nw ? wtot[lane] : M2{1.0, 0.0, 0.0, 1.0};
        for (int d = 1; d < nw; d <<= 1) {
            const M2 up = m2shfl_up(x, d);
            if (lane >= d) x = m2mul(x, up);
        }
        const M2 ex = m2shfl_up(x, 1);
        __syncwarp();
        if (lane < nw) wtot[lane] = lane == 0 ? M2{1.0, 0.0, 0.0, 1.0} : ex;
    }
    __syncthreads();
    M2 exl = m2shfl_up(inc, 1);                         // product of the earlier lanes of the warp
    if (lane == 0) exl = M2{1.0, 0.0, 0.0, 1.0};
    const M2 pre = m2mul(exl, wtot[wid]);               // all matrices before this thread
    double pp = pre.a, qq = pre.c;                      // (p, q) at k0 - 1 = pre (1, 0)^T
    double g[K], al[K], ee[K], be[K];
#pragma unroll
    for (int u = 0; u < K; ++u) {
        const int k = k0 + u;
        const double np = fma(D[u], pp, -sv[u] * qq), nq = pp;
        const double m = fmax(fabs(np), fabs(nq));
        const double sc = m > 0.0 ? ldexp(1.0, -ilogb(m)) : 1.0;
        pp = np * sc; qq = nq * sc;
        g[u] = qq / pp;                                 // 1 / den_k
        const bool in = k < n;
        al[u] = (in && k > 0) ? sub[u] * g[u] : 0.0;
        ee[u] = in ? cE[u] * g[u] : 0.0;
        be[u] = (in && k < n - 1) ? sup[u] * g[u] : 0.0;
        if (in) {
            const long q = (long)l * n + k;
            o.p[q] = (weighted ? D[u] : 1.0) * g[u];
            o.e[q] = ee[u];
            o.al[q] = al[u];
            o.be[q] = be[u];
            if (k == n - 1) o.t[l] = sup[u] * g[u];    // coupling to the I neighbour
        }
    }
    // kappa = max_k (T^{-1} c)_k: forward y = al y + e, backward z = be z + y
    double y[K], z[K];
    fwd_scan<K>(al, ee, y, sA, sB);
    bwd_scan<K>(be, y, z, sA, sB);
    double mx = 0.0;
#pragma unroll
    for (int u = 0; u < K; ++u) if (k0 + u < n) mx = fmax(mx, z[u]);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, d));
    if (lane == 0) smax[wid] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        for (int k = 0; k < nw; ++k) m = fmax(m, smax[k]);
        o.kap[l] = m;
    }
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
    // unpredicated loads from a clamped index (elements past the line end are masked where they
    // are used): a predicated load with a zero fill makes the next write of the register wait for
    // the load, which serialised the prefetch of line l+1 behind the scans of line l
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int kk = min(k0 + k, len - 1);
        r.v[k] = __ldg(v + base + (long)kk * ch.vstride);
        r.p[k] = __ldg(ch.p + fo + kk);
        r.e[k] = __ldg(ch.e + fo + kk);
        r.al[k] = __ldg(ch.al + fo + kk);
        r.be[k] = __ldg(ch.be + fo + kk);
    }
    // coupling to the I neighbour of the last element (written by the M_II sweep)
    r.tI = ch.t[l] * z[base + (long)(len - 1) * ch.vstride + ch.istep];   // used by the owner of element len-1 only
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
            const bool in = k0 + k < len;
            double bb = r.p[k] * r.v[k] + r.e[k] * zp[k];
            if (k0 + k == len - 1) bb += r.tI;
            b[k] = in ? bb : 0.0; al[k] = in ? r.al[k] : 0.0; be[k] = in ? r.be[k] : 0.0;
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

// TMA-staged variant (line length a multiple of 64, K elements per thread): the four factor
// arrays of a line are one 2D box each (the line viewed as len/16 rows of 16, 128B swizzle), the
// operand v is one box of its row (X lines) or len/256 boxes of a 2-column strip (Y lines,
// columns i&~1, i&~1 + 1); all land in a shared-memory stage with one mbarrier.  Each thread reads
// its K values from the stage, the block syncs, and thread 0 refills the stage for a later line
// while the scans of this line run.  Loading through the LSU (one 8-byte element per lane per
// row/column of the grid) had left the line chains waiting on the L1 tag stage and on load
// latency (ncu: stall_long_sb + stall_lg ~57% of samples).
struct LineMaps { CUtensorMap f[2][4]; CUtensorMap vx, vy; };

__device__ __forceinline__ int swz16(int o)            // 128B-swizzled offset of element o (16 per row)
{
    const int r = o >> 4, c = o & 15;
    return (r << 4) + ((((c >> 1) ^ (r & 7))) << 1) + (c & 1);
}

template <int K>
__global__ void __launch_bounds__(256) k_lines_tma(LineChain cx, LineChain cy, const LineChunk *chunks,
                                                   double *z, double *ysc, int N, long P, int nst,
                                                   const __grid_constant__ LineMaps m)
{
    extern __shared__ double lsm_raw[];
    __shared__ double sA[32], sB[64];
    __shared__ __align__(8) unsigned long long full[2];
    const LineChunk ck = chunks[blockIdx.x];
    const int chain = ck.chain;
    const LineChain &ch = chain == 0 ? cx : cy;
    const int len = ch.len;
    const int k0 = threadIdx.x * K;
    double *sm = lsm_raw + (((1024u - ((unsigned)__cvta_generic_to_shared(lsm_raw) & 1023u)) & 1023u) >> 3);
    const int stage = 6 * len;                          // doubles: 4 factor boxes + v (<= 2 len)
    const int vxr = len / 16 + 1, nvx = (vxr + 255) / 256, vxb = ((vxr + nvx - 1) / nvx + 7) / 8 * 8;   // X: row boxes (1 KB multiples)
    const unsigned vbytes = chain == 0 ? (unsigned)(nvx * vxb * 16) * 8u : (unsigned)len * 16u;
    const unsigned bytes = 4u * (unsigned)len * 8u + vbytes;
    const int vrows = len < 256 ? len : 256;
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s)
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int l, int s) {                    // thread 0: all boxes of line l into stage s
        const unsigned bar = (unsigned)__cvta_generic_to_shared(&full[s]);
        const unsigned dst = (unsigned)__cvta_generic_to_shared(sm + (size_t)s * stage);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
#pragma unroll
        for (int f = 0; f < 4; ++f) tma_load(dst + (unsigned)(f * len * 8), &m.f[chain][f], 0, l * (len >> 4), bar);
        const long g0 = ch.v0 + (long)l * ch.vline;     // grid index of element 0 of the line
        if (chain == 0) {
            for (int b = 0; b < nvx; ++b)
                tma_load(dst + (unsigned)((4 * len + 16 * vxb * b) * 8), &m.vx, 0, (int)((g0 - 1) >> 4) + vxb * b, bar);
        }
        else {
            const int i = (int)(g0 % P), x = i & ~1;
            for (int r0 = 0; r0 < len; r0 += vrows)
                tma_load(dst + (unsigned)((4 * len + 2 * r0) * 8), &m.vy, x, 1 + r0, bar);
        }
    };
    double zp[K];
#pragma unroll
    for (int k = 0; k < K; ++k) zp[k] = 0.0;
    const int nlines = ck.last - ck.start + 1;
    if (threadIdx.x == 0)
        for (int s = 0; s < nst && s < nlines; ++s) issue(ck.start + s, s);
    const bool owner = k0 <= len - 1 && len - 1 < k0 + K;   // holds the element coupled to I
    double tnext = 0.0;
    if (owner) {
        const long g0 = ch.v0 + (long)ck.start * ch.vline;
        tnext = ch.t[ck.start] * z[g0 + (long)(len - 1) * ch.vstride + ch.istep];
    }
#ifdef SPP_LINES_PROF
    long long q0 = 0, q1 = 0, q2 = 0, q3 = 0, q4 = 0;
#define LP(v) long long v; asm volatile("mov.u64 %0, %%clock64;" : "=l"(v) :: "memory")
#else
#define LP(v)
#endif
    for (int it = 0; it < nlines; ++it) {
        const int l = ck.start + it, s = it % nst;
        LP(ta);
        mbar_wait((unsigned)__cvta_generic_to_shared(&full[s]), (unsigned)((it / nst) & 1));
        LP(tb);
        const double *st = sm + (size_t)s * stage;
        double p[K], e[K], al[K], be[K], vv[K];
#pragma unroll
        for (int k = 0; k < K; k += 2) {                // pairs share a 16-byte swizzle unit
            const int o = swz16(k0 + k);
            const double2 a0 = *reinterpret_cast<const double2 *>(st + o);
            const double2 a1 = *reinterpret_cast<const double2 *>(st + len + o);
            const double2 a2 = *reinterpret_cast<const double2 *>(st + 2 * len + o);
            const double2 a3 = *reinterpret_cast<const double2 *>(st + 3 * len + o);
            p[k] = a0.x; p[k + 1] = a0.y; e[k] = a1.x; e[k + 1] = a1.y;
            al[k] = a2.x; al[k + 1] = a2.y; be[k] = a3.x; be[k + 1] = a3.y;
        }
        const long g0 = ch.v0 + (long)l * ch.vline;
        double *zs = sm + (size_t)nst * stage;          // z staging (free until the scans end)
        if (chain == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) vv[k] = st[4 * len + swz16(k0 + k + 1)];
        } else {
            // the strip holds (column pair) x rows: reading a thread's K consecutive rows
            // directly would put every lane on one bank; repack the line's column through the
            // z staging buffer (coalesced, XOR-swizzled within 16) first
            const int ic = (int)(g0 % P) & 1;
            __syncthreads();                            // the previous line's stores from zs are done
            for (int kk = threadIdx.x; kk < len; kk += blockDim.x) zs[kk ^ ((kk >> 4) & 15)] = st[4 * len + 2 * kk + ic];
            __syncthreads();
#pragma unroll
            for (int k = 0; k < K; ++k) vv[k] = zs[(k0 + k) ^ (((k0 + k) >> 4) & 15)];
        }
        const double tI = tnext;
        LP(tc);
        __syncthreads();                                // stage s fully read
        LP(td);
        if (threadIdx.x == 0 && it + nst < nlines) issue(l + nst, s);
        if (owner && it + 1 < nlines) {                 // I coupling of the next line, one line ahead
            const long g1 = g0 + ch.vline;
            tnext = ch.t[l + 1] * z[g1 + (long)(len - 1) * ch.vstride + ch.istep];
        }
        double b[K], y[K], zz[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const bool in = k0 + k < len;
            double bb = p[k] * vv[k] + e[k] * zp[k];
            if (k0 + k == len - 1) bb += tI;
            b[k] = in ? bb : 0.0;
            if (!in) { al[k] = 0.0; be[k] = 0.0; }
        }
        fwd_scan<K, false>(al, b, y, sA, sB);   // the backward scan follows; the z staging barrier ends the line
        bwd_scan<K, false>(be, y, zz, sA, sB);
        LP(te);
        // the line's results leave as coalesced segments through shared memory: X lines are row
        // segments of z, Y lines (columns of z) go line-major to the scratch (k_ysc_transpose)
#pragma unroll
        for (int k = 0; k < K; ++k) {
            zp[k] = zz[k];
            const int kk = k0 + k;
            zs[kk ^ ((kk >> 4) & 15)] = zz[k];          // XOR swizzle within 16: two-way on the stores, none on the reads
        }
        __syncthreads();
        if (l >= ck.first) {
            double *out = chain == 0 ? z + g0 : ysc + (long)l * len;
            for (int kk = threadIdx.x; kk < len; kk += blockDim.x) out[kk] = zs[kk ^ ((kk >> 4) & 15)];
        }
#ifdef SPP_LINES_PROF
        LP(tf);
        q0 += tb - ta; q1 += tc - tb; q2 += td - tc; q3 += te - td; q4 += tf - te;
#endif
    }
#ifdef SPP_LINES_PROF
    if ((threadIdx.x == 0 || threadIdx.x == 255) && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
        printf("[lines-prof] cta %d thr %d lines %d per line: wait %lld read %lld relsync %lld scans %lld store %lld\n",
               blockIdx.x, threadIdx.x, nlines, q0 / nlines, q1 / nlines, q2 / nlines, q3 / nlines, q4 / nlines);
#endif
}

// ------------------------------------------------------------------------------ host
// Chunks of the owned lines [l0, l1] of one chain (all lines on one GPU; a row strip's X lines
// or a bottom strip's share of the Y lines in a distributed solve; l1 < l0: none).
// A chunk starts `warm-up` lines upstream of its first owned line, where prod kappa over the
// warm-up is <= 1e-17 (so it equals the sequential chain to rounding); those lines' operands are
// a row strip's halo.  budget: CTAs for the chain.  Pure host function of the contractions.
std::vector<LineChunk> plan_chain_chunks(int chain, const std::vector<double> &k, int l0, int l1, int budget)
{
    std::vector<LineChunk> out;
    const int nl = (int)k.size(), cnt = l1 - l0 + 1;
    if (cnt <= 0) return out;
    const double target = std::log(1e-17);   // below fp64 rounding, as the MG halos
    budget = std::max(1, budget);
    std::vector<double> lg(nl + 1, 0.0);                 // prefix sums of log kappa
    for (int l = 0; l < nl; ++l) lg[l + 1] = lg[l] + std::log(std::max(k[l], 1e-300));
    // warm-up start of a chunk beginning at line f: the largest st <= f with
    // lg[f] - lg[st] <= target (prod kappa small enough), or 0.  lg decreases, so st(f) is
    // nondecreasing in f: one two-pointer pass (the plan runs inside every setup).
    std::vector<int> wst(nl + 1, 0);
    for (int f = 0, st = 0; f <= nl; ++f) {
        while (st < f && lg[f] - lg[st + 1] <= target) ++st;  // advance while st+1 still suffices
        wst[f] = (lg[f] - lg[st] <= target) ? st : 0;
    }
    int bestG = cnt; long bestCost = 1L << 40;
    for (int G = (cnt + budget - 1) / budget; G <= cnt; ++G) {   // smallest chunks that fit the budget first
        const int P = (cnt + G - 1) / G;
        if (P > budget) continue;
        long worst = 0;
        for (int f = l0; f <= l1; f += G) {
            const int last = std::min(l1, f + G - 1);
            worst = std::max<long>(worst, last - wst[f] + 1);
        }
        if (worst < bestCost) { bestCost = worst; bestG = G; }
    }
    for (int f = l0; f <= l1; f += bestG) out.push_back({chain, f, std::min(l1, f + bestG - 1), wst[f]});
    if (getenv("SPP_DEBUG_LINES"))
        fprintf(stderr, "[spp] line chain %d: lines %d..%d of %d, chunk %d lines, %d chunks, worst %ld lines (kappa %.6g .. %.6g)\n",
                chain, l0, l1, nl, bestG, (cnt + bestG - 1) / bestG, bestCost, *std::min_element(k.begin(), k.end()),
                *std::max_element(k.begin(), k.end()));
    return out;
}

// warm-up starts of chunks beginning at every line (as in plan_chain_chunks)
static std::vector<int> warm_starts(const std::vector<double> &k)
{
    const int nl = (int)k.size();
    const double target = std::log(1e-17);
    std::vector<double> lg(nl + 1, 0.0);
    for (int l = 0; l < nl; ++l) lg[l + 1] = lg[l] + std::log(std::max(k[l], 1e-300));
    std::vector<int> wst(nl + 1, 0);
    for (int f = 0, st = 0; f <= nl; ++f) {
        while (st < f && lg[f] - lg[st + 1] <= target) ++st;
        wst[f] = (lg[f] - lg[st] <= target) ? st : 0;
    }
    return wst;
}
// greedy chunks of lines l0..l1 whose span (warm-up + owned lines) is at most T (at least one
// owned line each); returns their number, appends them to *out when given
static int greedy_chunks(int chain, const std::vector<int> &wst, int l0, int l1, int T, std::vector<LineChunk> *out)
{
    int cnt = 0;
    for (int f = l0; f <= l1;) {
        const int last = std::min(l1, std::max(f, wst[f] + T - 1));
        if (out) out->push_back({chain, f, last, wst[f]});
        ++cnt;
        f = last + 1;
    }
    return cnt;
}
// One GPU, both chains in one launch of `budget` CTAs (one per SM): the CTAs are split between
// the chains so that the longest chunk, in time, is as short as possible.  A chunk's time is its
// span in lines times the chain's per-line cost; a Y line costs ~1.2 X lines (its operand column
// is repacked through shared memory; SPP_LINES_PROF: ~6.1k vs ~5.1k cycles per line at cfg4).
// With the same number of CTAs per chain, the Y chunks (warm-up ~22 lines at cfg4) ran 50 lines
// against the X chunks' 28.
void plan_chunks_balanced(Ctx *c, const std::vector<double> &kx, const std::vector<double> &ky, int nl, int budget)
{
    const std::vector<int> wx = warm_starts(kx), wy = warm_starts(ky);
    const double ycost = 1.2;
    auto need = [&](int tau) {
        return greedy_chunks(0, wx, 0, nl - 1, tau, nullptr) + greedy_chunks(1, wy, 0, nl - 1, std::max(1, (int)(tau / ycost)), nullptr);
    };
    int lo = 1, hi = (int)(2 * ycost * nl) + 2;         // need(hi) = 2 <= budget
    while (lo < hi) {                                   // smallest tau with need(tau) <= budget
        const int mid = (lo + hi) / 2;
        if (need(mid) <= std::max(2, budget)) hi = mid; else lo = mid + 1;
    }
    c->chunks.clear();
    greedy_chunks(0, wx, 0, nl - 1, lo, &c->chunks);
    greedy_chunks(1, wy, 0, nl - 1, std::max(1, (int)(lo / ycost)), &c->chunks);
    if (getenv("SPP_DEBUG_LINES"))
        fprintf(stderr, "[spp] line chains (balanced): %zu chunks, X span <= %d, Y span <= %d lines\n", c->chunks.size(), lo,
                std::max(1, (int)(lo / ycost)));
}

void plan_chunks(Ctx *c, const std::vector<double> &kx, const std::vector<double> &ky, const int lo[2],
                 const int hi[2], int budget)
{
    c->chunks.clear();
    for (int chain = 0; chain < 2; ++chain) {
        const auto v = plan_chain_chunks(chain, chain == 0 ? kx : ky, lo[chain], hi[chain], budget);
        c->chunks.insert(c->chunks.end(), v.begin(), v.end());
    }
}

// Setup of the line chains in two halves around one host synchronisation (setup_2d_ctx batches
// it with the MG levels' contraction factors): the factor scans and the kappa read-back, then
// the chunk plan.
cudaError_t setup_lines_launch(Ctx *c)
{
    const int n = c->n, nl = n - 1, N = c->N;
    const long per = (long)nl * n;
    double *base = c->fac;
    double *xp = base, *xe = base + per, *xa = base + 2 * per, *xb = base + 3 * per;
    double *yp = base + 4 * per, *ye = base + 5 * per, *ya = base + 6 * per, *yb = base + 7 * per;
    const int nb = (nl + 31) / 32;
    const LineFactorOut ox{xp, xe, xa, xb, c->tX, c->kapX, c->cbuf};
    const LineFactorOut oy{yp, ye, ya, yb, c->tY, c->kapY, c->cbuf + per};
    int TF = n / 8;
    if (TF < 32) TF = 32;
    if (TF > 256) TF = 256;
    const int K = (n + TF - 1) / TF;
    const char *seqf = getenv("SPP_SEQ_LINE_FACTOR");
    const bool seq = (seqf && seqf[0] == '1') || (K != 2 && K != 4 && K != 8 && K != 16);
    if (seq) k_line_factor<<<dim3(nb, 2), 32, 0, c->st>>>(N, c->P, c->aE, c->aN, c->rr, c->aW, c->aS, c->weighted, ox, oy);
    else if (K == 2) k_line_factor_scan<2><<<dim3(nl, 2), TF, 0, c->st>>>(N, c->P, c->aE, c->aN, c->rr, c->aW, c->aS, c->weighted, ox, oy);
    else if (K == 4) k_line_factor_scan<4><<<dim3(nl, 2), TF, 0, c->st>>>(N, c->P, c->aE, c->aN, c->rr, c->aW, c->aS, c->weighted, ox, oy);
    else if (K == 8) k_line_factor_scan<8><<<dim3(nl, 2), TF, 0, c->st>>>(N, c->P, c->aE, c->aN, c->rr, c->aW, c->aS, c->weighted, ox, oy);
    else k_line_factor_scan<16><<<dim3(nl, 2), TF, 0, c->st>>>(N, c->P, c->aE, c->aN, c->rr, c->aW, c->aS, c->weighted, ox, oy);
    c->launches++;
    SPP_CUDA_TRY(cudaGetLastError());
    c->kx.assign(nl, 0.0); c->ky.assign(nl, 0.0);
    SPP_CUDA_TRY(cudaMemcpyAsync(c->kx.data(), c->kapX, sizeof(double) * nl, cudaMemcpyDeviceToHost, c->st));
    SPP_CUDA_TRY(cudaMemcpyAsync(c->ky.data(), c->kapY, sizeof(double) * nl, cudaMemcpyDeviceToHost, c->st));
    return cudaSuccess;
}

// after the stream has synchronised (kappa on the host)
cudaError_t setup_lines_plan(Ctx *c)
{
    const int n = c->n, nl = n - 1, N = c->N;
    const long per = (long)nl * n;
    double *base = c->fac;
    double *xp = base, *xe = base + per, *xa = base + 2 * per, *xb = base + 3 * per;
    double *yp = base + 4 * per, *ye = base + 5 * per, *ya = base + 6 * per, *yb = base + 7 * per;
    if (c->line_lo[0] < 0) {                            // one GPU: every line, the GPU shared by both chains
        plan_chunks_balanced(c, c->kx, c->ky, nl, c->sm_count);
    } else {
        plan_chunks(c, c->kx, c->ky, c->line_lo, c->line_hi, c->sm_count);
    }
    // chains
    const long P = c->P;
    c->chX = LineChain{nl, n, 1, -P, (long)(N - 1) * P + 1, 1, xp, xe, xa, xb, c->tX};
    c->chY = LineChain{nl, n, P, -1, (long)1 * P + (N - 1), P, yp, ye, ya, yb, c->tY};
    if ((int)c->chunks.size() > c->nchunks_alloc) {
        if (c->d_chunks) cudaFree(c->d_chunks);
        SPP_CUDA_TRY(cudaMalloc(&c->d_chunks, sizeof(LineChunk) * c->chunks.size()));
        c->nchunks_alloc = (int)c->chunks.size();
    }
    if (!c->chunks.empty())
        SPP_CUDA_TRY(cudaMemcpyAsync(c->d_chunks, c->chunks.data(), sizeof(LineChunk) * c->chunks.size(),
                                     cudaMemcpyHostToDevice, c->st));
    int T = n / 8;
    if (T < 32) T = 32;
    if (T > 256) T = 256;
    c->lines_threads = T;
    return cudaSuccess;   // the chunk table's upload is stream-ordered before every use; c->chunks
                          // changes only in the next setup, after its own synchronisation
}

cudaError_t setup_lines(Ctx *c)
{
    SPP_CUDA_TRY(setup_lines_launch(c));
    SPP_CUDA_TRY(cudaStreamSynchronize(c->st));
    SPP_CUDA_TRY(setup_lines_plan(c));
    return cudaStreamSynchronize(c->st);
}

// dynamic shared memory of k_lines_tma: 227 KB per block minus its static part (rounded up)
constexpr int kLinesSmemMax = 227 * 1024 - 2048;

// per-device kernel attributes (spp_create, on the context's device)
cudaError_t lines_init()
{
    SPP_CUDA_TRY(cudaFuncSetAttribute(k_lines_tma<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kLinesSmemMax));
    SPP_CUDA_TRY(cudaFuncSetAttribute(k_lines_tma<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kLinesSmemMax));
    return cudaSuccess;
}

static size_t lines_tma_smem(int len, int nst)
{
    return ((size_t)nst * 6 * len + len) * sizeof(double) + 1024;   // stages + z staging (+ alignment)
}

// z (Y region) <- scratch: line l (column i = N-1-l), element k (row j = k+1); 32x32 tiles; lines
// la .. nl-1 (la > 0: a bottom strip's share of the Y lines)
__global__ void k_ysc_transpose(int nl, int len, long P, int N, const double *__restrict__ ysc, double *z, int la)
{
    __shared__ double t[32][33];
    const int l0 = la + blockIdx.x * 32, k0 = blockIdx.y * 32;
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int l = l0 + r, k = k0 + threadIdx.x;
        if (l < nl && k < len) t[r][threadIdx.x] = ysc[(long)l * len + k];
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int k = k0 + r, l = l0 + 31 - threadIdx.x;   // consecutive lanes: consecutive columns i
        if (k < len && l < nl && l >= l0) z[(long)(k + 1) * P + (N - 1 - l)] = t[31 - threadIdx.x][r];
    }
}

// the TMA-staged line kernel, when the line length allows it (multiple of 64, at most 4096)
static bool launch_lines_tma(Ctx *c, const double *v, double *z)
{
    const int len = c->n, T = c->lines_threads, K = (len + T - 1) / T;
    // 1 KB aligned boxes (the 128B swizzle phase) need len % 128 == 0
    if (len % 128 != 0 || len > 4096 || (K != 8 && K != 16) || T * K != len || c->no_lines_tma) return false;
    const int nst = lines_tma_smem(len, 2) <= (size_t)kLinesSmemMax ? 2 : 1;   // len 4096: one stage (196 KB)
    if (lines_tma_smem(len, nst) > (size_t)kLinesSmemMax) return false;
    const size_t sm = lines_tma_smem(len, nst);
    LineMaps m;
    const int nl = c->n - 1;
    const unsigned long long rows = (unsigned long long)nl * len / 16;
    const LineChain *chs[2] = {&c->chX, &c->chY};
    for (int ci = 0; ci < 2; ++ci) {
        const double *fa[4] = {chs[ci]->p, chs[ci]->e, chs[ci]->al, chs[ci]->be};
        for (int f = 0; f < 4; ++f) {
            const CUtensorMap *t = tmap2d(c, fa[f], 16, rows, 128, 16, (unsigned)(len / 16), true);
            if (!t) return false;
            m.f[ci][f] = *t;
        }
    }
    const int vxr = len / 16 + 1, nvx = (vxr + 255) / 256, vxb = ((vxr + nvx - 1) / nvx + 7) / 8 * 8;
    const CUtensorMap *tx = tmap2d(c, v, 16, (unsigned long long)c->G / 16, 128, 16, (unsigned)vxb, true);
    const CUtensorMap *ty = tmap2d(c, v, (unsigned long long)c->P, (unsigned long long)c->N + 1,
                                   (unsigned long long)c->P * 8, 2, (unsigned)std::min(len, 256), false);
    if (!tx || !ty) return false;
    m.vx = *tx; m.vy = *ty;
    const int nb = (int)c->chunks.size();
    double *ysc = c->cbuf;                              // free during the FGMRES iterations
    if (K == 8) k_lines_tma<8><<<nb, T, sm, c->st>>>(c->chX, c->chY, c->d_chunks, z, ysc, c->N, c->P, nst, m);
    else k_lines_tma<16><<<nb, T, sm, c->st>>>(c->chX, c->chY, c->d_chunks, z, ysc, c->N, c->P, nst, m);
    c->launches++;
    // the owned Y lines (a contiguous range) back into z
    int ya = nl, yb = -1;
    for (const auto &ck : c->chunks)
        if (ck.chain == 1) { ya = std::min(ya, ck.first); yb = std::max(yb, ck.last); }
    if (yb >= ya) {
        k_ysc_transpose<<<dim3((yb - ya + 32) / 32, (len + 31) / 32), dim3(32, 8), 0, c->st>>>(yb + 1, len, c->P, c->N,
                                                                                         ysc, z, ya);
        c->launches++;
    }
    return true;
}

void launch_lines(Ctx *c, const double *v, double *z)
{
    const int T = c->lines_threads, K = (c->n + T - 1) / T;
    const int nb = (int)c->chunks.size();
    if (nb == 0) return;
    double bytes = 0;   // algorithmic: v + 4 factors read, z written, per owned node of X and Y
    for (const auto &ck : c->chunks) bytes += (double)(ck.last - ck.first + 1) * c->n * 48.0;
    ProfScope ps(c, 2, bytes);
    if (launch_lines_tma(c, v, z)) return;
    if (K <= 1) k_lines<1><<<nb, T, 0, c->st>>>(c->chX, c->chY, c->d_chunks, v, z);
    else if (K <= 2) k_lines<2><<<nb, T, 0, c->st>>>(c->chX, c->chY, c->d_chunks, v, z);
    else if (K <= 4) k_lines<4><<<nb, T, 0, c->st>>>(c->chX, c->chY, c->d_chunks, v, z);
    else if (K <= 8) k_lines<8><<<nb, T, 0, c->st>>>(c->chX, c->chY, c->d_chunks, v, z);
    else k_lines<16><<<nb, T, 0, c->st>>>(c->chX, c->chY, c->d_chunks, v, z);
    c->launches++;
}

}  // namespace spp
