// k_core.cu -- setup, stencil, Krylov-vector and multigrid-transfer kernels (sm_100a, fp64).
//
// All grid functions use the padded layout of spp_internal.cuh.  Reductions are
// deterministic: producers run on a fixed grid of kRedBlocks blocks and write one partial per
// block; consumers re-sum the partials in a fixed order (every block redundantly), so no
// atomics and bit-identical results run to run.
#include "kernels.cuh"

namespace spp {

// ===================================================================================== setup
// 1D coefficients of the 5-point stencil in difference form (R12):
// aW_i = eps/(hbar_i h_i), aS_j = eps/(kbar_j k_j).  wx[i], wy[j] = h_i, k_j (i = 1..N): the
// piecewise-uniform formula on a Shishkin mesh, coordinate differences on a graded one (R21).
__global__ void k_coef_1d(int N, double eps, const double *wx, const double *wy, double *aW, double *aS)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= N; i += gridDim.x * blockDim.x) {
        if (i < 1 || i > N - 1) { aW[i] = 0.0; aS[i] = 0.0; continue; }
        const double h = wx[i], h1 = wx[i + 1], hb = 0.5 * (h + h1);
        const double k = wy[i], k1 = wy[i + 1], kb = 0.5 * (k + k1);
        aW[i] = eps / (hb * h);
        aS[i] = eps / (kb * k);
    }
}

// aE, aN, r, the sweep coefficients aE/D, aN/D, 1/D and the y-form couplings aE/D_E, aN/D_N on
// the padded global grid, with the input validation fused in (c1 > 0, c2 > 0, r >= 0, finite;
// P:208-212).  c1, c2, r are compact ((N-1)^2, x fastest).  D_E and D_N (the diagonal
// at the East / North neighbour) are recomputed from the neighbour's samples with the same
// arithmetic; beyond the last interior node they are absent (the coupling is 0).
__device__ __forceinline__ void coef_at(int i, int j, double eps, const double *wx, const double *wy,
                                        double c1, double c2, double r, const double *aW,
                                        const double *aS, double &e, double &no, double &D)
{
    const double h = wx[i], h1 = wx[i + 1], hb = 0.5 * (h + h1);
    const double k = wy[j], k1 = wy[j + 1], kb = 0.5 * (k + k1);
    e = eps / (hb * h1) + c1 / h1;
    no = eps / (kb * k1) + c2 / k1;
    D = ((aW[i] + e) + (aS[j] + no)) + r;
}

__global__ void __launch_bounds__(256, 6) k_coef_2d(int N, long P, double eps, const double *wx, const double *wy,
                          const double *c1, const double *c2, const double *r, const double *aW,
                          const double *aS, double *aE, double *aN, double *rr, double *ca,
                          double *cn, double *cd, double *ya, double *yn, int want_y, int *bad)
{
    const int m = N - 1;
    const long tot = (long)m * m;
    int fl = 0;                                        // the flags below, OR-ed over this thread's nodes
    for (GridWalk gw(tot, m, 1); gw.ok(); gw.next()) {
        const long p = gw.p; const int j = gw.j, i = gw.i;
        const double a = c1[p], b = c2[p], rv = r[p];
        // bit 0: invalid (c1 > 0, c2 >= 0, r >= 0, finite: P:208-212); bit 1: some c2 > 0;
        // bit 2: some c2 = 0 (c2 = 0 everywhere is the parabolic-layer variant)
        if (!(a > 0.0) || !(b >= 0.0) || !(rv >= 0.0) || !isfinite(a) || !isfinite(b) || !isfinite(rv)) fl |= 1;
        fl |= b > 0.0 ? 2 : 4;
        double e, no, D;
        coef_at(i, j, eps, wx, wy, a, b, rv, aW, aS, e, no, D);
        const long g = (long)j * P + i;
        aE[g] = e; aN[g] = no; rr[g] = rv;
        ca[g] = e / D; cn[g] = no / D; cd[g] = 1.0 / D;
        // the y-form couplings (unweighted M_II, SPP_MG_YFORM) only when the mode uses them;
        // otherwise ensure_y0 forms them on demand (the Jacobi-mode solve never does)
        if (!want_y) continue;
        double cdE = 0.0, cdN = 0.0, t0, t1, DD;
        if (i < m) { coef_at(i + 1, j, eps, wx, wy, c1[p + 1], c2[p + 1], r[p + 1], aW, aS, t0, t1, DD); cdE = 1.0 / DD; }
        if (j < m) { coef_at(i, j + 1, eps, wx, wy, c1[p + m], c2[p + m], r[p + m], aW, aS, t0, t1, DD); cdN = 1.0 / DD; }
        ya[g] = e * cdE; yn[g] = no * cdN;
    }
    // one atomic per warp (an atomic per node on one address serialised in L2: 885 vs ~370 us at 4096^2)
    fl = __reduce_or_sync(0xffffffffu, fl);
    if ((threadIdx.x & 31) == 0 && fl) atomicOr(bad, fl);
}

// Corner multigrid level l >= 1 (R8): re-discretisation on the 1D mesh
// that keeps every 2^l-th corner node plus x_0 and x_{n+1}; coefficients sampled at the coarse
// nodes.  lwx[q], lwy[q] (q = 1..nl+1) = that mesh's widths: 2^l tau/(N/2) inside and
// (1-tau)/(N/2) for the last interval on a Shishkin mesh, coordinate differences on a graded one.
__global__ void k_coef_level(int N, int nl, int step, long Pl, double eps, const double *lwx, const double *lwy,
                             const double *c1, const double *c2,
                             const double *r, double *aW, double *aS, double *hb, double *kb,
                             double *aE, double *aN, double *rr, double *ca, double *cn, double *cd)
{
    const int m = N - 1;
    const long tot = (long)nl * nl;
    for (GridWalk gw(tot, nl, 1); gw.ok(); gw.next()) {
        const int lq = gw.j, q = gw.i;
        const double h = lwx[q], h1 = lwx[q + 1], hbar = 0.5 * (h + h1);
        const double k = lwy[lq], k1 = lwy[lq + 1], kbar = 0.5 * (k + k1);
        const double aw = eps / (hbar * h), as = eps / (kbar * k);
        if (lq == 1) { aW[q] = aw; hb[q] = hbar; }
        if (q == 1) { aS[lq] = as; kb[lq] = kbar; }
        const long g = (long)(lq * step - 1) * m + (q * step - 1);
        const double e = eps / (hbar * h1) + c1[g] / h1;
        const double no = eps / (kbar * k1) + c2[g] / k1;
        const double rv = r[g];
        const double D = ((aw + e) + (as + no)) + rv;
        const long o = (long)lq * Pl + q;
        aE[o] = e; aN[o] = no; rr[o] = rv;
        ca[o] = e / D; cn[o] = no / D; cd[o] = 1.0 / D;
    }
}

// Level 0 1D arrays (the level-0 operator is A_CC itself; its coefficients are the global
// ones): copies of aW, aS on 1..n and hbar, kbar for the FE scaling S_0.
__global__ void k_level0_1d(int N, const double *wx, const double *wy, const double *aW,
                            const double *aS, double *lW, double *lS, double *hb, double *kb)
{
    const int n = N / 2;
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q <= n + 1; q += gridDim.x * blockDim.x) {
        if (q < 1 || q > n) { lW[q] = 0.0; lS[q] = 0.0; hb[q] = 0.0; kb[q] = 0.0; continue; }
        lW[q] = aW[q]; lS[q] = aS[q];
        hb[q] = 0.5 * (wx[q] + wx[q + 1]); kb[q] = 0.5 * (wy[q] + wy[q + 1]);
    }
}

// ===================================================================================== layout
// rows j0 .. j0+nrows-1 of the grid; the compact side holds exactly those rows (row j0 first)
__global__ void k_pack(int m, long P, const double *src, double *dst, int j0, int nrows)   // compact -> padded
{
    const long tot = (long)m * nrows;
    for (GridWalk gw(tot, m, j0); gw.ok(); gw.next()) {
        const long p = gw.p; const int j = gw.j, i = gw.i;
        dst[(long)j * P + i] = src[p];
    }
}
__global__ void k_unpack(int m, long P, const double *src, double *dst, int j0, int nrows)  // padded -> compact
{
    const long tot = (long)m * nrows;
    for (GridWalk gw(tot, m, j0); gw.ok(); gw.next()) {
        const long p = gw.p; const int j = gw.j, i = gw.i;
        dst[p] = src[(long)j * P + i];
    }
}

// ===================================================================================== reductions
__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

// block-wide sum; result valid in thread 0
__device__ __forceinline__ double block_sum(double v, double *sm)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sm[w] = v;
    __syncthreads();
    if (w == 0) {
        v = lane < nw ? sm[lane] : 0.0;
        v = warp_sum(v);
    }
    return v;
}

// every block re-sums the nparts * kRedBlocks partials (one kRedBlocks segment per row strip of a
// distributed solve; nparts = 1 on one GPU) in the same order
__device__ __forceinline__ double sum_partials(const double *part, double *sm, int nparts)
{
    __shared__ double s_res;
    if (threadIdx.x < 32) {
        double v = 0.0;
        for (int b = threadIdx.x; b < nparts * kRedBlocks; b += 32) v += part[b];
        v = warp_sum(v);
        if (threadIdx.x == 0) s_res = v;
    }
    __syncthreads();
    (void)sm;
    return s_res;
}

// ===================================================================================== stencil
// w = A z (difference form; R12); weighted: w = (A z)/D.
// Fused: partial of <w, v0> (first MGS dot) when v0 != nullptr.
// rows j0 .. j0+nrows-1 (a row strip: DESIGN.md §9; j0 = 1, nrows = m on one GPU)
__global__ void __launch_bounds__(kRedThreads) k_spmv(int m, long P, const double *__restrict__ z,
    const double *__restrict__ aE, const double *__restrict__ aN, const double *__restrict__ rr,
    const double *__restrict__ aW, const double *__restrict__ aS, int weighted, double *w,
    const double *__restrict__ v0, double *part, int j0, int nrows)
{
    __shared__ double sm[32];
    double acc = 0.0;
    const long rows = nrows;
    // one block-iteration = one row segment of 2*blockDim columns, double2 stores
    const int segw = 2 * blockDim.x;
    const long nseg = (P + segw - 1) / segw;
    for (long it = blockIdx.x; it < rows * nseg; it += gridDim.x) {
        const int j = (int)(it / nseg) + j0;
        const int i0 = (int)(it % nseg) * segw + 2 * threadIdx.x;
        const long g = (long)j * P + i0;
        if (i0 >= P) continue;
        double out[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int i = i0 + u;
            double val = 0.0;
            if (i >= 1 && i <= m) {
                const long q = g + u;
                const double c = z[q];
                const double e = aE[q], no = aN[q], rv = rr[q], ww = aW[i], ss = aS[j];
                val = ww * (c - z[q - 1]) + e * (c - z[q + 1]) + ss * (c - z[q - P]) + no * (c - z[q + P]) + rv * c;
                if (weighted) val /= ((ww + e) + (ss + no)) + rv;
            }
            out[u] = val;
        }
        *reinterpret_cast<double2 *>(w + g) = make_double2(out[0], out[1]);
        if (v0) {
            const double2 vv = *reinterpret_cast<const double2 *>(v0 + g);
            acc += out[0] * vv.x + out[1] * vv.y;
        }
    }
    if (part) {
        const double s = block_sum(acc, sm);
        if (threadIdx.x == 0) part[blockIdx.x] = s;
        zero_tail(part);
    }
}

// true residual statistics: sums of (f-Au)^2, ((f-Au)/D)^2, f^2, (f/D)^2
__global__ void __launch_bounds__(kRedThreads) k_resid_stats(int m, long P, const double *f,
    const double *Au, const double *aE, const double *aN, const double *rr, const double *aW,
    const double *aS, double *part4, long pstride, int j0, int nrows)
{
    __shared__ double sm[32];
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    const long tot = (long)m * nrows;
    for (GridWalk gw(tot, m, j0); gw.ok(); gw.next()) {
        const int j = gw.j, i = gw.i;
        const long g = (long)j * P + i;
        const double D = ((aW[i] + aE[g]) + (aS[j] + aN[g])) + rr[g];
        const double r = f[g] - Au[g];
        s0 += r * r; s1 += (r / D) * (r / D); s2 += f[g] * f[g]; s3 += (f[g] / D) * (f[g] / D);
    }
    double t;
    t = block_sum(s0, sm); if (threadIdx.x == 0) part4[blockIdx.x] = t;
    t = block_sum(s1, sm); if (threadIdx.x == 0) part4[pstride + blockIdx.x] = t;
    t = block_sum(s2, sm); if (threadIdx.x == 0) part4[2 * pstride + blockIdx.x] = t;
    t = block_sum(s3, sm); if (threadIdx.x == 0) part4[3 * pstride + blockIdx.x] = t;
    for (int a4 = 0; a4 < 4; ++a4) zero_tail(part4 + (size_t)a4 * pstride);
}

// ===================================================================================== Krylov vectors
// out = f / D (weighted) or f, partial ||out||^2; with Au != nullptr the residual f - Au in
// place of f (the restart vector of FGMRES(m), reading R23)
__global__ void __launch_bounds__(kRedThreads) k_rhs(int m, long P, const double *f, const double *aE,
    const double *aN, const double *rr, const double *aW, const double *aS, int weighted, double *out,
    double *part, int j0, int nrows, const double *Au)
{
    __shared__ double sm[32];
    double acc = 0.0;
    const long tot = (long)m * nrows;
    for (GridWalk gw(tot, m, j0); gw.ok(); gw.next()) {
        const int j = gw.j, i = gw.i;
        const long g = (long)j * P + i;
        double v = Au ? f[g] - Au[g] : f[g];
        if (weighted) v /= ((aW[i] + aE[g]) + (aS[j] + aN[g])) + rr[g];
        out[g] = v;
        acc += v * v;
    }
    const double s = block_sum(acc, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
    zero_tail(part);
}

// x *= alpha (alpha from host)
__global__ void k_scale(long n2, double *x, double alpha)
{
    const long n = n2 / 2;
    double2 *x2 = reinterpret_cast<double2 *>(x);
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
        double2 a = x2[p];
        a.x *= alpha; a.y *= alpha;
        x2[p] = a;
    }
}

// MGS step: h = sum(part_in) (stored to hslot by block 0);
// w -= h * x;  part_out = <w, y>  (y == w gives ||w||^2).
__global__ void __launch_bounds__(kRedThreads) k_mgs(long n2, double *w, const double *__restrict__ x,
    const double *part_in, double *hslot, const double *y, double *part_out, int nparts)
{
    __shared__ double sm[32];
    const double h = sum_partials(part_in, sm, nparts);
    if (blockIdx.x == 0 && threadIdx.x == 0) *hslot = h;
    double acc = 0.0;
    const long n = n2 / 2;
    double2 *w2 = reinterpret_cast<double2 *>(w);
    const double2 *x2 = reinterpret_cast<const double2 *>(x);
    const double2 *y2 = reinterpret_cast<const double2 *>(y);
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
        double2 a = w2[p];
        const double2 b = x2[p];
        a.x -= h * b.x; a.y -= h * b.y;
        w2[p] = a;
        if (y == w) acc += a.x * a.x + a.y * a.y;
        else { const double2 c = y2[p]; acc += a.x * c.x + a.y * c.y; }
    }
    const double s = block_sum(acc, sm);
    if (threadIdx.x == 0) part_out[blockIdx.x] = s;
    zero_tail(part_out);
}

// h = sqrt(sum(part_in)) -> hslot;  v = w / h (0 if h == 0)
__global__ void __launch_bounds__(kRedThreads) k_normalize(long n2, const double *w, const double *part_in,
                                                           double *hslot, double *v, int nparts)
{
    __shared__ double sm[32];
    const double h = sqrt(sum_partials(part_in, sm, nparts));
    if (blockIdx.x == 0 && threadIdx.x == 0) *hslot = h;
    const double inv = h > 0.0 ? 1.0 / h : 0.0;
    const long n = n2 / 2;
    const double2 *w2 = reinterpret_cast<const double2 *>(w);
    double2 *v2 = reinterpret_cast<double2 *>(v);
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
        const double2 a = w2[p];
        v2[p] = make_double2(a.x * inv, a.y * inv);
    }
}

// x = sum_j y_j Z_j  ("construction of the solution once converged")
__global__ void k_update_x(long n2, int k, const double *const *Z, const double *y, double *x, int accumulate)
{
    const long n = n2 / 2;
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < n; p += (long)gridDim.x * blockDim.x) {
        // x = sum_j y_j z_j, or x += ... after a restart (the oracle's order: x, then j = 0, 1, ...)
        double2 acc = accumulate ? reinterpret_cast<const double2 *>(x)[p] : make_double2(0.0, 0.0);
        for (int j = 0; j < k; ++j) {
            const double2 a = reinterpret_cast<const double2 *>(Z[j])[p];
            acc.x += y[j] * a.x; acc.y += y[j] * a.y;
        }
        reinterpret_cast<double2 *>(x)[p] = acc;
    }
}

// ===================================================================================== corner MG
// Corner right-hand side (first block row of eq:2D blocks):
//   b_C = s v_C + [j = n] aN z(i, n+1) + [i = n] aE z(n+1, j),   s = D (weighted) or 1,
// written to the level-0 value grid; partial ||S_0 b_C||^2 (S_0 = diag(hbar_i kbar_j)).
__global__ void __launch_bounds__(kRedThreads) k_corner_rhs(int N, long P, long P0, const double *v,
    const double *z, const double *aE, const double *aN, const double *rr, const double *aW,
    const double *aS, const double *hb, const double *kb, int weighted, double *bc, double *part, double *bc2,
    const double *cd, int scale2, int j0, int j1)
{
    __shared__ double sm[32];
    const int n = N / 2;
    double acc = 0.0;
    // corner rows j0 .. j1; one block-iteration = a row segment of 2*blockDim columns from the
    // ghost column 0, a column pair (i0, i0+1) per thread with 16-byte accesses (the pitches are
    // multiples of 16 doubles); the corner's ghost columns 0 and n+1 are written as zeros
    auto ld2 = [](const double *p) { return *reinterpret_cast<const double2 *>(p); };
    const int segw = 2 * blockDim.x;
    const int nseg = (n + 2 + segw - 1) / segw;
    const long nit = (long)(j1 - j0 + 1) * nseg;
    for (long it = blockIdx.x; it < nit; it += gridDim.x) {
        const int j = (int)(it / nseg) + j0;
        const int i0 = (int)(it % nseg) * segw + 2 * threadIdx.x;
        if (i0 > n) continue;
        const long g = (long)j * P + i0;
        const bool ok0 = i0 >= 1, ok1 = i0 + 1 <= n;
        const double2 vv = ld2(v + g), vE = ld2(aE + g), vN = ld2(aN + g);
        double2 s = make_double2(1.0, 1.0);
        if (weighted) {
            const double2 vr = ld2(rr + g), vW = ld2(aW + i0);
            const double vS = aS[j];
            s.x = ((vW.x + vE.x) + (vS + vN.x)) + vr.x;
            s.y = ((vW.y + vE.y) + (vS + vN.y)) + vr.y;
        }
        double b0 = s.x * vv.x, b1 = s.y * vv.y;
        if (j == n) { const double2 zn = ld2(z + g + P); b0 += vN.x * zn.x; b1 += vN.y * zn.y; }
        if (i0 == n) b0 += vE.x * z[g + 1];            // i = n is always the pair's first column (n even)
        b0 = ok0 ? b0 : 0.0;
        b1 = ok1 ? b1 : 0.0;
        const long o = (long)j * P0 + i0;
        *reinterpret_cast<double2 *>(bc + o) = make_double2(b0, b1);
        if (bc2) {
            double2 w = make_double2(b0, b1);
            if (scale2) { const double2 vd = ld2(cd + g); w.x *= vd.x; w.y *= vd.y; }   // b/D in z-form
            *reinterpret_cast<double2 *>(bc2 + o) = w;
        }
        const double2 vh = ld2(hb + i0);
        const double kj = kb[j];
        const double t0 = (vh.x * kj) * b0, t1 = (vh.y * kj) * b1;
        acc += t0 * t0;
        acc += t1 * t1;
    }
    const double s = block_sum(acc, sm);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
    zero_tail(part);
}

// z += e; rho = b - A z (level grid, difference form); partial ||S rho||^2.  If e == nullptr
// only the residual is formed.
__global__ void __launch_bounds__(kRedThreads) k_mg_resid(int nl, long Pv, long Pc, double *z,
    const double *e, const double *b, const double *aE, const double *aN, const double *rr,
    const double *aW, const double *aS, const double *hb, const double *kb, double *rho, double *part)
{
    __shared__ double sm[32];
    double acc = 0.0;
    const long tot = (long)nl * nl;
    for (GridWalk gw(tot, nl, 1); gw.ok(); gw.next()) {
        const int j = gw.j, i = gw.i;
        const long g = (long)j * Pv + i, c = (long)j * Pc + i;
        double zc, zw, ze, zs, zn;
        if (e) {
            zc = z[g] + e[g];
            zw = (i > 1) ? z[g - 1] + e[g - 1] : 0.0;
            ze = (i < nl) ? z[g + 1] + e[g + 1] : 0.0;
            zs = (j > 1) ? z[g - Pv] + e[g - Pv] : 0.0;
            zn = (j < nl) ? z[g + Pv] + e[g + Pv] : 0.0;
        } else {
            zc = z[g]; zw = z[g - 1]; ze = z[g + 1]; zs = z[g - Pv]; zn = z[g + Pv];
        }
        const double Az = aW[i] * (zc - zw) + aE[c] * (zc - ze) + aS[j] * (zc - zs) + aN[c] * (zc - zn) + rr[c] * zc;
        const double r = b[g] - Az;
        rho[g] = r;
        if (part) { const double t = (hb[i] * kb[j]) * r; acc += t * t; }
    }
    if (part) {
        const double s = block_sum(acc, sm);
        if (threadIdx.x == 0) part[blockIdx.x] = s;
        zero_tail(part);
    }
}

// prolongation and correction e += P e_c, geometric weights W (R21)
__global__ void k_prolong_add(int nl, long Pv, double *e, const double *ec, long Pcv, Wts W)
{
    const long tot = (long)nl * nl;
    for (GridWalk gw(tot, nl, 1); gw.ok(); gw.next()) {
        const int j = gw.j, i = gw.i;
        e[(long)j * Pv + i] += W.uni ? interp_w<true>(ec, Pcv, i, j, W) : interp_w<false>(ec, Pcv, i, j, W);
    }
}

// copy the corner iterate into the global preconditioned vector
__global__ void k_corner_out(int n, long P0, const double *zc, long P, double *z, const MGState *ms, int j0, int j1)
{
    if (ms) zc = ms->zcur;                          // corner graph: nullptr when no cycle ran (z = 0)
    const long tot = (long)n * (j1 - j0 + 1);
    for (GridWalk gw(tot, n, j0); gw.ok(); gw.next()) {
        const int j = gw.j, i = gw.i;
        z[(long)j * P + i] = zc ? zc[(long)j * P0 + i] : 0.0;
    }
}

// level grid compact <-> padded (test hooks)
__global__ void k_pack_level(int nl, long Pv, const double *src, double *dst)
{
    const long tot = (long)nl * nl;
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < tot; p += (long)gridDim.x * blockDim.x)
        dst[(long)(p / nl + 1) * Pv + (p % nl + 1)] = src[p];
}
__global__ void k_unpack_level(int nl, long Pv, const double *src, double *dst)
{
    const long tot = (long)nl * nl;
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < tot; p += (long)gridDim.x * blockDim.x)
        dst[p] = src[(long)(p / nl + 1) * Pv + (p % nl + 1)];
}

}  // namespace spp
