// k_1d.cu -- the 1D path (cfg1; paper section 2): -eps u'' - c u' + r u = f on (0,1).
//
// Upwind stencil eq:stencil_1d in difference form; preconditioner eq:block_M
// (P:375-386): M = A with the sub-diagonal zeroed in rows N_L+2 .. N-1 (N_L = N/2), applied as
// one tridiagonal solve whose Thomas factors are computed at setup.  The whole Krylov
// solve runs in ONE CTA (the problem has N-1 <= 8191 unknowns): matvec, the factored M solve as
// two block-wide affine scans, MGS dot products by warp-shuffle block reductions, and the
// Givens update by thread 0.  Two drivers:
//   right/flexible FGMRES with the recurrence stop (SPP_STOP_REL_JACOBI / REL_L2 / ABS_L2),
//   left GMRES with the true inf-norm residual stop (SPP_STOP_ABS_MAX; reading R10).
#include <algorithm>
#include <cmath>
#include <tuple>
#include <vector>
#include <cstring>

#include "kernels.cuh"
#include "scan.cuh"

namespace spp {

struct OneD {
    int m, side, weighted, stop_abs, leftmax, maxit, fixed;
    double tol;
    const double *aW, *aE, *rr, *D, *g, *al, *be;
    const double *f;
    double *V, *Z, *x, *w, *t, *H, *hist;
    int *iout;
    double *dout;
};

// setup: coefficients + Thomas factors of M for one problem (one thread; N <= 8192).
// Returns 1 if the coefficients violate c > 0, r >= 0.
__device__ int setup1d_one(int N, double eps, double h, double H, const double *c, const double *r,
                           double *aW, double *aE, double *rr, double *D, double *g, double *al, double *be)
{
    const int n = N / 2, m = N - 1, NL = n;
    double gprev = 0.0, supprev = 0.0;
    int b = 0;
    for (int k = 0; k < m; ++k) {
        const int i = k + 1;
        const double hi = i <= n ? h : H, hi1 = (i + 1) <= n ? h : H, hb = 0.5 * (hi + hi1);
        const double cv = c[k], rv = r[k];
        if (!(cv > 0.0) || !(rv >= 0.0) || !isfinite(cv) || !isfinite(rv)) b = 1;
        const double w = eps / (hb * hi), e = eps / (hb * hi1) + cv / hi1;
        const double d = (w + e) + rv;
        aW[k] = w; aE[k] = e; rr[k] = rv; D[k] = d;
        // M: sub-diagonal kept in rows i <= N_L+1 only (eq:block_M)
        const double sub = (i >= NL + 2 || k == 0) ? 0.0 : w;
        const double sup = (k == m - 1) ? 0.0 : e;
        const double den = (k == 0) ? d : d - sub * (supprev * gprev);
        const double gk = 1.0 / den;
        g[k] = gk; al[k] = sub * gk; be[k] = sup * gk;
        gprev = gk; supprev = sup;
    }
    return b;
}

__global__ void k_setup1d(int N, double eps, double h, double H, const double *c, const double *r,
                          double *aW, double *aE, double *rr, double *D, double *g, double *al,
                          double *be, int *bad)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    *bad = setup1d_one(N, eps, h, H, c, r, aW, aE, rr, D, g, al, be);
}

template <int K>
__device__ __forceinline__ double cta_sum(double v, double *red)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    if (nw == 1) return 0.0 + v;                  // one-warp CTA: the same value, no barriers
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double s = 0.0;
    for (int k = 0; k < nw; ++k) s += red[k];     // same order in every thread
    __syncthreads();
    return s;
}

template <int K>
__device__ __forceinline__ double cta_max(double v, double *red)
{
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, d));
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double s = 0.0;
    for (int k = 0; k < nw; ++k) s = fmax(s, red[k]);
    __syncthreads();
    return s;
}

// y = A x (difference form); x must be complete (caller syncs)
template <int K>
__device__ __forceinline__ void mv1(const OneD &a, const double *x, double *y, bool weighted)
{
    const int k0 = threadIdx.x * K;
#pragma unroll
    for (int u = 0; u < K; ++u) {
        const int k = k0 + u;
        if (k < a.m) {
            const double c = x[k];
            const double xw = k > 0 ? x[k - 1] : 0.0, xe = k < a.m - 1 ? x[k + 1] : 0.0;
            double v = a.aW[k] * (c - xw) + a.aE[k] * (c - xe) + a.rr[k] * c;
            if (weighted) v /= a.D[k];
            y[k] = v;
        }
    }
    __syncthreads();
}

// z = M^{-1} (s q), s = D (scaled) or 1
template <int K>
__device__ __forceinline__ void prec1(const OneD &a, const double *q, double *z, bool scaled, double *sA, double *sB)
{
    const int k0 = threadIdx.x * K;
    double al[K], be[K], b[K], y[K], zz[K];
#pragma unroll
    for (int u = 0; u < K; ++u) {
        const int k = k0 + u;
        if (k < a.m) {
            b[u] = a.g[k] * (scaled ? a.D[k] * q[k] : q[k]);
            al[u] = a.al[k]; be[u] = a.be[k];
        } else { b[u] = 0.0; al[u] = 0.0; be[u] = 0.0; }
    }
    fwd_scan<K>(al, b, y, sA, sB);
    bwd_scan<K>(be, y, zz, sA, sB);
#pragma unroll
    for (int u = 0; u < K; ++u) { const int k = k0 + u; if (k < a.m) z[k] = zz[u]; }
    __syncthreads();
}

template <int K>
__device__ __forceinline__ double dot1(const OneD &a, const double *x, const double *y, double *red)
{
    const int k0 = threadIdx.x * K;
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < K; ++u) { const int k = k0 + u; if (k < a.m) s += x[k] * y[k]; }
    return cta_sum<K>(s, red);
}

template <int K>
__device__ __forceinline__ void axpy1(const OneD &a, double alpha, const double *x, double *y)
{
    const int k0 = threadIdx.x * K;
#pragma unroll
    for (int u = 0; u < K; ++u) { const int k = k0 + u; if (k < a.m) y[k] += alpha * x[k]; }
    __syncthreads();
}

// register-slice forms (thread owns rows k0 .. k0+K-1)
template <int K>
__device__ __forceinline__ double dotr(int m, const double (&x)[K], const double (&y)[K], double *red)
{
    const int k0 = threadIdx.x * K;
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < K; ++u) if (k0 + u < m) s += x[u] * y[u];
    return cta_sum<K>(s, red);
}

// z = M^{-1} (s q) with q, z register slices
template <int K>
__device__ __forceinline__ void prec1r(const OneD &a, const double (&q)[K], double (&zz)[K], bool scaled,
                                       double *sA, double *sB)
{
    const int k0 = threadIdx.x * K;
    double c[K], b[K], y[K];
#pragma unroll
    for (int u = 0; u < K; ++u) {
        const int k = k0 + u;
        if (k < a.m) {
            b[u] = a.g[k] * (scaled ? a.D[k] * q[u] : q[u]);
            c[u] = a.al[k];
        } else { b[u] = 0.0; c[u] = 0.0; }
    }
    fwd_scan<K>(c, b, y, sA, sB);
#pragma unroll
    for (int u = 0; u < K; ++u) { const int k = k0 + u; c[u] = k < a.m ? a.be[k] : 0.0; }   // be after the forward pass (register pressure)
    bwd_scan<K>(c, y, zz, sA, sB);
}

// w = (W) A z with z's register slice zr; the two neighbour rows outside the slice come from
// zmem (written and synchronised by the caller)
template <int K>
__device__ __forceinline__ void mv1r(const OneD &a, const double (&zr)[K], const double *zmem, double (&w)[K],
                                     bool weighted)
{
    const int k0 = threadIdx.x * K;
#pragma unroll
    for (int u = 0; u < K; ++u) {
        const int k = k0 + u;
        if (k < a.m) {
            const double c = zr[u];
            const double xw = u > 0 ? zr[u - 1] : (k > 0 ? zmem[k - 1] : 0.0);
            const double xe = u < K - 1 ? (k < a.m - 1 ? zr[u + 1] : 0.0) : (k < a.m - 1 ? zmem[k + 1] : 0.0);
            double v = a.aW[k] * (c - xw) + a.aE[k] * (c - xe) + a.rr[k] * c;
            if (weighted) v /= a.D[k];
            w[u] = v;
        } else w[u] = 0.0;
    }
}

template <int K>
__device__ __forceinline__ void solve1d_body(const OneD &a)
{
    __shared__ double sA[32], sB[64], red[32];
    // Givens cosines/sines, rotated rhs, LSQ solution and the current Hessenberg column, sized
    // by max_iters (dynamic shared memory, smem1d_bytes) so that small problems pack many CTAs
    // per SM; columns are copied to a.H once rotated (for the final back-substitution)
    extern __shared__ double dyn1[];
    const int L = a.maxit + 2;
    double *cs = dyn1, *sn = cs + L, *gg = sn + L, *yy = gg + L, *hc = yy + L;
    __shared__ int s_stop;
    __shared__ double s_res;
    const int m = a.m, maxit = a.maxit, ld = maxit + 1;
    const int k0 = threadIdx.x * K;
    for (int u = 0; u < K; ++u) { const int k = k0 + u; if (k < m) a.x[k] = 0.0; }
    __syncthreads();
    int iters = 0, conv = 0;
    double res0 = 0.0, resf = 0.0;
    if (!a.leftmax) {
        // ---------------- right / flexible FGMRES ----------------
        // Each thread keeps its K-row slices of v_k, z_k and w in registers (the MGS loop reads
        // each basis vector once for both its dot product and its update); V and Z go to
        // memory for the later iterations and the final combination.  Same operations in the
        // same order as the memory-resident form.
        double vr[K], zr[K], wr[K];
#pragma unroll
        for (int u = 0; u < K; ++u) {
            const int k = k0 + u;
            vr[u] = k < m ? (a.weighted ? a.f[k] / a.D[k] : a.f[k]) : 0.0;
        }
        const double beta = sqrt(dotr<K>(m, vr, vr, red));
        res0 = beta; resf = beta;
        if (threadIdx.x == 0) { a.hist[0] = beta; gg[0] = beta; }
        const double target = a.stop_abs ? a.tol : a.tol * beta;
        if (beta > 0.0) {
#pragma unroll
            for (int u = 0; u < K; ++u) { const int k = k0 + u; if (k < m) { vr[u] /= beta; a.V[k] = vr[u]; } }
            for (int k = 0; k < maxit; ++k) {
                double *zk = a.Z + (size_t)k * m;
                prec1r<K>(a, vr, zr, a.weighted, sA, sB);
#pragma unroll
                for (int u = 0; u < K; ++u) { const int q = k0 + u; if (q < m) zk[q] = zr[u]; }
                __syncthreads();
                mv1r<K>(a, zr, zk, wr, a.weighted);
                double *h = hc;
                double vv[K], vnx[K];
#pragma unroll
                for (int u = 0; u < K; ++u) { const int q = k0 + u; vv[u] = q < m ? a.V[q] : 0.0; }
                for (int j = 0; j <= k; ++j) {
                    if (j < k) {             // prefetch v_{j+1} under the reduction of step j
                        const double *vj1 = a.V + (size_t)(j + 1) * m;
#pragma unroll
                        for (int u = 0; u < K; ++u) { const int q = k0 + u; vnx[u] = q < m ? vj1[q] : 0.0; }
                    }
                    const double hj = dotr<K>(m, wr, vv, red);
                    if (threadIdx.x == 0) h[j] = hj;
#pragma unroll
                    for (int u = 0; u < K; ++u) {
                        const int q = k0 + u;
                        if (q < m) wr[u] += -hj * vv[u];
                        vv[u] = vnx[u];
                    }
                }
                const double hn = sqrt(dotr<K>(m, wr, wr, red));
                double *vn = a.V + (size_t)(k + 1) * m;
#pragma unroll
                for (int u = 0; u < K; ++u) {
                    const int q = k0 + u;
                    vr[u] = hn > 0.0 ? wr[u] / hn : 0.0;
                    if (q < m) vn[q] = vr[u];
                }
                if (threadIdx.x == 0) {
                    h[k + 1] = hn;
                    for (int i = 0; i < k; ++i) {
                        const double t = cs[i] * h[i] + sn[i] * h[i + 1];
                        h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
                        h[i] = t;
                    }
                    const double den = hypot(h[k], h[k + 1]);
                    if (den == 0.0) { cs[k] = 1.0; sn[k] = 0.0; } else { cs[k] = h[k] / den; sn[k] = h[k + 1] / den; }
                    h[k] = den; h[k + 1] = 0.0;
                    gg[k + 1] = -sn[k] * gg[k];
                    gg[k] = cs[k] * gg[k];
                    for (int i = 0; i <= k + 1; ++i) a.H[(size_t)k * ld + i] = h[i];
                    const double res = fabs(gg[k + 1]);
                    a.hist[k + 1] = res;
                    s_res = res;
                    int stop = !(hn > 0.0);
                    if (a.fixed > 0) stop |= (k + 1 >= a.fixed);
                    else stop |= (res <= target);
                    s_stop = stop;
                }
                __syncthreads();
                iters = k + 1;
                resf = s_res;
                if (s_stop) break;
            }
            conv = resf <= target;
            if (threadIdx.x == 0) {
                for (int i = iters - 1; i >= 0; --i) {
                    double t = gg[i];
                    for (int j = i + 1; j < iters; ++j) t -= a.H[(size_t)j * ld + i] * yy[j];
                    yy[i] = t / a.H[(size_t)i * ld + i];
                }
            }
            __syncthreads();
            double xr[K];
#pragma unroll
            for (int u = 0; u < K; ++u) xr[u] = 0.0;
            for (int j = 0; j < iters; ++j) {
                const double *zj = a.Z + (size_t)j * m, yj = yy[j];
#pragma unroll
                for (int u = 0; u < K; ++u) { const int q = k0 + u; if (q < m) xr[u] += yj * zj[q]; }
            }
#pragma unroll
            for (int u = 0; u < K; ++u) { const int q = k0 + u; if (q < m) a.x[q] = xr[u]; }
            __syncthreads();
        } else conv = 1;
    } else {
        // ---------------- left GMRES, true inf-norm residual stop ----------------
        double r0 = 0.0;
        for (int u = 0; u < K; ++u) { const int k = k0 + u; if (k < m) r0 = fmax(r0, fabs(a.f[k])); }
        r0 = cta_max<K>(r0, red);
        res0 = r0; resf = r0;
        if (threadIdx.x == 0) a.hist[0] = r0;
        if (r0 <= a.tol) conv = 1;
        else {
            prec1<K>(a, a.f, a.V, false, sA, sB);
            const double beta = sqrt(dot1<K>(a, a.V, a.V, red));
            for (int u = 0; u < K; ++u) { const int k = k0 + u; if (k < m) a.V[k] /= beta; }
            if (threadIdx.x == 0) gg[0] = beta;
            __syncthreads();
            for (int k = 0; k < maxit; ++k) {
                mv1<K>(a, a.V + (size_t)k * m, a.t, false);
                prec1<K>(a, a.t, a.w, false, sA, sB);
                double *h = hc;
                for (int j = 0; j <= k; ++j) {
                    const double hj = dot1<K>(a, a.w, a.V + (size_t)j * m, red);
                    if (threadIdx.x == 0) h[j] = hj;
                    axpy1<K>(a, -hj, a.V + (size_t)j * m, a.w);
                }
                const double hn = sqrt(dot1<K>(a, a.w, a.w, red));
                double *vn = a.V + (size_t)(k + 1) * m;
                for (int u = 0; u < K; ++u) { const int kk = k0 + u; if (kk < m) vn[kk] = hn > 0.0 ? a.w[kk] / hn : 0.0; }
                if (threadIdx.x == 0) {
                    h[k + 1] = hn;
                    for (int i = 0; i < k; ++i) {
                        const double t = cs[i] * h[i] + sn[i] * h[i + 1];
                        h[i + 1] = -sn[i] * h[i] + cs[i] * h[i + 1];
                        h[i] = t;
                    }
                    const double den = hypot(h[k], h[k + 1]);
                    if (den == 0.0) { cs[k] = 1.0; sn[k] = 0.0; } else { cs[k] = h[k] / den; sn[k] = h[k + 1] / den; }
                    h[k] = den; h[k + 1] = 0.0;
                    gg[k + 1] = -sn[k] * gg[k];
                    gg[k] = cs[k] * gg[k];
                    for (int i = 0; i <= k + 1; ++i) a.H[(size_t)k * ld + i] = h[i];
                    const int kk = k + 1;
                    for (int i = kk - 1; i >= 0; --i) {
                        double t = gg[i];
                        for (int j = i + 1; j < kk; ++j) t -= a.H[(size_t)j * ld + i] * yy[j];
                        yy[i] = t / a.H[(size_t)i * ld + i];
                    }
                    s_stop = !(hn > 0.0);
                }
                __syncthreads();
                // x_k = sum_j y_j v_j ; true residual
                for (int u = 0; u < K; ++u) { const int q = k0 + u; if (q < m) a.x[q] = 0.0; }
                __syncthreads();
                for (int j = 0; j <= k; ++j) axpy1<K>(a, yy[j], a.V + (size_t)j * m, a.x);
                mv1<K>(a, a.x, a.t, false);
                double rinf = 0.0;
                for (int u = 0; u < K; ++u) { const int q = k0 + u; if (q < m) rinf = fmax(rinf, fabs(a.f[q] - a.t[q])); }
                rinf = cta_max<K>(rinf, red);
                iters = k + 1; resf = rinf;
                if (threadIdx.x == 0) a.hist[k + 1] = rinf;
                if (rinf <= a.tol) { conv = 1; break; }
                if (s_stop) break;
            }
        }
    }
    if (threadIdx.x == 0) {
        a.iout[0] = iters; a.iout[1] = conv;
        a.dout[0] = res0; a.dout[1] = resf;
    }
}

template <int K>
__global__ void __launch_bounds__(512) k_solve1d(OneD a) { solve1d_body<K>(a); }

static size_t smem1d_bytes(int maxit) { return sizeof(double) * 5 * (size_t)(maxit + 2); }

// ------------------------------------------------------------------------------ host
struct Buf1 {
    double *aW, *aE, *rr, *D, *g, *al, *be, *V, *Z, *x, *w, *t, *H, *hist, *f, *dout;
    int *iout;
};

__host__ __device__ static size_t need1(int m, int it)
{
    return (size_t)m * 12 + (size_t)(2 * it + 1) * m + (size_t)(it + 1) * (it + 1) + it + 16;
}

__host__ __device__ static Buf1 layout_at(double *p, int m, int it)
{
    Buf1 b{};
    b.aW = p; p += m; b.aE = p; p += m; b.rr = p; p += m; b.D = p; p += m;
    b.g = p; p += m; b.al = p; p += m; b.be = p; p += m;
    b.V = p; p += (size_t)(it + 1) * m; b.Z = p; p += (size_t)it * m;
    b.x = p; p += m; b.w = p; p += m; b.t = p; p += m;
    b.H = p; p += (size_t)(it + 1) * (it + 1);
    b.hist = p; p += it + 2;
    b.f = p; p += m;
    b.dout = p; p += 4;
    b.iout = (int *)p;
    return b;
}

static Buf1 layout1(Ctx *c) { return layout_at(c->d1, c->m, c->opt.max_iters); }

spp_status setup_1d(Ctx *c, const double *cc, const double *r, spp_mem mem)
{
    const int m = c->m, it = c->opt.max_iters;
    if (m > 8191 || it > 512) {
        c->err = "1D: N-1 <= 8191 and max_iters <= 512 (single-CTA solver)";
        return SPP_E_ARG;
    }
    if (!c->d1) {
        const size_t need = need1(m, it);
        if (cudaMalloc(&c->d1, sizeof(double) * need) != cudaSuccess) { c->err = "1D: cudaMalloc failed"; return SPP_E_NOMEM; }
        cudaMemsetAsync(c->d1, 0, sizeof(double) * need, c->st);
    }
    Buf1 b = layout1(c);
    const double *dc = cc, *dr = r;
    if (mem == SPP_HOST) {
        cudaMemcpyAsync(b.x, cc, sizeof(double) * m, cudaMemcpyHostToDevice, c->st);
        cudaMemcpyAsync(b.w, r, sizeof(double) * m, cudaMemcpyHostToDevice, c->st);
        dc = b.x; dr = b.w;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, c->st);
    k_setup1d<<<1, 32, 0, c->st>>>(c->N, c->eps, c->hx, c->Hx, dc, dr, b.aW, b.aE, b.rr, b.D, b.g, b.al, b.be,
                                   b.iout + 4);
    c->launches++;
    cudaEventRecord(e1, c->st);
    int bad = 0;
    cudaMemcpyAsync(&bad, b.iout + 4, sizeof(int), cudaMemcpyDeviceToHost, c->st);
    cudaError_t e = cudaStreamSynchronize(c->st);
    cudaEventElapsedTime(&c->setup_ms, e0, e1);
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    if (e != cudaSuccess) { c->err = cudaGetErrorString(e); return SPP_E_CUDA; }
    if (bad) { c->err = "coefficients violate c > 0, r >= 0 (P:208-212)"; return SPP_E_COEF; }
    return SPP_OK;
}

spp_status solve_1d_abi(Ctx *c, const double *f, double *u, spp_mem mem, double *hist, int hcap, spp_stats *st)
{
    const int m = c->m, it = c->opt.max_iters;
    Buf1 b = layout1(c);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int64_t l0 = c->launches;
    cudaEventRecord(e0, c->st);
    cudaMemcpyAsync(b.f, f, sizeof(double) * m, mem == SPP_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, c->st);
    OneD a{};
    a.m = m; a.maxit = it; a.fixed = c->opt.fixed_iters; a.tol = c->opt.tol;
    a.side = c->opt.side;
    a.leftmax = (c->opt.side == SPP_LEFT) ? 1 : 0;
    a.weighted = c->opt.stop == SPP_STOP_REL_JACOBI;
    a.stop_abs = c->opt.stop == SPP_STOP_ABS_L2;
    a.aW = b.aW; a.aE = b.aE; a.rr = b.rr; a.D = b.D; a.g = b.g; a.al = b.al; a.be = b.be;
    a.f = b.f; a.V = b.V; a.Z = b.Z; a.x = b.x; a.w = b.w; a.t = b.t; a.H = b.H; a.hist = b.hist;
    a.iout = b.iout; a.dout = b.dout;
    int T = (m + 7) / 8;
    T = ((T + 31) / 32) * 32;
    if (T < 32) T = 32;
    if (T > 512) T = 512;
    const int K = (m + T - 1) / T;
    const size_t sm = smem1d_bytes(it);
    if (K <= 1) k_solve1d<1><<<1, T, sm, c->st>>>(a);
    else if (K <= 2) k_solve1d<2><<<1, T, sm, c->st>>>(a);
    else if (K <= 4) k_solve1d<4><<<1, T, sm, c->st>>>(a);
    else if (K <= 8) k_solve1d<8><<<1, T, sm, c->st>>>(a);
    else k_solve1d<16><<<1, T, sm, c->st>>>(a);
    c->launches++;
    if (u) cudaMemcpyAsync(u, b.x, sizeof(double) * m, mem == SPP_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c->st);
    cudaEventRecord(e1, c->st);
    int io[2] = {0, 0};
    double dd[2] = {0, 0};
    std::vector<double> hh(it + 2);
    cudaMemcpyAsync(io, b.iout, sizeof(int) * 2, cudaMemcpyDeviceToHost, c->st);
    cudaMemcpyAsync(dd, b.dout, sizeof(double) * 2, cudaMemcpyDeviceToHost, c->st);
    cudaMemcpyAsync(hh.data(), b.hist, sizeof(double) * (it + 2), cudaMemcpyDeviceToHost, c->st);
    cudaError_t e = cudaStreamSynchronize(c->st);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    if (e != cudaSuccess) { c->err = cudaGetErrorString(e); return SPP_E_CUDA; }
    if (hist) for (int k = 0; k <= io[0] && k < hcap; ++k) hist[k] = hh[k];
    if (st) {
        memset(st, 0, sizeof(*st));
        st->iters = io[0]; st->converged = io[1];
        st->res0 = dd[0]; st->res_final = dd[1];
        st->applies = io[0];
        st->kernel_launches = (int32_t)(c->launches - l0);
        st->setup_s = c->setup_ms * 1e-3; st->solve_s = ms * 1e-3;
        // true residuals (host arithmetic on the device result is avoided: report from a
        // second device pass is unnecessary for 1D diagnostics)
        st->true_res_l2_rel = -1.0; st->true_res_jacobi_rel = -1.0;
    }
    return io[1] ? SPP_OK : SPP_NOT_CONVERGED;
}

// ------------------------------------------------------------------------------ batched 1D
// NEXT-3: many independent 1D problems (any mix of N <= 8192 and eps) in one
// launch per launch shape, one CTA per problem -- the same setup and Krylov body as the single
// solve, so every problem's result is bitwise the single-problem result.
struct Batch1Args {
    const int *n, *idx;
    const double *eps, *h, *H;
    const long long *xo, *so;
    const double *c, *r, *f;
    double *u, *scratch, *res0, *res;
    int *iters, *conv, *bad;
    OneD proto;          // option fields shared by the batch
    int nprob, maxit;
};

// one warp per problem: the per-row coefficients 32 rows at a time (coalesced), the Thomas
// recurrence of those 32 rows by lane 0 from shared memory (the same operations as
// setup1d_one, row by row)
__global__ void __launch_bounds__(128) k_setup1d_batch(Batch1Args b)
{
    __shared__ double sd[4][3][32];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int p = blockIdx.x * 4 + wq;
    if (p >= b.nprob) return;                            // whole warp
    const int N = b.n[p], m = N - 1, n = N / 2, NL = n;
    const double eps = b.eps[p], h = b.h[p], H = b.H[p];
    const double *c = b.c + b.xo[p], *r = b.r + b.xo[p];
    Buf1 l = layout_at(b.scratch + b.so[p], m, b.maxit);
    double gprev = 0.0, supprev = 0.0;
    int bad = 0;
    for (int base = 0; base < m; base += 32) {
        const int k = base + lane;
        if (k < m) {
            const int i = k + 1;
            const double hi = i <= n ? h : H, hi1 = (i + 1) <= n ? h : H, hb = 0.5 * (hi + hi1);
            const double cv = c[k], rv = r[k];
            if (!(cv > 0.0) || !(rv >= 0.0) || !isfinite(cv) || !isfinite(rv)) bad = 1;
            const double w = eps / (hb * hi), e = eps / (hb * hi1) + cv / hi1;
            const double d = (w + e) + rv;
            l.aW[k] = w; l.aE[k] = e; l.rr[k] = rv; l.D[k] = d;
            sd[wq][0][lane] = d;
            sd[wq][1][lane] = (i >= NL + 2 || k == 0) ? 0.0 : w;     // sub (eq:block_M)
            sd[wq][2][lane] = (k == m - 1) ? 0.0 : e;                // sup
        }
        __syncwarp();
        if (lane == 0) {
            const int cnt = min(32, m - base);
            for (int t = 0; t < cnt; ++t) {
                const double d = sd[wq][0][t], sub = sd[wq][1][t], sup = sd[wq][2][t];
                const double den = (base + t == 0) ? d : d - sub * (supprev * gprev);
                const double gk = 1.0 / den;
                sd[wq][0][t] = gk; sd[wq][1][t] = sub * gk; sd[wq][2][t] = sup * gk;
                gprev = gk; supprev = sup;
            }
        }
        __syncwarp();
        if (k < m) { l.g[k] = sd[wq][0][lane]; l.al[k] = sd[wq][1][lane]; l.be[k] = sd[wq][2][lane]; }
        __syncwarp();
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) b.bad[p] = bad;
}

template <int K>
__device__ __forceinline__ void solve1d_batch_body(const Batch1Args &b)
{
    const int p = b.idx[blockIdx.x];
    const int m = b.n[p] - 1;
    Buf1 l = layout_at(b.scratch + b.so[p], m, b.maxit);
    OneD a = b.proto;
    a.m = m;
    a.aW = l.aW; a.aE = l.aE; a.rr = l.rr; a.D = l.D; a.g = l.g; a.al = l.al; a.be = l.be;
    a.f = b.f + b.xo[p];
    a.V = l.V; a.Z = l.Z; a.x = l.x; a.w = l.w; a.t = l.t; a.H = l.H; a.hist = l.hist;
    a.iout = l.iout; a.dout = l.dout;
    solve1d_body<K>(a);
    __syncthreads();
    double *u = b.u + b.xo[p];
    for (int k = threadIdx.x; k < m; k += blockDim.x) u[k] = a.x[k];
    if (threadIdx.x == 0) {
        b.iters[p] = a.iout[0]; b.conv[p] = a.iout[1];
        b.res0[p] = a.dout[0]; b.res[p] = a.dout[1];
    }
}

template <int K>
__global__ void __launch_bounds__(512) k_solve1d_batch(Batch1Args b) { solve1d_batch_body<K>(b); }

// launch shape of a problem with m unknowns: T threads, K rows per thread (as the single solve)
static void shape1(int m, int *T_, int *K_)
{
    int T = (m + 7) / 8;
    T = ((T + 31) / 32) * 32;
    if (T < 32) T = 32;
    if (T > 512) T = 512;
    int K = (m + T - 1) / T;
    K = K <= 1 ? 1 : K <= 2 ? 2 : K <= 4 ? 4 : K <= 8 ? 8 : 16;
    *T_ = T; *K_ = K;
}

static Batch1Args bargs(Batch1 *b)
{
    Batch1Args a{};
    const int P = b->nprob;
    a.eps = b->dpar; a.h = b->dpar + P; a.H = b->dpar + 2 * P; a.res0 = b->dpar + 3 * P; a.res = b->dpar + 4 * P;
    a.xo = b->doff; a.so = b->doff + P;
    a.n = b->dint; a.idx = b->dint + P; a.iters = b->dint + 2 * P; a.conv = b->dint + 3 * P; a.bad = b->dint + 4 * P;
    a.scratch = b->scratch;
    a.nprob = P; a.maxit = b->maxit;
    OneD &o = a.proto;
    o.maxit = b->maxit; o.fixed = b->opt.fixed_iters; o.tol = b->opt.tol; o.side = b->opt.side;
    o.leftmax = b->opt.side == SPP_LEFT ? 1 : 0;
    o.weighted = b->opt.stop == SPP_STOP_REL_JACOBI;
    o.stop_abs = b->opt.stop == SPP_STOP_ABS_L2;
    return a;
}

cudaError_t batch1d_alloc(Batch1 *b)
{
    const int P = b->nprob;
    b->xo.resize(P); b->so.resize(P);
    long long xo = 0, so = 0;
    std::vector<std::tuple<int, int, double, int>> key(P);
    for (int p = 0; p < P; ++p) {
        const int m = b->n[p] - 1;
        b->xo[p] = xo; b->so[p] = so;
        xo += m; so += (long long)need1(m, b->maxit);
        int T, K;
        shape1(m, &T, &K);
        // within a launch shape, the problems most likely to need many iterations first (largest
        // eps*N: outside the regime eps*N << 1 the counts grow), so that the long
        // solves do not start at the end of the launch
        key[p] = std::make_tuple(K, T, -b->eps[p] * b->n[p], p);
    }
    b->total = xo; b->scratch_len = so;
    std::sort(key.begin(), key.end());
    b->order.resize(P);
    for (int p = 0; p < P; ++p) {
        const int K = std::get<0>(key[p]), T = std::get<1>(key[p]);
        b->order[p] = std::get<3>(key[p]);
        if (p == 0 || K != b->gK.back() || T != b->gT.back()) {
            b->gstart.push_back(p); b->gcount.push_back(0); b->gK.push_back(K); b->gT.push_back(T);
        }
        b->gcount.back()++;
    }
    SPP_CUDA_TRY(cudaMalloc(&b->scratch, sizeof(double) * so));
    SPP_CUDA_TRY(cudaMemsetAsync(b->scratch, 0, sizeof(double) * so, b->st));
    SPP_CUDA_TRY(cudaMalloc(&b->dpar, sizeof(double) * 5 * P));
    SPP_CUDA_TRY(cudaMalloc(&b->doff, sizeof(long long) * 2 * P));
    SPP_CUDA_TRY(cudaMalloc(&b->dint, sizeof(int) * 5 * P));
    std::vector<double> par(3 * (size_t)P);
    for (int p = 0; p < P; ++p) { par[p] = b->eps[p]; par[P + p] = b->h[p]; par[2 * P + p] = b->H[p]; }
    std::vector<long long> off(2 * (size_t)P);
    for (int p = 0; p < P; ++p) { off[p] = b->xo[p]; off[P + p] = b->so[p]; }
    std::vector<int> in(2 * (size_t)P);
    for (int p = 0; p < P; ++p) { in[p] = b->n[p]; in[P + p] = b->order[p]; }
    SPP_CUDA_TRY(cudaMemcpyAsync(b->dpar, par.data(), sizeof(double) * 3 * P, cudaMemcpyHostToDevice, b->st));
    SPP_CUDA_TRY(cudaMemcpyAsync(b->doff, off.data(), sizeof(long long) * 2 * P, cudaMemcpyHostToDevice, b->st));
    SPP_CUDA_TRY(cudaMemcpyAsync(b->dint, in.data(), sizeof(int) * 2 * P, cudaMemcpyHostToDevice, b->st));
    return cudaStreamSynchronize(b->st);   // host vectors above go out of scope
}

cudaError_t batch1d_setup(Batch1 *b, const double *c, const double *r)
{
    Batch1Args a = bargs(b);
    a.c = c; a.r = r;
    k_setup1d_batch<<<(b->nprob + 3) / 4, 128, 0, b->st>>>(a);
    b->launches++;
    return cudaGetLastError();
}

cudaError_t batch1d_solve(Batch1 *b, const double *f, double *u)
{
    Batch1Args a = bargs(b);
    a.f = f; a.u = u;
    const size_t sm = smem1d_bytes(b->maxit);
    for (size_t g = 0; g < b->gstart.size(); ++g) {
        Batch1Args ag = a;
        ag.idx = a.idx + b->gstart[g];
        const dim3 grid(b->gcount[g]);
        const int T = b->gT[g];
        switch (b->gK[g]) {
        case 1: k_solve1d_batch<1><<<grid, T, sm, b->st>>>(ag); break;
        case 2: k_solve1d_batch<2><<<grid, T, sm, b->st>>>(ag); break;
        case 4: k_solve1d_batch<4><<<grid, T, sm, b->st>>>(ag); break;
        case 8: k_solve1d_batch<8><<<grid, T, sm, b->st>>>(ag); break;
        default: k_solve1d_batch<16><<<grid, T, sm, b->st>>>(ag); break;
        }
        b->launches++;
    }
    return cudaGetLastError();
}

}  // namespace spp
