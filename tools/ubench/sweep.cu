// cycles per wavefront step of the one-warp coarse GS sweep, variants
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__global__ void k(double *out, long long *t, int n)
{
    extern __shared__ double sm[];
    const int st = n + 2, A = st * st;
    double *b = sm, *e = sm + A, *aE = sm + 2 * A, *aN = sm + 3 * A, *cd = sm + 4 * A, *aW = sm + 5 * A, *aS = aW + st;
    for (int k = threadIdx.x; k < 5 * A + 2 * st; k += blockDim.x) sm[k] = 0.25 + 1e-3 * (k % 7);
    __syncthreads();
    long long t0 = clock64();
    for (int rep = 0; rep < 10; ++rep)
    if (threadIdx.x < 32) {
        const int tt = threadIdx.x;
        const bool act = tt < n;
        const int j = n - tt;
        const double as = act ? aS[j] : 0.0;
        double vlast = 0.0;
        if (V == 0) {
            for (int s = 0; s < 2 * n - 1; ++s) {
                const int i = n - (s - tt);
                double vN = __shfl_up_sync(0xffffffffu, vlast, 1);
                if (tt == 0) vN = 0.0;
                if (act && s >= tt && i >= 1) {
                    const int q = j * st + i;
                    const double v = (((b[q] + aW[i] * e[q - 1]) + as * e[q - st]) + aE[q] * vlast) + aN[q] * vN;
                    vlast = v * cd[q];
                    e[q] = vlast;
                }
            }
        } else if (V == 1) {                       // branch-free: clamped index, select
            for (int s = 0; s < 2 * n - 1; ++s) {
                const int i = n - (s - tt);
                double vN = __shfl_up_sync(0xffffffffu, vlast, 1);
                if (tt == 0) vN = 0.0;
                const bool ok = act && s >= tt && i >= 1;
                const int q = (ok ? j : 1) * st + (ok ? i : 1);
                const double v = (((b[q] + aW[ok ? i : 1] * e[q - 1]) + as * e[q - st]) + aE[q] * vlast) + aN[q] * vN;
                const double w = v * cd[q];
                vlast = ok ? w : vlast;
                if (ok) e[q] = w;
            }
        } else if (V == 3) {                       // branch-free, operands one step ahead
            const int jj = act ? j : 1;
            int i = n + tt;                        // column of step s (valid when 1 <= i <= n and act)
            auto ld = [&](int ii, double &B, double &W, double &S, double &E, double &N, double &C) {
                const int ic = (ii >= 1 && ii <= n) ? ii : 1, q = jj * st + ic;
                B = b[q]; W = aW[ic] * e[q - 1]; S = e[q - st]; E = aE[q]; N = aN[q]; C = cd[q];
            };
            double B, W, S, E, N, C;
            ld(n - (0 - tt), B, W, S, E, N, C);
            for (int s = 0; s < 2 * n - 1; ++s) {
                i = n - (s - tt);
                const bool ok = act && i >= 1 && i <= n;
                double Bn, Wn, Sn, En, Nn, Cn;
                ld(i - 1, Bn, Wn, Sn, En, Nn, Cn);
                double vN = __shfl_up_sync(0xffffffffu, vlast, 1);
                if (tt == 0) vN = 0.0;
                const double v = (((B + W) + as * S) + E * vlast) + N * vN;
                const double w = v * C;
                vlast = ok ? w : vlast;
                if (ok) e[jj * st + i] = w;
                B = Bn; W = Wn; S = Sn; E = En; N = Nn; C = Cn;
            }
        } else {                                   // no shared memory in the loop (registers only)
            double x = 0.5;
            for (int s = 0; s < 2 * n - 1; ++s) {
                double vN = __shfl_up_sync(0xffffffffu, vlast, 1);
                if (tt == 0) vN = 0.0;
                const double v = (((x + 0.25 * x) + as * x) + 0.25 * vlast) + 0.25 * vN;
                vlast = v * 0.5;
            }
            e[tt] = vlast;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) t[V] = t1 - t0;
    out[threadIdx.x] = e[threadIdx.x];
}
int main()
{
    double *o; long long *t, h[4];
    cudaMalloc(&o, 256 * 8); cudaMalloc(&t, 64);
    for (int n : {16, 32}) {
        const size_t sm = (5 * (n + 2) * (n + 2) + 2 * (n + 2)) * 8;
        for (int r = 0; r < 2; ++r) { k<0><<<1, 256, sm>>>(o, t, n); k<1><<<1, 256, sm>>>(o, t, n); k<2><<<1, 256, sm>>>(o, t, n); k<3><<<1, 256, sm>>>(o, t, n); }
        cudaError_t e = cudaDeviceSynchronize(); if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, t, 32, cudaMemcpyDeviceToHost);
        for (int v = 0; v < 4; ++v) printf("n=%d variant %d: %.1f cycles/step\n", n, v, h[v] / (10.0 * (2 * n - 1)));
    }
    return 0;
}
