// Microbenchmark: dependent-chain latencies of DFMA, 64-bit SHFL, LDS.64, STS+LDS round trip on B200.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, int n, double a, double b)
{
    __shared__ double sm[1024];
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, a, b);                       // DFMA chain
    long long t1 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_up_sync(0xffffffffu, x, 1) + 1e-9;   // SHFL64 + DADD chain
    long long t2 = clock64();
    sm[threadIdx.x] = x;
    __syncwarp();
    int idx = threadIdx.x;
    for (int i = 0; i < n; ++i) { x = sm[idx] + 1.0; idx = ((int)x) & 31; }   // LDS + DADD + F2I chain
    long long t3 = clock64();
    for (int i = 0; i < n; ++i) x = x * a;                              // DMUL chain
    long long t4 = clock64();
    for (int i = 0; i < n; ++i) { float f = (float)x; x = (double)(f * 1.0001f); }  // conversions
    long long t5 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
__global__ void kthr(double *out, long long *cyc, int n, double a, double b)
{   // DFMA throughput: 8 independent chains per thread
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (threadIdx.x == 0) cyc[5] = t1 - t0;
}
int main()
{
    double *o; long long *c, h[8];
    cudaMalloc(&o, 8192); cudaMalloc(&c, 64);
    const int n = 10000;
    k<<<1, 32>>>(o, c, n, 0.999999, 1e-7);
    kthr<<<1, 32>>>(o, c, n, 0.999999, 1e-7);
    cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
    printf("cycles per dependent op (1 warp): DFMA %.1f  SHFL64+DADD %.1f  LDS+DADD+F2I %.1f  DMUL %.1f  F2F pair+FMUL %.1f\n",
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n, h[3] / (double)n, h[4] / (double)n);
    printf("DFMA issue, 8 independent chains (1 warp): %.2f cycles per DFMA\n", h[5] / (8.0 * n));
    for (int wps = 1; wps <= 32; wps *= 2) {
        kthr<<<1, 32 * wps>>>(o, c, n, 0.999999, 1e-7);
        cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
        printf("  %2d warps/SM: %.2f cycles per 8 DFMA per warp -> %.2f warp-DFMA/cycle/SM\n", wps, h[5] / (double)n, 8.0 * n * wps / h[5]);
    }
    return 0;
}
