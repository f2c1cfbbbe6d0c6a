// dependent-chain latencies of the ops on the GS step chain (one warp, clock64)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *t, double a, double b, int iters)
{
    __shared__ double sm[64];
    if (threadIdx.x < 64) sm[threadIdx.x] = threadIdx.x;
    __syncwarp();
    double x = a + threadIdx.x;
    long long t0, t1;
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); x = fma(x, a, b); }
    t1 = clock64(); if (threadIdx.x == 0) t[0] = (t1 - t0);
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = x * a; x = x * b; x = x * a; x = x * b; }
    t1 = clock64(); if (threadIdx.x == 0) t[1] = (t1 - t0);
    // SHFL chain (double: 2 shfl)
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { x = __shfl_up_sync(0xffffffffu, x, 1) + 0.0; x = __shfl_up_sync(0xffffffffu, x, 1); x = __shfl_up_sync(0xffffffffu, x, 1); x = __shfl_up_sync(0xffffffffu, x, 1); }
    t1 = clock64(); if (threadIdx.x == 0) t[2] = (t1 - t0);
    // LDS chain (address from value)
    int idx = threadIdx.x & 31;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { idx = (int)sm[idx]; idx = (int)sm[idx]; idx = (int)sm[idx]; idx = (int)sm[idx]; }
    t1 = clock64(); if (threadIdx.x == 0) t[3] = (t1 - t0);
    // STS -> syncwarp -> LDS by the next lane (the coarse sweep's North hand-off), 4 per iter
    double v = x;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            sm[threadIdx.x] = v; __syncwarp();
            v = sm[(threadIdx.x + 31) & 31] * a; __syncwarp();
        }
    }
    t1 = clock64(); if (threadIdx.x == 0) t[4] = (t1 - t0);
    // integer add chain (baseline)
    int z = idx;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { z = z * 3 + 1; z = z * 3 + 1; z = z * 3 + 1; z = z * 3 + 1; }
    t1 = clock64(); if (threadIdx.x == 0) t[5] = (t1 - t0);
    out[threadIdx.x] = x + v + idx + z;
}
int main()
{
    double *o; long long *t, h[8];
    cudaMalloc(&o, 64 * 8); cudaMalloc(&t, 64);
    const int it = 1000;
    for (int rep = 0; rep < 2; ++rep) k<<<1, 32>>>(o, t, 1.0000001, 1e-9, it);
    cudaMemcpy(h, t, 48, cudaMemcpyDeviceToHost);
    const char *nm[6] = {"DFMA", "DMUL", "SHFL+DADD(1/4)", "LDS(int cvt)", "STS>sync>LDS>DMUL>sync", "IMAD"};
    for (int i = 0; i < 6; ++i) printf("%-26s %.1f cycles/op\n", nm[i], (double)h[i] / (4.0 * it));
    return 0;
}
