// Microbenchmark: cycles per line of the k_lines block-wide affine scans (fwd + bwd), 256 threads,
// K = 8 elements per thread, 126 CTAs (one per SM) as in the real launch.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2108_13468_b200/csrc/scan.cuh"
using namespace spp;
__global__ void k(double *out, long long *cyc, int lines)
{
    __shared__ double sA[32], sB[64];
    double zp[8], al[8], be[8], b[8], y[8], zz[8];
    for (int k = 0; k < 8; ++k) { zp[k] = 0.1 * k; al[k] = 0.3 + 0.01 * k; be[k] = 0.2 + 0.01 * threadIdx.x * 1e-3; }
    __syncthreads();
    long long t0 = clock64();
    for (int l = 0; l < lines; ++l) {
        for (int k = 0; k < 8; ++k) b[k] = 0.5 * zp[k] + 1.0;
        double a2[8], b2[8];
        for (int k = 0; k < 8; ++k) { a2[k] = al[k]; b2[k] = be[k]; }
        fwd_scan<8>(a2, b, y, sA, sB);
        bwd_scan<8>(b2, y, zz, sA, sB);
        for (int k = 0; k < 8; ++k) zp[k] = zz[k] * 0.5;
    }
    long long t1 = clock64();
    double s = 0; for (int k = 0; k < 8; ++k) s += zp[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main()
{
    double *o; long long *c, h[128];
    cudaMalloc(&o, 126 * 256 * 8); cudaMalloc(&c, 128 * 8);
    k<<<126, 256>>>(o, c, 10); cudaDeviceSynchronize();
    k<<<126, 256>>>(o, c, 200); cudaMemcpy(h, c, 126 * 8, cudaMemcpyDeviceToHost);
    printf("cycles per line (fwd+bwd scan, 256 threads, K=8): %.0f  (%s)\n", h[0] / 200.0, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
