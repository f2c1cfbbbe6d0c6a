// Microbenchmark of the k_wave step chain: per "chunk" 12 LDS.128 + 8 steps of
// (4 SHFL64-halves, FSEL, 4 DFMA) + 4 STS.128, one warp, data in shared memory.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double *out, long long *cyc, int nchunks)
{
    __shared__ __align__(16) double sq[3 * 512 + 64];
    for (int i = threadIdx.x; i < 3 * 512; i += 32) sq[i] = 0.5 + 1e-3 * i;
    __syncwarp();
    const int lane = threadIdx.x;
    const int rowoff = (31 - lane) * 16, sw = (31 - lane) & 7;
    double z1 = 0.1 * lane, z2 = 0.2;
    long long t0 = clock64();
    for (int c = 0; c < nchunks; ++c) {
#pragma unroll
        for (int G = 0; G < 2; ++G) {
            double2 Q[4], A1[4], A2[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int st = 4 * G + u;
                const int xo = rowoff + (((7 - st) ^ sw) << 1);
                Q[u] = *reinterpret_cast<const double2 *>(sq + xo);
                A1[u] = *reinterpret_cast<const double2 *>(sq + 512 + xo);
                A2[u] = *reinterpret_cast<const double2 *>(sq + 1024 + xo);
            }
            double Z[8];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                double n0, n1;
                if (MODE == 0) { n0 = __shfl_up_sync(0xffffffffu, z2, 1); n1 = __shfl_up_sync(0xffffffffu, z1, 1); }
                else { n0 = z2 * 0.5; n1 = z1 * 0.5; }   // no shuffle (chain without communication)
                if (lane == 0) { n0 = 0.25; n1 = 0.125; }
                double za = fma(A1[u].y, z1, fma(A2[u].y, n0, Q[u].y));
                double zc = fma(A1[u].x, za, fma(A2[u].x, n1, Q[u].x));
                Z[2 * u] = za; Z[2 * u + 1] = zc;
                z2 = za; z1 = zc;
            }
            if (MODE != 2) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int st = 4 * G + u;
                    const int xo = rowoff + (((7 - st) ^ sw) << 1);
                    *reinterpret_cast<double2 *>(sq + xo) = make_double2(Z[2 * u + 1] * 1e-3, Z[2 * u] * 1e-3);
                }
            }
        }
    }
    long long t1 = clock64();
    out[lane] = z1 + z2;
    if (lane == 0) cyc[MODE] = t1 - t0;
}
int main()
{
    double *o; long long *c, h[4];
    cudaMalloc(&o, 4096); cudaMalloc(&c, 64);
    const int n = 2000;
    k<0><<<1, 32>>>(o, c, n); k<1><<<1, 32>>>(o, c, n); k<2><<<1, 32>>>(o, c, n);
    cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("cycles per chunk (16 columns): with shuffles %.0f, without shuffles %.0f, shuffles no in-place store %.0f\n",
           h[0] / (double)n, h[1] / (double)n, h[2] / (double)n);
    return 0;
}
