// Microbenchmark of the k_wave chunk body under SM-level contention: W compute warps, each
// doing per chunk 24 LDS.128 operand loads + 8 shuffle/DFMA steps + 8 STS.128 (in place), with
// optional write-back traffic (32 LDS.64 + 16 DMUL + 16 STG) and an optional bulk-copy warp that
// writes 16 KB per warp-chunk into shared memory (the TMA traffic of the real kernel).
#include <cstdio>
#include <cuda_runtime.h>
template <bool WB, bool BULK>
__global__ void __launch_bounds__(160) k(double *out, const double *src, long long *cyc, int nchunks, int W)
{
    extern __shared__ __align__(1024) double sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *sq = sm + w * 4096;                    // 32 KB per warp (two slots of 3 x 512 + pad)
    double *scratch = sm + 5 * 4096;               // bulk-copy target (16 KB)
    __shared__ __align__(8) unsigned long long bar;
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)));
    for (int i = threadIdx.x; i < 4 * 4096; i += blockDim.x) sm[i] = 0.5 + 1e-3 * (i & 1023);
    __syncthreads();
    if (w == W) {                                  // bulk-copy warp
        if (!BULK || lane != 0) return;
        unsigned ph = 0;
        const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
        for (int c = 0; c < nchunks * W; ++c) {
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(16384u) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"((unsigned)__cvta_generic_to_shared(scratch)), "l"(src + (c & 63) * 2048), "r"(16384u), "r"(b) : "memory");
            asm volatile("{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W%=;\n}" ::"r"(b), "r"(ph) : "memory");
            ph ^= 1;
        }
        return;
    }
    if (w > W) return;
    const int rowoff = (31 - lane) * 16, sw = (31 - lane) & 7;
    double z1 = 0.1 * lane, z2 = 0.2;
    double *o = out + (size_t)w * 65536 + lane;
    long long t0 = clock64();
    for (int c = 0; c < nchunks; ++c) {
        double *s = sq + (c & 1) * 2048;
        const double *p = sq + ((c + 1) & 1) * 2048;
        double2 Q[8], A1[8], A2[8];
#pragma unroll
        for (int st = 0; st < 8; ++st) {
            const int xo = rowoff + (((7 - st) ^ sw) << 1);
            Q[st] = *reinterpret_cast<const double2 *>(s + xo);
            A1[st] = *reinterpret_cast<const double2 *>(s + 512 + xo);
            A2[st] = *reinterpret_cast<const double2 *>(s + 1024 + xo);
        }
        double Y[16];
        if (WB) {
#pragma unroll
            for (int e = 0; e < 16; ++e) Y[e] = p[(31 - 2 * e - (lane >> 4)) * 16 + (lane & 15)] * p[1536 + (31 - 2 * e - (lane >> 4)) * 16 + (lane & 15)];
        }
        double Z[16];
#pragma unroll
        for (int st = 0; st < 8; ++st) {
            double n0 = __shfl_up_sync(0xffffffffu, z2, 1), n1 = __shfl_up_sync(0xffffffffu, z1, 1);
            if (lane == 0) { n0 = 0.25; n1 = 0.125; }
            double za = fma(A1[st].y, z1, fma(A2[st].y, n0, Q[st].y));
            double zc = fma(A1[st].x, za, fma(A2[st].x, n1, Q[st].x));
            Z[2 * st] = za; Z[2 * st + 1] = zc; z2 = za; z1 = zc;
            if (WB) { o[(2 * st) * 4096] = Y[2 * st]; o[(2 * st + 1) * 4096] = Y[2 * st + 1]; }
        }
#pragma unroll
        for (int st = 0; st < 8; ++st) {
            const int xo = rowoff + (((7 - st) ^ sw) << 1);
            *reinterpret_cast<double2 *>(s + xo) = make_double2(Z[2 * st + 1] * 1e-3, Z[2 * st] * 1e-3);
        }
        __syncwarp();
    }
    long long t1 = clock64();
    o[0] += z1 + z2;
    if (lane == 0) cyc[w] = t1 - t0;
}
int main()
{
    double *o, *src; long long *c, h[8];
    cudaMalloc(&o, 8 << 20); cudaMalloc(&src, 2 << 20); cudaMalloc(&c, 64);
    cudaMemset(src, 0, 2 << 20);
    const int n = 2000, smem = 6 * 4096 * 8;
    cudaFuncSetAttribute(k<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int W : {1, 2, 4}) {
        for (int mode = 0; mode < 4; ++mode) {
            cudaMemset(c, 0, 64);
            if (mode == 0) k<false, false><<<1, 32 * (W + 1), smem>>>(o, src, c, n, W);
            if (mode == 1) k<true, false><<<1, 32 * (W + 1), smem>>>(o, src, c, n, W);
            if (mode == 2) k<false, true><<<1, 32 * (W + 1), smem>>>(o, src, c, n, W);
            if (mode == 3) k<true, true><<<1, 32 * (W + 1), smem>>>(o, src, c, n, W);
            cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
            printf("W=%d wb=%d bulk=%d: cycles per chunk (warp 0) %.0f  err=%s\n", W, mode & 1, mode >> 1, h[0] / (double)n,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
