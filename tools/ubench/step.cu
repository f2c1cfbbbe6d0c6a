// cycles per 8-step chunk of the k_wave step body (z-form fast path), one warp per SM sub-partition,
// variants: V0 = the shipped body (3 LDS.128 per step at that step, 4 SHFL, FSEL for lane 0),
// V1 = operands from registers (no LDS), V2 = V0 without the lane-0 select (E from the shuffle),
// V3 = V0 with the operand loads issued one step ahead, after the step's shuffles.
// NOISE warps per CTA add the write-back warp's smem traffic (16 LDS.64 + 16 STS.64 per chunk).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double shfl_up_v(double x)
{
    unsigned lo = (unsigned)__double_as_longlong(x), hi = (unsigned)(__double_as_longlong(x) >> 32), rl, rh;
    asm volatile("shfl.sync.up.b32 %0, %2, 1, 0, 0xffffffff;\n\tshfl.sync.up.b32 %1, %3, 1, 0, 0xffffffff;"
                 : "=r"(rl), "=r"(rh) : "r"(lo), "r"(hi));
    return __longlong_as_double(((long long)rh << 32) | rl);
}
template <int V>
__global__ void k(double *out, long long *cyc, int nch, int noise, int S)
{
    extern __shared__ __align__(1024) double sm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 6 * 1536; i += blockDim.x) sm[i] = 0.25 + 1e-4 * (i & 255);
    __syncthreads();
    if (w >= S) {                                  // noise warps
        if (w >= S + noise) return;
        double acc = 0;
        double *p = sm + 3 * 1536 + ((w - S) & 3) * 512;
        for (int c = 0; c < nch * 4; ++c) {
#pragma unroll
            for (int e = 0; e < 16; ++e) acc += p[(e * 32 + lane) & 511];
#pragma unroll
            for (int e = 0; e < 16; ++e) p[(e * 32 + lane + 7) & 511] = acc;
        }
        if (acc == 12345.0) out[threadIdx.x] = acc;
        return;
    }
    const int rowoff = (31 - lane) * 16, sw = (31 - lane) & 7;
    int xo[8];
#pragma unroll
    for (int st = 0; st < 8; ++st) xo[st] = rowoff + (((7 - st) ^ sw) << 1);
    auto lds2 = [](const double *pp) {
        double2 v;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(pp)));
        return v;
    };
    double z1 = 0.0, z2 = 0.0;
    double2 E[8];
#pragma unroll
    for (int st = 0; st < 8; ++st) E[st] = make_double2(1e-3 * st, 2e-3 * st);
    double2 Qr = make_double2(0.1, 0.2), A1r = make_double2(0.3, 0.2), A2r = make_double2(0.25, 0.2);
    long long t0 = clock64();
    for (int c = 0; c < nch; ++c) {
        const double *sq = sm + (c % 3) * 1536;
        double Z[16];
        double2 Qn, A1n, A2n;
        if (V == 3) { Qn = lds2(sq + xo[0]); A1n = lds2(sq + 512 + xo[0]); A2n = lds2(sq + 1024 + xo[0]); }
#pragma unroll
        for (int st = 0; st < 8; ++st) {
            double2 Q, A1, A2;
            double n0, n1;
            if (V == 4) {   // shuffles pinned ahead of the step's loads
                n0 = shfl_up_v(z2); n1 = shfl_up_v(z1);
                Q = lds2(sq + xo[st]); A1 = lds2(sq + 512 + xo[st]); A2 = lds2(sq + 1024 + xo[st]);
            } else if (V == 0 || V == 2) {
                Q = lds2(sq + xo[st]); A1 = lds2(sq + 512 + xo[st]); A2 = lds2(sq + 1024 + xo[st]);
                n0 = __shfl_up_sync(0xffffffffu, z2, 1); n1 = __shfl_up_sync(0xffffffffu, z1, 1);
            } else { n0 = __shfl_up_sync(0xffffffffu, z2, 1); n1 = __shfl_up_sync(0xffffffffu, z1, 1); }
            if (V == 0 || V == 2 || V == 4) {}
            else if (V == 1) { Q = Qr; A1 = A1r; A2 = A2r; }
            else {
                Q = Qn; A1 = A1n; A2 = A2n;
                if (st < 7) { Qn = lds2(sq + xo[st + 1]); A1n = lds2(sq + 512 + xo[st + 1]); A2n = lds2(sq + 1024 + xo[st + 1]); }
            }
            if (V != 2 && lane == 0) { n0 = E[st].x; n1 = E[st].y; }
            double za = fma(A1.y, z1, fma(A2.y, n0, Q.y));
            double zc = fma(A1.x, za, fma(A2.x, n1, Q.x));
            Z[2 * st] = za; Z[2 * st + 1] = zc;
            z2 = za; z1 = zc;
        }
#pragma unroll
        for (int st = 0; st < 8; ++st) *reinterpret_cast<double2 *>(const_cast<double *>(sq) + xo[st]) = make_double2(Z[2 * st + 1], Z[2 * st]);
        __syncwarp();
    }
    long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x * 8 + w] = t1 - t0;
    out[threadIdx.x] = z1 + z2;
}

template <int V>
void run(const char *nm, int warps_noise, int S)
{
    double *o; long long *c, h;
    cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 1 << 16);
    const int smem = 6 * 1536 * 8 + 4 * 512 * 8;
    cudaFuncSetAttribute(k<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int nch = 400;
    for (int r = 0; r < 2; ++r) k<V><<<1, 32 * (S + warps_noise), smem>>>(o, c, nch, warps_noise, S);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-36s S %d noise %d: %.0f cycles per chunk (%.1f per step)\n", nm, S, warps_noise, (double)h / nch, (double)h / nch / 8);
}

int main()
{
    for (int S : {1, 2, 5})
    for (int nz : {0, S}) {
        run<0>("V0 shipped (LDS at the step)", nz, S);
        run<1>("V1 operands in registers", nz, S);
        run<2>("V2 V0 without lane-0 select", nz, S);
        run<3>("V3 loads one step ahead", nz, S);
        run<4>("V4 shuffles pinned first", nz, S);
    }
    return 0;
}
