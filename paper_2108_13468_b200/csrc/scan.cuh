// scan.cuh -- block-wide affine scans (first-order linear recurrences) used by the
// tridiagonal line solves: forward  y_k = al_k y_{k-1} + b_k  (y_{-1} = 0) and backward
// z_k = be_k z_{k+1} + y_k  (z_len = 0).  Each thread owns K consecutive elements; the
// recurrence is composed as affine maps through a warp shuffle scan and one shared-memory
// level (sA[32], sB[64]; skipped for a one-warp block, whose results are bitwise the same).
// All threads of the block must call these.
#pragma once
#include <cuda_runtime.h>

namespace spp {

// TAIL = false drops the trailing barrier when the caller's next shared-memory use is another scan
// or is itself behind a barrier (the scratch slots are disjoint between phases; see k_lines_tma).
template <int K, bool TAIL = true>
__device__ __forceinline__ void fwd_scan(double (&al)[K], double (&b)[K], double (&y)[K],
                                         double *sA, double *sB)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // thread aggregate of y -> al_K-1 (... (al_0 y + b_0) ...) + b_K-1
    double A = 1.0, B = 0.0;
#pragma unroll
    for (int k = 0; k < K; ++k) { B = al[k] * B + b[k]; A = al[k] * A; }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double Au = __shfl_up_sync(0xffffffffu, A, d), Bu = __shfl_up_sync(0xffffffffu, B, d);
        if (lane >= d) { B = A * Bu + B; A = A * Au; }
    }
    if (nw == 1) {                                     // one warp (short lines): no block level
        const double Be = __shfl_up_sync(0xffffffffu, B, 1);
        double yin = lane == 0 ? 0.0 : Be;
#pragma unroll
        for (int k = 0; k < K; ++k) { yin = al[k] * yin + b[k]; y[k] = yin; }
        __syncwarp();                                  // the caller's shared-memory ordering, as the barrier
        return;
    }
    if (lane == 31) { sA[w] = A; sB[w] = B; }
    __syncthreads();
    if (w == 0) {
        double WA = lane < nw ? sA[lane] : 1.0, WB = lane < nw ? sB[lane] : 0.0;
        for (int d = 1; d < nw; d <<= 1) {             // nw warps: log2(nw) levels
            const double Au = __shfl_up_sync(0xffffffffu, WA, d), Bu = __shfl_up_sync(0xffffffffu, WB, d);
            if (lane >= d) { WB = WA * Bu + WB; WA = WA * Au; }
        }
        // exclusive: value entering warp `lane` (y_{-1} = 0)
        const double ex = __shfl_up_sync(0xffffffffu, WB, 1);
        if (lane < nw) sB[32 + lane] = (lane == 0) ? 0.0 : ex;
    }
    // value entering this thread = lanes before it in the warp applied to the warp inflow
    const double Ae = __shfl_up_sync(0xffffffffu, A, 1), Be = __shfl_up_sync(0xffffffffu, B, 1);
    __syncthreads();
    const double yw = sB[32 + w];
    double yin = (lane == 0) ? yw : Ae * yw + Be;
#pragma unroll
    for (int k = 0; k < K; ++k) { yin = al[k] * yin + b[k]; y[k] = yin; }
    if (TAIL) __syncthreads();
}

template <int K, bool TAIL = true>
__device__ __forceinline__ void bwd_scan(double (&be)[K], double (&y)[K], double (&z)[K],
                                         double *sA, double *sB)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double A = 1.0, B = 0.0;   // map z_in (from the right) -> z at this thread's first element
#pragma unroll
    for (int k = K - 1; k >= 0; --k) { B = be[k] * B + y[k]; A = be[k] * A; }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const double Ad = __shfl_down_sync(0xffffffffu, A, d), Bd = __shfl_down_sync(0xffffffffu, B, d);
        if (lane + d < 32) { B = A * Bd + B; A = A * Ad; }
    }
    if (nw == 1) {
        const double Bd = __shfl_down_sync(0xffffffffu, B, 1);
        double zin = lane == 31 ? 0.0 : Bd;
#pragma unroll
        for (int k = K - 1; k >= 0; --k) { zin = be[k] * zin + y[k]; z[k] = zin; }
        __syncwarp();
        return;
    }
    if (lane == 0) { sA[w] = A; sB[w] = B; }
    __syncthreads();
    if (w == 0) {
        const int r = nw - 1 - lane;       // reversed warp order
        double WA = lane < nw ? sA[r] : 1.0, WB = lane < nw ? sB[r] : 0.0;
        for (int d = 1; d < nw; d <<= 1) {             // nw warps: log2(nw) levels
            const double Au = __shfl_up_sync(0xffffffffu, WA, d), Bu = __shfl_up_sync(0xffffffffu, WB, d);
            if (lane >= d) { WB = WA * Bu + WB; WA = WA * Au; }
        }
        const double ex = __shfl_up_sync(0xffffffffu, WB, 1);
        if (lane < nw) sB[32 + r] = (lane == 0) ? 0.0 : ex;
    }
    const double Ae = __shfl_down_sync(0xffffffffu, A, 1), Be = __shfl_down_sync(0xffffffffu, B, 1);
    __syncthreads();
    const double zw = sB[32 + w];
    double zin = (lane == 31) ? zw : Ae * zw + Be;
#pragma unroll
    for (int k = K - 1; k >= 0; --k) { zin = be[k] * zin + y[k]; z[k] = zin; }
    if (TAIL) __syncthreads();
}

}  // namespace spp
