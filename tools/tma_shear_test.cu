// Feasibility probe: a 2D TMA tensor map whose row stride (pitch-2)*8 B is smaller than
// its row extent (an overlapping "sheared" view), loaded as a 32x16 box with 128B swizzle.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

struct Maps { CUtensorMap a, b, c; };
__global__ void k2(const __grid_constant__ Maps m, int x0, int y0, double *out, int mode)
{
    __shared__ alignas(1024) double box[32 * 16];
    __shared__ alignas(8) uint64_t bar;
    unsigned sb = (unsigned)__cvta_generic_to_shared(&bar), sd = (unsigned)__cvta_generic_to_shared(box);
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sb));
    if (mode & 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sb), "r"(32 * 16 * 8));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(sd), "l"(&m.b), "r"(x0), "r"(y0), "r"(sb) : "memory");
        if (mode & 2) asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(&m.c), "r"(x0 - 16), "r"(y0) : "memory");
    }
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], 0; @!p bra W; }" ::"r"(sb));
    for (int i = threadIdx.x; i < 512; i += blockDim.x) out[i] = box[i];
}

__global__ void k(const __grid_constant__ CUtensorMap tm, int x0, int y0, double *out)
{
    __shared__ alignas(1024) double box[32 * 16];
    __shared__ alignas(8) uint64_t bar;
    unsigned sb = (unsigned)__cvta_generic_to_shared(&bar), sd = (unsigned)__cvta_generic_to_shared(box);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sb));
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sb), "r"(32 * 16 * 8));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(sd), "l"(&tm), "r"(x0), "r"(y0), "r"(sb) : "memory");
    }
    __syncthreads();
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], 0; @!p bra W; }" ::"r"(sb));
    for (int i = threadIdx.x; i < 512; i += blockDim.x) out[i] = box[i];
}

int main()
{
    const int pitch = 64, rows = 200;
    double *h = new double[(size_t)pitch * rows];
    for (int r = 0; r < rows; ++r) for (int c = 0; c < pitch; ++c) h[r * pitch + c] = r * 1000 + c;
    double *d, *o;
    cudaMalloc(&d, sizeof(double) * pitch * rows);
    cudaMalloc(&o, sizeof(double) * 512);
    cudaMemcpy(d, h, sizeof(double) * pitch * rows, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    if (!enc) { printf("no entry point\n"); return 1; }
    CUtensorMap tm;
    // element (X, R) at base + R*(pitch-2) + X  ->  physical column X - 2R of row R
    cuuint64_t dim[2] = {(cuuint64_t)(pitch + 2 * rows), (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)(pitch - 2) * 8};
    cuuint32_t box[2] = {16, 32}, es[2] = {1, 1};
    CUresult rc = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)rc);
    if (rc) return 2;
    const int x0 = 2 * 100 + 10, y0 = 100;     // rows 100..131; physical col of X=x0 in row R: x0 - 2R
    k<<<1, 128>>>(tm, x0, y0, o);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    double ho[512];
    cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 32; ++r)
        for (int x = 0; x < 16; ++x) {
            // 128B swizzle: 16-byte unit u = x/2 of row r stored at unit u ^ (r % 8)
            const int u = (x >> 1) ^ (r & 7);
            const double got = ho[r * 16 + u * 2 + (x & 1)];
            const int R = y0 + r, col = x0 + x - 2 * R;
            const double want = (col >= 0 && col < pitch) ? R * 1000 + col : -1;
            if (col >= 0 && col < pitch && got != want) { if (bad < 5) printf("r=%d x=%d got %g want %g\n", r, x, got, want); bad++; }
        }
    printf("mismatches %d\n", bad);
    Maps mm{tm, tm, tm};
    // negative coordinates: x < 0, y < 0, both
    int cx[3] = {-20, 10, -20}, cy[3] = {5, -7, -7};
    for (int q = 0; q < 3; ++q) {
        k2<<<1, 128>>>(mm, cx[q], cy[q], o, 0);
        cudaError_t e3 = cudaDeviceSynchronize();
        printf("neg coords (%d,%d): %s\n", cx[q], cy[q], cudaGetErrorString(e3));
        if (e3) return 5;
        k2<<<1, 128>>>(mm, cx[q] + 16, cy[q], o, 2);
        e3 = cudaDeviceSynchronize();
        printf("neg prefetch (%d,%d): %s\n", cx[q], cy[q], cudaGetErrorString(e3));
        if (e3) return 6;
    }
    for (int mode = 0; mode < 4; ++mode) {
        k2<<<1, 128>>>(mm, x0, y0, o, mode);
        cudaError_t e2 = cudaDeviceSynchronize();
        printf("k2 mode %d: %s\n", mode, cudaGetErrorString(e2));
        if (e2) return 4;
    }
    return bad ? 3 : 0;
}
