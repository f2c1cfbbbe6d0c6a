// Probe 2: the exact tensor-map geometry of the failing level-0 GS sweep (pitch 80, 66 rows,
// base 168960 B into a larger allocation), dynamic shared memory aligned by hand.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>

struct Maps { CUtensorMap a, b, c; };
__global__ void k(const __grid_constant__ Maps m, int x0, int y0, int which)
{
    extern __shared__ double raw[];
    double *sm = (double *)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ alignas(8) uint64_t bar;
    unsigned sb = (unsigned)__cvta_generic_to_shared(&bar), sd = (unsigned)__cvta_generic_to_shared(sm);
    if (threadIdx.x == 0) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    const CUtensorMap *tm = which == 0 ? &m.a : which == 1 ? &m.b : &m.c;
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(sb), "r"(32 * 16 * 8));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(sd), "l"(tm), "r"(x0), "r"(y0), "r"(sb) : "memory");
    }
    asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], 0; @!p bra W; }" ::"r"(sb));
}

int main(int argc, char **argv)
{
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    double *blk;
    cudaMalloc(&blk, 8 << 20);
    cudaMemset(blk, 0, 8 << 20);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    long pitch = atol(argv[1]), rows = atol(argv[2]), off = atol(argv[3]), extra = atol(argv[4]);
    int x = atoi(argv[5]), y = atoi(argv[6]);
    Maps mm;
    cuuint64_t dim[2] = {(cuuint64_t)(pitch + 2 * rows + extra), (cuuint64_t)rows};
    cuuint64_t str[1] = {(cuuint64_t)(pitch - 2) * 8};
    cuuint32_t box[2] = {16, 32}, es[2] = {1, 1};
    CUresult rc = enc(&mm.a, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, blk + off, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    k<<<1, 64, 93184>>>(mm, x, y, 0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("pitch %ld rows %ld off %ld dim0 %ld (x,y)=(%d,%d): rc=%d %s\n", pitch, rows, off, (long)dim[0], x, y, (int)rc, cudaGetErrorString(e));
    return e ? 1 : 0;
}
