// tma.cuh -- TMA tensor loads and mbarrier waits shared by the sweep and line kernels (sm_100a)
#pragma once
#include <cuda.h>

namespace spp {

__device__ __forceinline__ void tma_load(unsigned dst, const CUtensorMap *tm, int x, int y, unsigned bar)
{
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(dst), "l"(tm), "r"(x), "r"(y), "r"(bar) : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap *tm, int x, int y)
{
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(tm), "r"(x), "r"(y) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity)
{
    asm volatile("{\n .reg .pred p;\n W%=: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W%=;\n}"
                 ::"r"(bar), "r"(parity) : "memory");
}

}  // namespace spp
