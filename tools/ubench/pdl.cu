// per-kernel cost of a chain of small dependent kernels replayed as a CUDA graph, with and without
// programmatic dependent launch (griddepcontrol.wait at kernel start, launch_dependents early)
#include <cstdio>
#include <cuda_runtime.h>

template <bool PDL>
__global__ void k(double *x, int n, int work)
{
    if (PDL) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (PDL) asm volatile("griddepcontrol.launch_dependents;");
    double acc = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double v = x[i];
        for (int r = 0; r < work; ++r) v = v * 1.0000001 + 1e-9;
        x[i] = v;
        acc += v;
    }
    if (acc == 1234.5) x[0] = acc;
}

template <bool PDL>
float run(int nk, int grid, int n, int work)
{
    double *x;
    cudaMalloc(&x, sizeof(double) * (n + 1));
    cudaMemset(x, 0, sizeof(double) * (n + 1));
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < nk; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid; cfg.blockDim = 256; cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at; cfg.numAttrs = PDL ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k<PDL>, x, n, work);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphExec_t ge;
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return -1; }
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaGraphLaunch(ge, s);
    cudaEventRecord(a, s);
    for (int r = 0; r < 5; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
    return ms * 1e3f / (5 * nk);
}

int main()
{
    for (int grid : {1, 148, 592})
        for (int n : {256, 65536, 1 << 20}) {
            const float t0 = run<false>(500, grid, n, 4), t1 = run<true>(500, grid, n, 4);
            printf("grid %4d n %8d: plain %.2f us/kernel, PDL %.2f us/kernel\n", grid, n, t0, t1);
        }
    return 0;
}
