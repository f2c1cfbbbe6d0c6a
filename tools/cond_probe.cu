#include <cstdio>
#include <cuda_runtime.h>
__global__ void body(int *cnt, cudaGraphConditionalHandle h) {
  int c = ++(*cnt);
  cudaGraphSetConditional(h, c < 5 ? 1 : 0);
}
__global__ void init(int *cnt, cudaGraphConditionalHandle h) { *cnt = 0; cudaGraphSetConditional(h, 1); }
int main() {
  int *cnt; cudaMalloc(&cnt, 4);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  printf("handle %s\n", cudaGetErrorString(cudaGraphConditionalHandleCreate(&h, g, 0, 0)));
  // init node via capture into g
  cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeGlobal);
  init<<<1,1,0,s>>>(cnt, h);
  cudaStreamCaptureStatus st; const cudaGraphNode_t *deps; size_t nd; cudaGraph_t gg;
  cudaStreamGetCaptureInfo(s, &st, nullptr, &gg, &deps, &nd);
  cudaGraphNodeParams p = {}; p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
  cudaGraphNode_t cn;
  printf("add %s\n", cudaGetErrorString(cudaGraphAddNode(&cn, g, deps, nd, &p)));
  cudaStreamUpdateCaptureDependencies(s, &cn, 1, cudaStreamSetCaptureDependencies);
  cudaGraph_t bodyg = p.conditional.phGraph_out[0];
  cudaStream_t s2; cudaStreamCreate(&s2);
  printf("cap2 %s\n", cudaGetErrorString(cudaStreamBeginCaptureToGraph(s2, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed)));
  body<<<1,1,0,s2>>>(cnt, h);
  cudaGraph_t tmp; printf("end2 %s\n", cudaGetErrorString(cudaStreamEndCapture(s2, &tmp)));
  cudaGraph_t out; printf("end %s\n", cudaGetErrorString(cudaStreamEndCapture(s, &out)));
  cudaGraphExec_t ex; printf("inst %s\n", cudaGetErrorString(cudaGraphInstantiate(&ex, g, 0)));
  printf("launch %s\n", cudaGetErrorString(cudaGraphLaunch(ex, s)));
  cudaStreamSynchronize(s); int hc; cudaMemcpy(&hc, cnt, 4, cudaMemcpyDeviceToHost); printf("count %d (expect 5)\n", hc);
  printf("launch2 %s\n", cudaGetErrorString(cudaGraphLaunch(ex, s)));
  cudaStreamSynchronize(s); cudaMemcpy(&hc, cnt, 4, cudaMemcpyDeviceToHost); printf("count %d %s\n", hc, cudaGetErrorString(cudaGetLastError()));
}
