#include <cstdio>
#include <cuda_runtime.h>
__global__ void body(int* it, cudaGraphConditionalHandle h, int n) {
  if (threadIdx.x == 0) { int v = ++(*it); cudaGraphSetConditional(h, v < n ? 1 : 0); }
}
__global__ void k_init(cudaGraphConditionalHandle h) { cudaGraphSetConditional(h, 1); }
int main() {
  int* it; cudaMalloc(&it, 4); cudaMemset(it, 0, 4);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  printf("handle: %s\n", cudaGetErrorString(e));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cn;
  e = cudaGraphAddNode(&cn, g, nullptr, 0, &cp);
  printf("cond node: %s\n", cudaGetErrorString(e));
  cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
  cudaStream_t s; cudaStreamCreate(&s);
  // capture the body into bodyg
  e = cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
  printf("begin capture: %s\n", cudaGetErrorString(e));
  body<<<1, 32, 0, s>>>(it, h, 1000);
  e = cudaStreamEndCapture(s, &bodyg);
  printf("end capture: %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ge;
  e = cudaGraphInstantiate(&ge, g, 0);
  printf("instantiate: %s\n", cudaGetErrorString(e));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, s);
  e = cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaStreamSynchronize(s);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int hv; cudaMemcpy(&hv, it, 4, cudaMemcpyDeviceToHost);
  printf("launch: %s iterations %d in %.3f ms (%.2f us/iter)\n", cudaGetErrorString(e), hv, ms, 1e3 * ms / hv);
  return 0;
}
