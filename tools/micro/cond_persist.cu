// Does a graph conditional handle created WITHOUT cudaGraphCondAssignDefault
// keep the value a kernel of the previous launch set?  Graph: IF(h){body:
// hits++} -> setter(h = 1).  Three launches: persisted -> hits == 2.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_body(int *hits) { atomicAdd(hits, 1); }
__global__ void k_set(cudaGraphConditionalHandle h, int v) { cudaGraphSetConditional(h, v); }

int main() {
  int *hits;
  cudaMalloc(&hits, 4);
  cudaMemset(hits, 0, 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaGraph_t g;
  cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 0, 0);  // default 0, no per-launch reset
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  cudaGraphNode_t nC;
  if (cudaGraphAddNode(&nC, g, nullptr, 0, &cp) != cudaSuccess) { printf("add cond failed\n"); return 1; }
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  k_body<<<1, 1, 0, s>>>(hits);
  cudaStreamEndCapture(s, &body);
  cudaStreamBeginCaptureToGraph(s, g, &nC, nullptr, 1, cudaStreamCaptureModeThreadLocal);
  k_set<<<1, 1, 0, s>>>(h, 1);
  cudaStreamEndCapture(s, &g);
  cudaGraphExec_t ex;
  if (cudaGraphInstantiate(&ex, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return 1; }
  for (int i = 0; i < 3; ++i) cudaGraphLaunch(ex, s);
  cudaStreamSynchronize(s);
  int hh = -1;
  cudaMemcpy(&hh, hits, 4, cudaMemcpyDeviceToHost);
  printf("hits after 3 launches: %d (%s) err=%s\n", hh, hh == 2 ? "persists" : "reset/undefined",
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
