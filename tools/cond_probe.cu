#include <cuda_runtime.h>
#include <cstdio>
__global__ void setc(cudaGraphConditionalHandle h, const double* v, double tol) {
  cudaGraphSetConditional(h, (*v < tol) ? 1u : 0u);
}
__global__ void body(double* x) { *x += 1.0; }
int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  double* d; cudaMalloc(&d, 16); cudaMemset(d, 0, 16);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 0, 0);
  cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  setc<<<1,1,0,s>>>(h, d, 2.0);
  cudaStreamCaptureStatus st; const cudaGraphNode_t* deps; size_t nd;
  cudaStreamGetCaptureInfo(s, &st, nullptr, nullptr, &deps, &nd);
  cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
  cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeIf; cp.conditional.size = 1;
  cudaGraphNode_t cn;
  cudaError_t e = cudaGraphAddNode(&cn, g, deps, nd, &cp);
  printf("add %d\n", (int)e);
  cudaStreamUpdateCaptureDependencies(s, &cn, 1, cudaStreamSetCaptureDependencies);
  cudaGraph_t g2; cudaStreamEndCapture(s, &g2);
  cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
  cudaStreamBeginCaptureToGraph(s, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  body<<<1,1,0,s>>>(d);
  cudaStreamEndCapture(s, &bodyg);
  cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0); printf("inst %d\n", (int)e);
  for (int i = 0; i < 3; ++i) cudaGraphLaunch(ex, s);
  double hv; cudaMemcpy(&hv, d, 8, cudaMemcpyDeviceToHost); printf("val %g (expect 2)\n", hv);
  return 0;
}
