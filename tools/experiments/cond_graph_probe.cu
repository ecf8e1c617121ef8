#include <cuda_runtime.h>
#include <cstdio>
__global__ void setc(cudaGraphConditionalHandle h, const int* c) { cudaGraphSetConditional(h, *c > 0 ? 1u : 0u); }
__global__ void body(int* c) { atomicSub(c, 1); }
int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int* c; cudaMalloc(&c, 4); int v = 5; cudaMemcpy(c, &v, 4, cudaMemcpyHostToDevice);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
  cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
  cudaGraphNode_t node; cudaError_t e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
  printf("add %s\n", cudaGetErrorString(e));
  cudaGraph_t bg = cp.conditional.phGraph_out[0];
  e = cudaStreamBeginCaptureToGraph(s, bg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  printf("cap %s\n", cudaGetErrorString(e));
  body<<<1,1,0,s>>>(c); setc<<<1,1,0,s>>>(h, c);
  e = cudaStreamEndCapture(s, &bg); printf("end %s\n", cudaGetErrorString(e));
  cudaGraphExec_t ex; e = cudaGraphInstantiate(&ex, g, 0); printf("inst %s\n", cudaGetErrorString(e));
  e = cudaGraphLaunch(ex, s); cudaStreamSynchronize(s); cudaMemcpy(&v, c, 4, cudaMemcpyDeviceToHost);
  printf("launch %s v=%d\n", cudaGetErrorString(e), v);
}
