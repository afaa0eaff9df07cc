#include <cuda_runtime.h>
#include <cstdio>
__global__ void setc(cudaGraphConditionalHandle h, const int* flag) { if (threadIdx.x == 0) cudaGraphSetConditional(h, *flag); }
__global__ void body(int* out) { out[0] += 1; }
int main() {
  cudaStream_t s; cudaStreamCreate(&s);
  int *d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  int one = 1; cudaMemcpy(d + 1, &one, 4, cudaMemcpyHostToDevice);
  cudaGraph_t g; cudaGraphCreate(&g, 0);
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault);
  printf("handle %d\n", (int)e);
  cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  setc<<<1, 32, 0, s>>>(h, d + 1);
  cudaStreamCaptureStatus st; const cudaGraphNode_t* deps; size_t nd; cudaGraph_t cg;
  e = cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd);
  printf("info %d nd %zu\n", (int)e, nd);
  cudaGraphNodeParams cp = {}; cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeIf; cp.conditional.size = 1;
  cudaGraphNode_t cn;
  e = cudaGraphAddNode(&cn, cg, deps, nd, &cp);
  printf("addnode %d\n", (int)e);
  e = cudaStreamUpdateCaptureDependencies(s, &cn, 1, cudaStreamSetCaptureDependencies);
  printf("upd %d\n", (int)e);
  cudaStream_t s2; cudaStreamCreate(&s2);
  cudaStreamBeginCaptureToGraph(s2, cp.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
  body<<<1, 1, 0, s2>>>(d);
  cudaGraph_t tmp; e = cudaStreamEndCapture(s2, &tmp); printf("body end %d\n", (int)e);
  body<<<1, 1, 0, s>>>(d);
  e = cudaStreamEndCapture(s, &g); printf("end %d\n", (int)e);
  cudaGraphExec_t x; e = cudaGraphInstantiate(&x, g, 0); printf("inst %d\n", (int)e);
  for (int i = 0; i < 3; ++i) cudaGraphLaunch(x, s);
  cudaStreamSynchronize(s);
  int out; cudaMemcpy(&out, d, 4, cudaMemcpyDeviceToHost); printf("out %d (expect 6)\n", out);
  one = 0; cudaMemcpy(d + 1, &one, 4, cudaMemcpyHostToDevice);
  for (int i = 0; i < 3; ++i) cudaGraphLaunch(x, s);
  cudaStreamSynchronize(s);
  cudaMemcpy(&out, d, 4, cudaMemcpyDeviceToHost); printf("out %d (expect 9)\n", out);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
