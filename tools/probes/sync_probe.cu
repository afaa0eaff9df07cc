// Floors for a latency-bound iteration: a CUDA graph of 6 dependent near-empty
// kernels vs one cooperative kernel with 5 grid syncs (592 CTAs x 128 threads).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_empty(double* x) { if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1.0; }
__global__ void k_sync5(double* x) {
  cg::grid_group G = cg::this_grid();
  for (int i = 0; i < 5; ++i) {
    if (threadIdx.x == 0 && blockIdx.x == 0) x[i] += 1.0;
    G.sync();
  }
}

int main() {
  double* x; cudaMalloc(&x, 64 * sizeof(double)); cudaMemset(x, 0, 64 * sizeof(double));
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 592, iters = 2000;
  // graph of 6 dependent kernels
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 6; ++i) k_empty<<<blocks, 128, 0, s>>>(x);
  cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
  for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(e0, s);
  for (int i = 0; i < iters; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(e1, s); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("graph of 6 empty kernels (%d CTAs): %.2f us per graph\n", blocks, ms * 1000 / iters);
  void* args[] = {&x};
  for (int i = 0; i < 10; ++i) cudaLaunchCooperativeKernel((void*)k_sync5, blocks, 128, args, 0, s);
  cudaEventRecord(e0, s);
  for (int i = 0; i < iters; ++i) cudaLaunchCooperativeKernel((void*)k_sync5, blocks, 128, args, 0, s);
  cudaEventRecord(e1, s); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("cooperative kernel with 5 grid syncs (%d CTAs): %.2f us per launch\n", blocks, ms * 1000 / iters);
  // graph containing the cooperative kernel
  cudaGraph_t g2; cudaGraphExec_t ge2;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  cudaLaunchCooperativeKernel((void*)k_sync5, blocks, 128, args, 0, s);
  cudaStreamEndCapture(s, &g2); cudaGraphInstantiate(&ge2, g2, 0);
  for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge2, s);
  cudaEventRecord(e0, s);
  for (int i = 0; i < iters; ++i) cudaGraphLaunch(ge2, s);
  cudaEventRecord(e1, s); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("graph with that cooperative kernel: %.2f us per graph\n", ms * 1000 / iters);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
