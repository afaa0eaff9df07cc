// Per-replay cost of a CUDA graph of K dependent kernels that do almost no
// work (grid G x 256 threads, one store each): the floor of a K-kernel
// iteration on this GPU.
#include <cuda_runtime.h>
#include <cstdio>
__global__ void tiny(double* p, int i) { p[blockIdx.x * blockDim.x + threadIdx.x] = i; }
int main() {
  double* d;
  cudaMalloc(&d, 1 << 26);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int grid : {1, 148, 296, 1184}) {
    for (int K : {1, 2, 6, 12}) {
      cudaGraph_t g;
      cudaGraphExec_t x;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      for (int k = 0; k < K; ++k) tiny<<<grid, 256, 0, s>>>(d, k);
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&x, g, 0);
      for (int i = 0; i < 50; ++i) cudaGraphLaunch(x, s);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
      const int R = 2000;
      for (int i = 0; i < R; ++i) cudaGraphLaunch(x, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %5d  kernels %2d: %.2f us per replay, %.2f us per kernel\n", grid, K,
             1000.0 * ms / R, 1000.0 * ms / R / K);
    }
  }
  return 0;
}
