// Probe: cost of an IF conditional graph node (body: a cooperative kernel)
// against an unconditional cooperative kernel that exits at once, inside a
// captured 3-kernel chain.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// cond_probe.cu -o /tmp/cond_probe && /tmp/cond_probe
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_a(int* flag, cudaGraphConditionalHandle h, int use_h) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (use_h && *flag) cudaGraphSetConditional(h, 1);
  }
}
__global__ void k_fix(int* flag, int* cnt) {
  if (!*flag) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(cnt, 1);
}
__global__ void k_c(int* cnt) {
  if (blockIdx.x == 0 && threadIdx.x == 0) cnt[1] += 1;
}

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

static int launch_fix(cudaStream_t s, int* flag, int* cnt, int blocks) {
  void* kp[] = {&flag, &cnt};
  CK(cudaLaunchCooperativeKernel((const void*)k_fix, dim3(blocks), dim3(256), kp, 0, s));
  return 0;
}

int main() {
  int *flag, *cnt;
  CK(cudaMalloc(&flag, 4));
  CK(cudaMalloc(&cnt, 8));
  CK(cudaMemset(flag, 0, 4));
  CK(cudaMemset(cnt, 0, 8));
  int nsm = 0, per = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_fix, 256, 0);
  const int blocks = nsm * (per > 4 ? 4 : per);
  {  // conditional nodes at all: a manually built graph
    cudaGraph_t mg;
    CK(cudaGraphCreate(&mg, 0));
    cudaGraphConditionalHandle hh;
    CK(cudaGraphConditionalHandleCreate(&hh, mg, 0, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hh;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    cudaError_t e = cudaGraphAddNode(&node, mg, nullptr, 0, &cp);
    printf("manual graph: cudaGraphAddNode -> %s\n", cudaGetErrorString(e));
    cudaGetLastError();
  }
  cudaStream_t s, side;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
  for (int mode = 0; mode < 2; ++mode) {
    cudaGraph_t g;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    cudaGraphConditionalHandle h = 0;
    if (mode == 1) {
      cudaStreamCaptureStatus st;
      cudaGraph_t cg;
      CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, nullptr, nullptr));
      CK(cudaGraphConditionalHandleCreate(&h, cg, 0, cudaGraphCondAssignDefault));
    }
    for (int rep = 0; rep < 8; ++rep) {
      k_a<<<blocks, 256, 0, s>>>(flag, h, mode);
      if (mode == 0) {
        if (launch_fix(s, flag, cnt, blocks)) return 1;
      } else {
        cudaStreamCaptureStatus st;
        cudaGraph_t cg;
        const cudaGraphNode_t* deps;
        size_t nd;
        CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &cg, &deps, &nd));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 1;
        cudaGraphNode_t node;
        cudaError_t ea = cudaGraphAddNode(&node, cg, deps, nd, &cp);
        if (ea != cudaSuccess) {
          printf("capture AddNode: %s (nd=%zu, status=%d)\n", cudaGetErrorString(ea), nd, (int)st);
          cudaGetLastError();
          cudaGraphConditionalHandle h2;
          CK(cudaGraphConditionalHandleCreate(&h2, cg, 0, 0));
          cp.conditional.handle = h2;
          ea = cudaGraphAddNode(&node, cg, deps, nd, &cp);
          printf("retry with a fresh handle, flags 0: %s\n", cudaGetErrorString(ea));
          if (ea != cudaSuccess) return 1;
        }
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(side, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        if (launch_fix(side, flag, cnt, blocks)) return 1;
        cudaGraph_t body_out;
        CK(cudaStreamEndCapture(side, &body_out));
        CK(cudaStreamUpdateCaptureDependencies(s, &node, 1, cudaStreamSetCaptureDependencies));
      }
      k_c<<<1, 32, 0, s>>>(cnt);
    }
    CK(cudaStreamEndCapture(s, &g));
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, g, 0));
    for (int f = 0; f < 2; ++f) {
      CK(cudaMemset(flag, f, 4));
      CK(cudaMemset(cnt, 0, 8));
      for (int i = 0; i < 20; ++i) CK(cudaGraphLaunch(ex, s));
      CK(cudaStreamSynchronize(s));
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      const int N = 500;
      CK(cudaEventRecord(e0, s));
      for (int i = 0; i < N; ++i) CK(cudaGraphLaunch(ex, s));
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      int hc[2];
      CK(cudaMemcpy(hc, cnt, 8, cudaMemcpyDeviceToHost));
      printf("mode %s flag %d: %.3f us per 3-kernel step (fix ran %d times of %d)\n",
             mode ? "conditional" : "always", f, ms * 1e3 / (N * 8), hc[0], (N + 20) * 8);
    }
  }
  return 0;
}
