#pragma once
#include "common.cuh"

namespace bsp {

constexpr int kMaxTaps = 31;

struct FilterTaps {
  double w[kMaxTaps];
  int size, r;
};

struct FilterArgs {
  FilterTaps w;
  int nx, ny;
  const double* in;
  double* out;
  double* act;      // fwd only, nullable: act = out^eta
  double eta;
  const int* gate0;
};

__global__ void k_filter_fwd(FilterArgs p);
__global__ void k_filter_adj(FilterArgs p);
size_t filter_smem_bytes(int r);
dim3 filter_grid(int nx, int ny);

}  // namespace bsp
