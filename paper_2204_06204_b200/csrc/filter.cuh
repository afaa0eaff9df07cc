#pragma once
#include "common.cuh"

namespace bsp {

constexpr int kMaxTaps = 31;

struct DevState;

struct FilterTaps {
  double w[kMaxTaps];
  double cum[kMaxTaps + 1];  // cum[k] = w[0] + ... + w[k-1]: O(1) boundary masses
  int size, r;
};

struct FilterArgs {
  FilterTaps w;
  int nx, ny;
  const double* in;
  double* out;
  double* act;              // fwd only, nullable: act = out^eta
  double eta;
  const int* gate0;
  // adjoint only, nullable st: reduce sum(out) over active elements -> st->gsum
  DevState* st;
  const uint8_t* active;
  RedBuf rb;
};

__global__ void k_filter_fwd(FilterArgs p);
__global__ void k_filter_adj(FilterArgs p);
size_t filter_smem_bytes(int r);
dim3 filter_grid(int nx, int ny);

}  // namespace bsp
