#pragma once
#include "common.cuh"

namespace bsp {

struct DevState;
struct RecRow;

struct HLArgs {
  const double* v;           // [E] current design
  const double* g;           // [E] ascent direction (nullable -> plain projection of v)
  double* v_next;            // [E]
  const uint8_t* active;     // [E] nullable (no passive region)
  long long E;
  double n_active;
  double lo, hi, budget;
  double alpha;              // used when st == nullptr
  const double* alphas;      // per-iteration step sizes (solver mode)
  int mean_projection;
  double tol_dv, tol_res;
  double* part;              // [gridDim * 4] scratch
  DevState* st;              // nullable (solver mode when set)
  RecRow* rec;               // solver mode record rows
  double* diag;              // nullable [6]: mean, boxsum, lambda, rounds, dv_inf, volume
};

__global__ void k_highlevel(HLArgs p);
int highlevel_blocks(int device);
cudaError_t launch_highlevel(const HLArgs& a, int blocks, cudaStream_t s);

}  // namespace bsp
