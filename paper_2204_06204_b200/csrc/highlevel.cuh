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
  double alpha;              // used when alphas == nullptr
  const double* alphas;      // per-iteration step sizes (solver mode)
  int mean_projection;
  double tol_dv, tol_res;
  RedBuf rb;                 // k_hl_write reduction scratch
  double* part;              // [fix_blocks * 4] scratch of the cooperative k_hl_fix
  DevState* st;              // device state: gsum in, measurements out
  RecRow* rec;               // nullable: solver-mode record rows (+ termination, k++)
};

__global__ void k_hl_write(HLArgs p);
__global__ void k_hl_fix(HLArgs p);
__global__ void k_masked_sum(const double* g, const uint8_t* active, long long n, RedBuf rb,
                             DevState* st);
int highlevel_blocks(int device);
int write_blocks(long long E, int nsm);
// k_hl_write (+ cooperative k_hl_fix, a no-op unless the budget is active)
cudaError_t launch_highlevel(const HLArgs& a, int fix_blocks, int nsm, cudaStream_t s);

}  // namespace bsp
