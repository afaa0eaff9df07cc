#pragma once
#include "common.cuh"

namespace bsp {

struct DevState;

struct KryArgs {
  const double* Q;     // basis, column j at Q + j*ldq (q_0 = b)
  long long ldq;       // column stride (doubles), >= n
  long long n;         // DOFs
  double* Rbuf;        // leaf R factors [leaves * 24 * 24]
  DevState* st;
  const double* u;     // combine: base (nullable -> 0)
  double* out;         // combine: output
  double beta;
  double* coef_out;    // nullable: raw LSQ coefficients (diagnostics)
  int no_solve;        // row slabs: the single-CTA merge level stores R (no solve)
};

__global__ void k_tsqr_leaf(KryArgs p);
__global__ void k_tsqr_merge(KryArgs p, const double* Rin, int nin, double* Rout);
__global__ void k_kry_combine(KryArgs p);
size_t tsqr_smem_bytes();
int tsqr_threads();          // block size of k_tsqr_leaf / k_tsqr_merge
cudaError_t tsqr_prepare();  // one-time set-up of the TSQR kernels (none needed today)
int tsqr_max_cols();
int tsqr_fan_in();
int tsqr_leaves(long long n);

}  // namespace bsp
