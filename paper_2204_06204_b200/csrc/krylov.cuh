#pragma once
#include "common.cuh"

namespace bsp {

struct DevState;

constexpr int kTsqrMaxCols = 64;  // widest TSQR: count + 1 <= 64 (krylov_dim <= 62 formed)
// powers formed for a request of npow = min(krylov_dim + 1, n)
inline int krylov_formed(int npow) { return npow < kTsqrMaxCols - 1 ? npow : kTsqrMaxCols - 1; }

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
  int npow_req;        // powers the reference would form (min(dim + 1, n)); > 63 truncates
};

__global__ void k_tsqr_leaf(KryArgs p);
__global__ void k_tsqr_merge(KryArgs p, const double* Rin, int nin, double* Rout);
__global__ void k_kry_combine(KryArgs p);
size_t tsqr_smem_bytes();
// the narrow (24-column) variant, as the row-slab path uses it
int tsqr_threads();          // block size of k_tsqr_leaf / k_tsqr_merge
cudaError_t tsqr_prepare();  // one-time set-up of the TSQR kernels (none needed today)
int tsqr_max_cols();
int tsqr_fan_in();
int tsqr_leaves(long long n);
// either variant, chosen by the column count nc = count + 1 (capped at 64)
int tsqr_rdim(int nc);       // R factor stride of the variant (24 or 64)
int tsqr_fan_in(int nc);
int tsqr_leaves(long long n, int nc);
cudaError_t launch_tsqr_leaf(int nc, int blocks, const KryArgs& ka, cudaStream_t s);
cudaError_t launch_tsqr_merge(int nc, int nout, const KryArgs& ka, const double* rin, int nin,
                              double* rout, cudaStream_t s);

}  // namespace bsp
