// Device-resident state of one bilevel run (the loop of reference
// solvers.py:416-475 lives on the GPU; the host only reads records).
#pragma once
#include "common.cuh"

namespace bsp {

constexpr int kMaxKrylov = 64;   // basis norms / coefficients (at most 63 powers are formed)
constexpr int kMaxPower = 2;     // power-iteration norms (ping-pong: any iteration count)

struct DevState {
  long long k;          // iteration number of the iteration about to run (1-based)
  long long k_base;     // first iteration of the current batch (alphas index base)
  long long div_k;      // iteration that produced a non-finite residual
  long long conv_k;     // iteration at which the termination test fired
  int done;             // 0 running, 1 converged, 2 diverged
  int kry_count;        // Krylov powers accepted (reference `count`)
  int kry_stop;         // basis stopped (b == 0 or zero growth)
  int kry_rank;         // rank after the 1e-13 cut (diagnostic)
  int pow_stop;         // power iteration hit a zero vector
  int lam_rounds;       // lambda-search rounds of the last projection (diag)
  int lam_needed;       // box early exit failed: k_hl_fix must run
  int kry_trunc;        // krylov_dim > 62 and the rank cut fell beyond the 63 formed powers
  double res_inf, compliance, rnorm;
  double dv_inf, volume, lambda;
  double rho;           // power iteration Rayleigh quotient
  double gsum;          // sum of g over active elements (mean projection)
  double norms[kMaxKrylov];   // Krylov: norms[0]=|b|, norms[i+1]=growth_i
  double coef[kMaxKrylov];    // Krylov combination weights on q_i
  double pw[kMaxPower];       // power iteration norms
  double scratch[16];
};

// record row written by the high-level step finaliser
struct RecRow {
  double compliance, res_inf, dv_inf, volume;
  unsigned long long t_ns;  // %globaltimer when the iteration's record row was written
};

}  // namespace bsp
