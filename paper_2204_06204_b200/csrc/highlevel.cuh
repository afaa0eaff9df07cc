#pragma once
#include "common.cuh"
#include "filter.cuh"
#include "solver_state.cuh"

namespace bsp {

// Grids up to this many elements may run the lambda search inside the last
// block of k_hl_write instead of launching the cooperative k_hl_fix
// (BSP_SMALL_FIX=<E>).  Off by default: measured on B200 at C2 (110k cells) it
// saves 4 us per steady-state iteration but the early iterations need the
// search often, and one SM streaming the design from HBM per round loses more
// (L2-flushed bench 0.047 -> 0.053 ms/iter).
constexpr long long kSmallFix = 0;
long long small_fix_limit();  // kSmallFix, or BSP_SMALL_FIX from the environment

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
  double* defer_out;         // row slabs: last block stores its 6 totals here (no hook)
  int host_lambda;           // row slabs: an active budget stops the batch (done = 3)
  long long small_fix;       // E <= small_fix: lambda search in k_hl_write's last block
  int nx, ny;                // k_hl_adj4: the grid (launch geometry)
};

// record row + termination (solvers.py:464-475)
BSP_DEV void hl_finalize(const HLArgs& p, double dv, double vol, double lam, int rounds);
// last-block logic of k_hl_write on the grid totals
// tot = (box sum, volume, n_mid, S_mid, max dv, max w)
BSP_DEV void hl_write_hook(const HLArgs& p, const double* tot);

__global__ void k_hl_write(HLArgs p);
__global__ void k_hl_fix(HLArgs p);
__global__ void k_masked_sum(const double* g, const uint8_t* active, long long n, RedBuf rb,
                             DevState* st);
int highlevel_blocks(int device);
int write_blocks(long long E, int nsm);
// k_hl_write (+ cooperative k_hl_fix, a no-op unless the budget is active)
cudaError_t launch_highlevel(const HLArgs& a, int fix_blocks, int nsm, cudaStream_t s);
// k_hl_write alone (the solver then launches k_hl_fix itself)
cudaError_t launch_hl_write(const HLArgs& a, int nsm, cudaStream_t s);
// the cooperative k_hl_fix alone (after k_hl_write or the fused k_hl_adj4)
cudaError_t launch_hl_fix(const HLArgs& a, int fix_blocks, cudaStream_t s);
// adjoint filter + high-level step in one pass (filter.cu): radius-3 filters
// without a passive region; the mean projection's sum of g must already be in
// st->gsum (the residual kernel's SF_SUM_SENS)
bool hl_adjoint_fusable(const FilterTaps& w, int nx, long long E, bool forked);
cudaError_t launch_hl_adjoint(const FilterTaps& w, const double* sens, const HLArgs& h,
                              cudaStream_t s);

}  // namespace bsp

namespace bsp {
BSP_DEV void hl_finalize(const HLArgs& p, double dv, double vol, double lam, int rounds) {
  DevState* st = p.st;
  st->dv_inf = dv;
  st->volume = vol;
  st->lambda = lam;
  st->lam_rounds = rounds;
  if (p.rec) {
    const long long k = st->k;
    RecRow& row = p.rec[k - st->k_base];
    row.compliance = st->compliance;
    row.res_inf = st->res_inf;
    row.dv_inf = dv;
    row.volume = vol;
    row.t_ns = globaltimer_ns();
    if (dv < p.tol_dv && st->res_inf < p.tol_res) {
      st->done = 1;
      st->conv_k = k;
    }
    st->k = k + 1;
  }
}

BSP_DEV void hl_write_hook(const HLArgs& p, const double* tot) {
  DevState* st = p.st;
  st->scratch[3] = tot[5];  // max w (lambda bracket)
  if (tot[0] > p.budget) {
    // projection.py:59-61 fails: the lambda search takes over, starting from
    // the root of the linear piece at lam = 0 (exact when no element changes
    // regime, e.g. the ulp-level overshoots of a mean-projected step)
    st->lam_needed = 1;
    st->scratch[4] = tot[2] > 0.0 ? (tot[0] - p.budget) / tot[2] : -1.0;
    st->scratch[5] = tot[0];
    if (p.host_lambda) st->done = 3;
  } else {
    hl_finalize(p, tot[4], tot[1], 0.0, 0);
  }
}
}  // namespace bsp
