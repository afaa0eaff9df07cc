// Masked matrix-free Q4 stiffness operator K(a)·u on the structured grid.
// Restates reference fea.py:150-181 (apply_stiffness), fea.py:197-201
// (element_energies), fea.py:184-189 (stiffness_diagonal, fused as d = kd·Σa),
// and the residual/compliance block of solvers.py:447-455.
//
// B200 mapping:
//  * one warp owns 32 consecutive element columns and emits 31 node columns;
//    each lane walks a vertical strip of R element rows with a 2-row register
//    window (u of the element's top and bottom node pairs), so every u, a
//    value is loaded from HBM once per strip (+1 halo row per strip);
//  * the left node of each element comes from the neighbouring lane by
//    __shfl_up, the right-column partial sums go back by __shfl_down -> no
//    shared memory, no atomics, deterministic summation order;
//  * element algebra runs in the per-component Hadamard mode basis
//    (dx, dy, hourglass), ~46 fp64 ops per element instead of 72 for the
//    dense 8x8 product, which keeps the kernel under the HBM roofline at B200's
//    fp64 rate (64 DFMA/clk/SM);
//  * epilogue fusions: r = Ku - f, d^2 scaling (Jacobi), axpy with a base
//    vector, element energies x SIMP prefactor, and a deterministic grid
//    reduction of (u.Ku, |t|^2, dot, max|t|) with a finalisation hook.
#pragma once
#include "common.cuh"

namespace bsp {

enum StiffFlags : int {
  SF_SUB_LOAD = 1,   // t = Ku - f
  SF_D2DIV = 2,      // t /= diag(K)^2   (PFBTO Jacobi squared, solvers.py:278)
  SF_AXPY = 4,       // out = base - beta * t
  SF_ENERGY = 8,     // sens[e] = pre(vp) * 1/2 u_e^T ke u_e
  SF_REDUCE = 16,    // grid reduction + hook
  SF_REDUCE_DOT = 32,  // (internal) stage and reduce the dot vector
  SF_STAGE_VP = 64,    // (internal) stage v_phys for the SIMP prefactor
  SF_IN_MASKED = 128,  // input is zero on fixed DOFs: skip input masking
  SF_D1DIV = 256,      // t /= diag(K)     (damped-Jacobi smoother sweep)
  SF_BASE_U = 512,     // (internal, TMA kernel) axpy base == input: read it from the u stage
  SF_A_POW = 1024,     // `a` holds v_phys: the activation is act_pow(a, eta), computed
                       // in-kernel (the filter then writes no activation array)
  SF_PROLONG = 2048,   // (TMA kernel) input u := u + M P~ pc on the fly: the multigrid
                       // prolongation fused into the first post-smoothing sweep
  SF_RED_NOMAX = 8192,   // (internal, TMA kernel) the reduction skips max|t|
  SF_RED_NOS0 = 16384,   // (internal, TMA kernel) the reduction skips u.Ku
  SF_SUM_SENS = 4096,  // (TMA kernel, with SF_ENERGY) reduce sum(sens) into the dot slot;
                       // the residual hook stores it as the mean projection's sum of g
                       // (sum C^T s = sum s: the renormalised filter has C 1 = 1)
};

enum StiffHook : int {
  HK_STORE = 0,      // red_out[0..3] = (u.Ku, |t|^2, dot, max|t|)
  HK_RESIDUAL = 1,   // solver: compliance/res_inf/divergence/Krylov b-norm
  HK_KRYLOV = 2,     // solver: Krylov power i norm
  HK_POWER = 3,      // power iteration: rho = u.Ku (or dot), norm
  HK_POWER_DOT = 4,  // power iteration on K M^-2 K: rho = dot
};

struct DevState;  // solver state (solver.cuh)

// Launch shapes with a compile-time flag set (dead epilogues removed); other
// flag sets run the run-time-flags instance of the cp.async kernel.  The
// SF_IN_MASKED shapes and the public unmasked matvec (0) also have a TMA
// instance (stiffness_tma.cu).
constexpr int kResid = SF_SUB_LOAD | SF_REDUCE | SF_ENERGY | SF_STAGE_VP | SF_IN_MASKED;
#define BSP_STIFF_SHAPES_MASKED(X)                      \
  X(SF_IN_MASKED)                                       \
  X(SF_IN_MASKED | SF_REDUCE)                           \
  X(SF_IN_MASKED | SF_AXPY)                             \
  X(SF_IN_MASKED | SF_D2DIV)                            \
  X(SF_IN_MASKED | SF_REDUCE | SF_REDUCE_DOT)           \
  X(kResid)                                             \
  X(kResid | SF_AXPY)                                   \
  X(kResid | SF_D2DIV)                                  \
  X(SF_IN_MASKED | SF_SUB_LOAD)                         \
  X(SF_IN_MASKED | SF_SUB_LOAD | SF_REDUCE)             \
  X(SF_IN_MASKED | SF_SUB_LOAD | SF_D1DIV | SF_AXPY)   \
  X(kResid | SF_D2DIV | SF_A_POW)                       \
  X(kResid | SF_AXPY | SF_A_POW)                        \
  X(SF_IN_MASKED | SF_AXPY | SF_A_POW)
#define BSP_STIFF_SHAPES(X) X(0) BSP_STIFF_SHAPES_MASKED(X)
#define BSP_STIFF_SHAPES_TMA(X)                                   \
  X(0)                                                            \
  BSP_STIFF_SHAPES_MASKED(X)                                      \
  X(kResid | SF_AXPY | SF_BASE_U)                                 \
  X(kResid | SF_AXPY | SF_BASE_U | SF_A_POW)                      \
  X(SF_IN_MASKED | SF_SUB_LOAD | SF_D1DIV | SF_AXPY | SF_BASE_U)             \
  X(SF_IN_MASKED | SF_SUB_LOAD | SF_D1DIV | SF_AXPY | SF_BASE_U | SF_PROLONG)  \
  X(kResid | SF_D2DIV | SF_A_POW | SF_SUM_SENS)                               \
  X(kResid | SF_AXPY | SF_BASE_U | SF_A_POW | SF_SUM_SENS)                    \
  X(kResid | SF_SUM_SENS)                                                     \
  X(SF_IN_MASKED | SF_REDUCE | SF_RED_NOMAX)                                  \
  X(SF_IN_MASKED | SF_REDUCE | SF_RED_NOMAX | SF_RED_NOS0)                    \
  X(SF_IN_MASKED | SF_REDUCE | SF_REDUCE_DOT | SF_RED_NOMAX | SF_RED_NOS0)

struct StiffArgs {
  GridView g;
  const double* a;         // [E] activation
  const double2* u;        // [N] input
  const double* in_div;    // nullable device scalar: u_eff = u / in_div
  const double2* rhs;      // nullable: SF_SUB_LOAD subtracts rhs instead of the grid load
  double2* out;            // [N] output (nullable)
  const double2* base;     // SF_AXPY base vector
  double beta;             // SF_AXPY coefficient
  const double2* dotv;     // nullable: reduce dot(dotv/dot_div, Ku)
  const double* dot_div;   // nullable device scalar
  const double* vp;        // SF_ENERGY: physical density (nullable -> prefactor 1)
  double eta;
  double* sens;            // SF_ENERGY output [E]
  RedBuf rb;
  double* red_out;         // HK_STORE target [4]
  DevState* st;
  int hook, hook_i;
  const int* gate0;        // nullable: skip when *gate0 != 0
  const int* gate1;
  int flags;
  int R;                   // element rows per strip
  int red_need;            // SF_REDUCE totals the caller reads: bit 0 u.Ku, 1 |t|^2,
                           // 2 dot, 3 max|t|; 0 = all (launch_stiff maps it to SF_RED_*)
  int red_y0, red_y1;      // SF_REDUCE covers node rows [red_y0, red_y1) (row slabs)
  const double2* pc;       // SF_PROLONG: the coarse-level vector ((nxc + 1) x (nyc + 1) nodes)
  int nxc, nyc;
};

// Finalisation of the solver's residual reduction (solvers.py:447-455):
// compliance, residual_inf, divergence flag and the Krylov start norm from the
// grid totals tot = (u.Ku, |r|^2, dot, max|r|).  Shared by the in-kernel hook
// and the row-slab path (after the all-gather of per-rank totals).
template <class State>
BSP_DEV void residual_hook(State* st, const double* tot) {
  const double comp = 0.5 * tot[0];
  // the kernels' maxima skip NaNs; a NaN anywhere made |r|^2 (tot[1]) NaN
  const double rinf = tot[1] != tot[1] ? tot[1] : tot[3];
  st->compliance = comp;
  st->res_inf = rinf;
  const double nb = sqrt(tot[1]);
  st->rnorm = nb;
  st->norms[0] = nb;
  st->kry_count = 0;
  st->kry_stop = (nb == 0.0) ? 1 : 0;
  if (!(isfinite(rinf) && isfinite(comp))) {
    st->done = 2;
    st->div_k = st->k;
  }
}

}  // namespace bsp
