/* bisimp_b200.h — C ABI of the B200-native bilevel-SIMP hot path.
 *
 * Drop-in boundary for the per-iteration hot path of the reference package
 * `bisimp` (arXiv 2204.06204, /root/reference/pkg/src/bisimp).  The reference
 * is pure Python (numpy/scipy) with no FFI layer of its own; its callers
 * (cli._execute, cli.py:73; Session._run_worker, service/sessions.py:106-107)
 * call `bisimp.solvers.run` and the L2 numerical functions directly.  This
 * header is what a ctypes/cffi binding of that path binds: every entry point
 * below names the reference function it replaces (file:line).  The Python
 * package `paper_2204_06204_b200` is exactly such a binding (see
 * INTEGRATION.md).
 *
 * Conventions
 *  - All arrays are fp64, C-contiguous.  Element e = ey*nx+ex; node
 *    j = y*(nx+1)+x; DOFs 2j (ux), 2j+1 (uy) interleaved (fea.py:8-11).
 *  - Pointers named d_* are DEVICE pointers (cudaMalloc / torch CUDA tensors);
 *    h_* are HOST pointers.  `stream` is a cudaStream_t (NULL = legacy stream).
 *  - Device ops are stream-ordered and asynchronous unless they return a host
 *    scalar.  Inputs are never modified; outputs are caller-owned.
 *  - A bsp_grid / bsp_solver is not reentrant: use one host thread (or one
 *    stream) per handle at a time.
 *  - Return codes: BSP_OK or an error; bsp_last_error() gives the message of
 *    the calling thread's last failure.  Error classes map to the reference's
 *    exceptions: BSP_EINVAL -> ValueError, BSP_ENONFINITE -> DivergenceError
 *    (solvers.py:450-455), BSP_ESOLVE -> LinearSolveError (fea.py:272-275).
 */
#ifndef BISIMP_B200_H
#define BISIMP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BSP_OK 0
#define BSP_EINVAL 1
#define BSP_ENONFINITE 2
#define BSP_ECUDA 3
#define BSP_ENOMEM 4
#define BSP_EUNSUPPORTED 5
#define BSP_ESOLVE 6

/* low-level algorithms (solvers.py:40, ALGORITHMS) + north-star extensions */
#define BSP_ALGO_FBTO 0          /* u - beta r                      (solvers.py:273-274) */
#define BSP_ALGO_PFBTO_JACOBI 1  /* u - beta K (r / diag^2)         (solvers.py:275-278) */
#define BSP_ALGO_CPFBTO_KRYLOV 2 /* u - beta krylov_apply(r)        (solvers.py:279-280) */
#define BSP_ALGO_PGD_EXACT 3     /* exact_solve every iteration     (solvers.py:445-446) */
/* North-star approximate inverses without a reference implementation
 * (SURVEY §8(a')): u - beta M~^{-1} r, the contraction lemma's "any
 * preconditioner" with beta = 1 by default. */
#define BSP_ALGO_PCG_JACOBI 4    /* u - beta PCG_k(K(a), r), Jacobi preconditioner */
#define BSP_ALGO_MG_VCYCLE 5     /* u - beta V(r), one geometric-multigrid V-cycle   */
#define BSP_ALGO_MG_PCG 6        /* u - beta PCG_k(K(a), r), V-cycle preconditioner  */

const char* bsp_last_error(void);
int bsp_version(void);

/* ---------------------------------------------------------------- grid ---- */
typedef struct bsp_grid bsp_grid;

/* GridModel (fea.py:104-143) resident on the current CUDA device.
 * h_ke: 8x8 row-major element stiffness (element_stiffness, fea.py:61-87);
 * h_fixed: n_dofs bytes (0/1) fixed-DOF mask; h_load: n_dofs load vector. */
int bsp_grid_create(int nx, int ny, const double* h_ke, const uint8_t* h_fixed,
                    const double* h_load, bsp_grid** out);
/* The same grid from index lists (problems.resolve, problems.py:138-164, as
 * O(boundary) lists): n_fixed fixed DOF indices and n_load (DOF, value)
 * pairs, scattered on the device.  For grids of 10^8 DOFs this avoids the
 * O(n) host arrays and their upload. */
int bsp_grid_create_sparse(int nx, int ny, const double* h_ke, long long n_fixed,
                           const long long* h_fixed_dofs, long long n_load,
                           const long long* h_load_dofs, const double* h_load_vals,
                           bsp_grid** out);
int bsp_grid_destroy(bsp_grid* g);
/* n_dofs, n_elements, flags (bit0: isotropic mode structure, bit1: uniform diag) */
int bsp_grid_info(const bsp_grid* g, long long* n_dofs, long long* n_elem, int* flags);

/* apply_stiffness(grid, a, u) -> y   (fea.py:150-181) */
int bsp_apply_stiffness(bsp_grid* g, const double* d_a, const double* d_u, double* d_y,
                        void* stream);
/* Same product for an input already zero on the fixed DOFs (every vector
 * the solver produces is); skips the input masking.  Results are undefined if
 * d_u is non-zero on a fixed DOF. */
int bsp_apply_stiffness_premasked(bsp_grid* g, const double* d_a, const double* d_u, double* d_y,
                                  void* stream);
/* stiffness_diagonal(grid, a) -> d   (fea.py:184-189) */
int bsp_stiffness_diagonal(bsp_grid* g, const double* d_a, double* d_d, void* stream);
/* element_energies(grid, u) -> e     (fea.py:197-201) */
int bsp_element_energies(bsp_grid* g, const double* d_u, double* d_e, void* stream);
/* r = K(a)u - f with h_out[4] = {u.Ku, |r|^2, 0, max|r|} (solvers.py:447-449;
 * compliance_energy fea.py:192-194 is 0.5*h_out[0]).  Synchronous. */
int bsp_residual(bsp_grid* g, const double* d_a, const double* d_u, double* d_r,
                 double* h_out, void* stream);
/* sensitivity(grid, v_phys, u, eta, filter) -> g   (solvers.py:181-190) */
int bsp_sensitivity(bsp_grid* g, const double* d_vphys, const double* d_u, double eta,
                    const double* h_taps, int n_taps, double* d_out, void* stream);
/* estimate_rho_max (fea.py:278-301): d_x0 = the seeded start vector already
 * masked and normalised on the host; synchronous, returns rho in *h_rho. */
int bsp_estimate_rho_max(bsp_grid* g, const double* d_a, const double* d_x0, int iters,
                         double* h_rho, void* stream);
/* _estimate_squared_jacobi_rho (solvers.py:348-364) on K M^-2 K at activation a */
int bsp_estimate_sqjacobi_rho(bsp_grid* g, const double* d_a, const double* d_x0, int iters,
                              double* h_rho, void* stream);
/* krylov_apply(grid, a, b, dim) -> out   (solvers.py:222-255); synchronous;
 * h_rank (nullable) receives the LSQ rank after the 1e-13 cut. */
int bsp_krylov_apply(bsp_grid* g, const double* d_a, const double* d_b, int dim, double* d_out,
                     int* h_rank, void* stream);
/* low_level_step(grid, a, u, config, beta, residual) -> u_next  (solvers.py:258-281);
 * d_residual nullable (then r = K(a)u - f). */
int bsp_low_level_step(bsp_grid* g, int algorithm, const double* d_a, const double* d_u,
                       double beta, const double* d_residual, int krylov_dim, double* d_out,
                       void* stream);
/* exact_solve(grid, a, tol, x0) -> u   (fea.py:230-275): restarted
 * multigrid-preconditioned CG to |K u - f|_inf <= tol (the reference's
 * SuperLU + refinement postcondition); d_x0 nullable.  Synchronous.
 * BSP_ESOLVE if max_iters CG steps cannot reach tol. */
int bsp_exact_solve(bsp_grid* g, const double* d_a, double tol, const double* d_x0,
                    long long max_iters, double* d_u, void* stream);

/* ----------------------------------------------------- filter / design ---- */
/* apply_filter / apply_filter_adjoint (filtering.py:46-72).  h_taps: the
 * n_taps (odd, <= 31) normalised Gaussian weights of gaussian_weights()
 * (filtering.py:30-35), computed by the caller; d_act (nullable, forward
 * only) receives out**eta (solvers.py:443). */
int bsp_filter(const double* d_in, double* d_out, double* d_act, double eta, int nx, int ny,
               const double* h_taps, int n_taps, int adjoint, void* stream);
/* mean_project(g) (solvers.py:193-197) */
int bsp_mean_project(const double* d_g, long long n, double* d_out, void* stream);
/* project_simplex(v, bounds) (projection.py:50-91); bounds validated here. */
int bsp_project_simplex(const double* d_v, long long n, double lo, double hi, double budget,
                        double* d_out, void* stream);
/* high_level_step(v, g, alpha_k, bounds, active, mean_projection) (solvers.py:284-302);
 * d_active: nullable byte mask (1 = active); budget refers to active entries. */
int bsp_high_level_step(const double* d_v, const double* d_g, long long n, double alpha,
                        double lo, double hi, double budget, const uint8_t* d_active,
                        int mean_projection, double* d_out, void* stream);

/* --------------------------------------------- density frames (f)3 ---- */
/* v_phys -> little-endian float32 frame (service/sessions.py:97,
 * `v_phys.astype("<f4").tobytes()`; round-to-nearest-even, byte-identical). */
int bsp_density_frame(const double* d_vphys, long long E, float* d_out, void* stream);
/* v_phys -> PGM pixels floor(255(1 - v) + 0.5) as uint8 (outputs.py:21-30,
 * byte-identical).  d_bad (nullable device int, zeroed by the caller) is
 * OR-ed with 1 when any value lies outside [0, 1] (outputs.py:25-26). */
int bsp_density_pixels(const double* d_vphys, long long E, uint8_t* d_out, int* d_bad,
                       void* stream);

/* ------------------------------------------- approximate inverses (a') ---- */
/* Geometric multigrid hierarchy over a grid (no reference implementation;
 * SURVEY §8(a')).  Level l+1 halves each axis (ceil) down to <= 40 nodes;
 * rediscretised coarse activation (mean of the 4 children), bilinear
 * prolongation P masked on both sides, R = P^T, a coarse DOF is fixed iff a
 * fine DOF of the same component in its prolongation footprint is fixed;
 * damped-Jacobi smoothing; dense direct solve on the coarsest level. */
typedef struct bsp_mg bsp_mg;
int bsp_mg_create(bsp_grid* g, int max_levels, bsp_mg** out);
int bsp_mg_destroy(bsp_mg* mg);
/* *levels = number of levels incl. the fine grid; *coarse_dofs = coarsest n */
int bsp_mg_info(const bsp_mg* mg, int* levels, int* coarse_dofs);
/* dimensions and (nullable) fixed-DOF mask (n_l bytes) of one level */
int bsp_mg_level(const bsp_mg* mg, int level, int* nx, int* ny, uint8_t* h_fixed);
/* coarse activations + coarsest inverse for activation d_a (kept by pointer) */
int bsp_mg_setup(bsp_mg* mg, const double* d_a, void* stream);
/* d_x = V(d_b): one V-cycle (nu pre/post sweeps, weight omega) */
int bsp_mg_vcycle(bsp_mg* mg, const double* d_b, double* d_x, double omega, int nu, void* stream);
/* d_out = d_base - beta * x, x = `steps` preconditioned-CG iterations from 0 on
 * K(a) x = b (Jacobi if mg == NULL, else one V-cycle per step; steps == 0
 * applies the preconditioner once).  d_base nullable (= 0).  Runs bsp_mg_setup
 * itself when mg != NULL. */
int bsp_pcg_apply(bsp_grid* g, bsp_mg* mg, const double* d_a, const double* d_b, int steps,
                  double omega, int nu, const double* d_base, double beta, double* d_out,
                  void* stream);

/* ------------------------------------------------------ seeded start ---- */
/* numpy's normal stream on the device: d_out[0..n) =
 * np.random.default_rng(seed).standard_normal(n) (PCG64 + numpy's ziggurat;
 * the reference's power-iteration start, fea.py:289-292, solvers.py:352-355).
 * h_state = the PCG64 state after SeedSequence seeding: {state lo, state hi,
 * inc lo, inc hi} (numpy's PCG64(seed).state).  Bit-identical to numpy except
 * that a tail sample (|x| > 3.65, ~1 in 3800) uses CUDA's log1p. */
int bsp_standard_normal(const uint64_t* h_state, long long n, double* d_out, void* stream);
/* The start vector itself: standard_normal(n_dofs), fixed DOFs zeroed,
 * scaled to unit 2-norm (fea.py:289-292). */
int bsp_start_vector(bsp_grid* g, const uint64_t* h_state, double* d_x, void* stream);

/* -------------------------------------------------------------- solver ---- */
/* The body of run()'s outer loop (solvers.py:416-475) resident on the GPU:
 * one iteration = filter+activation, residual+reductions+energies, filter
 * adjoint, low-level step, projected high-level step + record.  Iterations
 * are captured once into CUDA graphs and replayed; termination and
 * divergence are decided on the device. */
typedef struct bsp_solver bsp_solver;

typedef struct bsp_solver_config {
  size_t struct_size;     /* sizeof(bsp_solver_config) as the CALLER compiled it: the
                             ABI version.  Must be >= BSP_SOLVER_CONFIG_MIN_SIZE; fields
                             past struct_size take their defaults (below), so a caller
                             built against an older header keeps working. */
  int algorithm;          /* BSP_ALGO_* (not PGD_EXACT) */
  double eta;             /* SIMP exponent (problems.py:82) */
  int n_taps;             /* FilterSpec.size (filtering.py:20), any odd size >= 1 */
  const double* taps;     /* n_taps weights gaussian_weights(FilterSpec)
                             (filtering.py:30-35), host memory, copied at create */
  double v_lo, v_hi;      /* SimplexBounds v_lo / v_hi */
  double budget;          /* SimplexBounds v_bar */
  double beta;            /* low-level step size (resolved by the caller) */
  int krylov_dim;         /* SolverConfig.krylov_dim (any >= 1) */
  double tol_dv, tol_res; /* termination (solvers.py:473) */
  int mean_projection;
  int max_batch;          /* max iterations per bsp_solver_run call */
  /* ---- optional (defaults when struct_size ends before them) ---------- */
  /* BSP_ALGO_PCG_JACOBI / MG_VCYCLE / MG_PCG only: */
  int inner_steps;        /* CG steps per outer iteration (0: one preconditioner
                             application; < 0 or absent: 20 for PCG_JACOBI, 4 for
                             MG_PCG, 0 for MG_VCYCLE) */
  double mg_omega;        /* damped-Jacobi smoother weight (absent: 0.6) */
  int mg_nu;              /* smoother sweeps before and after the coarse correction
                             (absent: 2) */
  int mg_levels;          /* max multigrid levels (<= 0 or absent: as many as the grid
                             allows) */
} bsp_solver_config;

/* The fields every caller must provide: up to and including max_batch. */
#define BSP_SOLVER_CONFIG_MIN_SIZE \
  (offsetof(bsp_solver_config, max_batch) + sizeof(int))

#define BSP_FRAME_F32 0
#define BSP_FRAME_PGM 1

#define BSP_ST_RUNNING 0
#define BSP_ST_CONVERGED 1
#define BSP_ST_DIVERGED 2
/* 4: stopped because krylov_dim > 62 met a basis that is numerically full
 * rank past the 63 powers the TSQR holds (never seen: the rank cut falls
 * near column 21) */
#define BSP_ST_UNSUPPORTED 4

/* h_active: nullable E-byte mask (passive regions); h_v0: initial design (E). */
int bsp_solver_create(bsp_grid* g, const bsp_solver_config* cfg, const uint8_t* h_active,
                      const double* h_v0, bsp_solver** out);
int bsp_solver_destroy(bsp_solver* s);
/* Run iterations k_first .. k_first+n_iters-1 (k_first must be the next
 * iteration).  h_alphas[i] = alpha_k for k = k_first+i (SolverConfig.step_size,
 * solvers.py:100-102).  h_rec receives n_iters rows of
 * {compliance, residual_inf, dv_inf, volume} (ConvergenceRecord columns,
 * solvers.py:120-146).  *h_done = iterations completed; *h_status =
 * BSP_ST_*; on divergence *h_status = BSP_ST_DIVERGED and h_rec[*h_done]
 * holds {compliance, residual_inf} of the failing iteration. */
int bsp_solver_run(bsp_solver* s, long long k_first, int n_iters, const double* h_alphas,
                   double* h_rec, int* h_done, int* h_status);
/* The three stages of bsp_solver_run, for callers that time or interleave
 * iterations: stage the step sizes of iterations k_base..k_base+n-1 (async;
 * k_base must be the next iteration), enqueue iteration k (one CUDA-graph
 * replay, async; k must be the next iteration and lie in the staged window,
 * else BSP_EINVAL), then read back the records of k_first..k_first+n_iters-1
 * and synchronise. */
int bsp_solver_set_alphas(bsp_solver* s, long long k_base, int n, const double* h_alphas);
int bsp_solver_launch(bsp_solver* s, long long k);
int bsp_solver_finish(bsp_solver* s, long long k_first, int n_iters, double* h_rec, int* h_done,
                      int* h_status);
/* Copy a state field of the LAST COMPLETED iteration to the host:
 * 0 u (measured, iterate k), 1 v (iterate k), 2 v_phys, 3 activation,
 * 4 u_next (k+1), 5 v_next (k+1). */
int bsp_solver_read(bsp_solver* s, int field, double* h_out);
/* The sink's state of the last completed iteration (solvers.py:367-378): u, v,
 * v_phys, activation in one call (pinned staging, one synchronisation). */
int bsp_solver_read_state(bsp_solver* s, double* h_u, double* h_v, double* h_vp, double* h_a);
/* Density frame of the last completed iteration, converted on the device
 * (SURVEY §8(f)3): kind BSP_FRAME_F32 writes E little-endian float32 values of
 * v_phys (the service frame payload, service/sessions.py:97); BSP_FRAME_PGM
 * writes the E PGM pixels floor(255(1 - v_phys) + 0.5) (outputs.py:21-30) and
 * returns BSP_EINVAL when a density lies outside [0, 1] (outputs.py:25-26).
 * Moves 4E or E bytes instead of the 8(n + 3E) of bsp_solver_read_state. */
int bsp_solver_read_frame(bsp_solver* s, int kind, void* h_out);
/* One iteration through HOST buffers (the e2e drop-in call): uploads v, u,
 * runs iteration k with step alpha, downloads v_next, u_next and the record
 * row {compliance, residual_inf, dv_inf, volume}.  Returns BSP_ENONFINITE on
 * a non-finite residual. */
int bsp_solver_step_host(bsp_solver* s, long long k, double alpha, const double* h_v,
                         const double* h_u, double* h_v_next, double* h_u_next,
                         double* h_rec4);
/* Device-clock stamps (%globaltimer, ns) of the first n record rows read by
 * the last bsp_solver_run / bsp_solver_finish: the moment each iteration's
 * record row was written on the device.  run(..., clock=time.perf_counter)
 * maps them onto the caller's clock instead of synchronising per iteration. */
int bsp_solver_stamps(bsp_solver* s, int n, long long* h_ns);
/* The device's %globaltimer now (ns), read by a one-thread kernel on `stream`
 * (synchronises it): the calibration point of bsp_solver_stamps. */
int bsp_device_clock(void* stream, long long* h_ns);
/* Device-time breakdown/diagnostics: h_out[0] = 1 if iterations replay as
 * CUDA graphs, h_out[1] = kernels per iteration, h_out[2] = last lambda
 * rounds, h_out[3] = last Krylov rank. */
int bsp_solver_info(bsp_solver* s, double* h_out);
/* The stream the solver runs on (cudaStream_t), for event timing. */
void* bsp_solver_stream(bsp_solver* s);

/* ------------------------------------------------ row slabs (multi-GPU) ---- */
/* The outer loop of run() (solvers.py:416-475) with the grid split into row
 * slabs across ranks: rank r owns element rows [e0, e1) of a
 * balanced split and stores the window [e0 - H, e1 + H) (H = filter radius
 * + 1).  Per iteration: 3 all-gathers of 8-double partial totals (summed in
 * rank order on every rank: identical, deterministic scalars) and 2 grouped
 * NCCL halo exchanges.  fbto, pfbto_jacobi, pcg_jacobi (per CG step: one
 * halo exchange of p, two all-gathered dot products), mg_pcg (the same CG with
 * a block-Jacobi multigrid preconditioner: one V-cycle per rank on the
 * principal submatrix of its owned node rows) and cpfbto_krylov (per
 * power: one halo exchange and an all-gathered norm; per iteration one
 * all-gather of the ranks' TSQR factors).  An active volume budget (rare)
 * ends the batch; the host then runs the lambda search with one all-gather per
 * round.  The reference has no distributed code. */
typedef struct bsp_dist bsp_dist;
/* NCCL unique id (ncclUniqueId bytes, *nbytes = 128) for rank 0 to broadcast */
int bsp_nccl_unique_id(uint8_t* out, int* nbytes);
/* owned element rows [e0, e1) and window [w0, w1) of `rank` */
int bsp_dist_slab_rows(int ny, int world, int rank, int halo, int* e0, int* e1, int* w0, int* w1);
/* nccl_id == NULL: local transport, all `world` slabs in this process (host
 * arrays are then global); else one slab per process (host arrays = this rank's
 * window: node rows [w0, w1], element rows [w0, w1)).  n_active = global count
 * of active elements; cfg->budget global. */
int bsp_dist_create(int nx, int ny, int world, int rank, const uint8_t* nccl_id,
                    const double* h_ke, const uint8_t* h_fixed, const double* h_load,
                    const bsp_solver_config* cfg, const uint8_t* h_active, double n_active,
                    const double* h_v0, bsp_dist** out);
int bsp_dist_destroy(bsp_dist* d);
/* fbto / pfbto created with cfg.beta <= 0: beta = 1/rho of the set-up power
 * iteration (reference solvers.py:334-364, fea.py:278-301) computed ON THE
 * SLABS -- halo-exchanged inputs, owned-row partials all-gathered and summed in
 * rank order -- instead of on the full grid by every rank.  d_normals: the
 * seeded standard normals of the GLOBAL grid on this rank's device (the
 * reference's start vector before masking and normalisation).  Captures the
 * iteration graphs; bsp_dist_run refuses to run before it. */
int bsp_dist_estimate_beta(bsp_dist* d, const double* d_normals, int iters, double* h_rho);
/* same contract as bsp_solver_run */
int bsp_dist_run(bsp_dist* d, long long k_first, int n_iters, const double* h_alphas,
                 double* h_rec, int* h_done, int* h_status);
/* owned rows of field 0 u, 1 v, 2 v_phys, 3 activation of the last completed
 * iteration (local transport: the global array) */
int bsp_dist_read(bsp_dist* d, int field, double* h_out);
/* h_out[0] graphs, [1] host lambda iterations, [2] lambda rounds, [3] H, [4] slabs here */
int bsp_dist_info(bsp_dist* d, double* h_out);
/* h_ms[0] = one end-of-iteration halo exchange, h_ms[1] = one all-gather (ms, device) */
int bsp_dist_comm_bench(bsp_dist* d, int iters, double* h_ms);
void* bsp_dist_stream(bsp_dist* d);

#ifdef __cplusplus
}
#endif
#endif /* BISIMP_B200_H */
