// Geometric multigrid V-cycle and preconditioned-CG approximate inverses
// (north-star subsystems with no reference implementation, SURVEY §8(a')).
//
// Hierarchy: level 0 is the caller's grid.  Level l+1 has ceil(nx_l/2) x
// ceil(ny_l/2) elements, stops at <= kCoarseNodes nodes.  Each level is a
// bsp_grid with the same element stiffness (2-D Q4 stiffness is scale
// invariant), a rediscretised activation a_{l+1} = mean of the 4 children
// (virtual children outside the grid count as 0), and a fixed mask where a
// coarse DOF is fixed iff a fine DOF of the same component inside its
// prolongation footprint is fixed.  P = bilinear interpolation masked on both
// sides, R = P^T.  Smoother: damped Jacobi (omega, nu sweeps pre and post, the
// first pre-sweep from zero), so the V-cycle is a symmetric operator.  The
// coarsest level is solved directly with an explicit dense inverse rebuilt
// once per activation (bsp_mg_setup).
#pragma once
#include <vector>

#include "grid.cuh"

namespace bsp {
constexpr int kCoarseNodes = 40;   // coarsest level: <= 40 nodes (80 DOFs)
constexpr int kMaxLevels = 24;
}  // namespace bsp

struct bsp_mg {
  bsp_grid* g0 = nullptr;             // level 0 (not owned)
  int L = 0;                          // coarse levels 1..L
  std::vector<bsp_grid*> lv;          // lv[0] = g0; lv[l>=1] owned
  std::vector<double*> a;             // a[0] = activation of the last setup (not owned)
  std::vector<double*> B, X, Y, T;    // per-level rhs / iterate / ping-pong / residual
  double* Ainv = nullptr;             // coarsest dense inverse (nc x nc)
  double* ke = nullptr;               // device copy of the 8x8 element stiffness
  int nc = 0;                         // coarsest DOFs
  // setup runs on a side stream (forked from the caller's stream, joined by
  // the next V-cycle before level 1 / the coarse solve), so the coarse
  // inverse overlaps the fine-level sweeps
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_coarse = nullptr, ev_factor = nullptr;
  bool wait_coarse = false, wait_factor = false;
};

namespace bsp {
// coarse activation, restriction, prolongation, Jacobi start, coarsest solve
int mg_setup_enqueue(bsp_mg* mg, const double* a0, const int* gate, cudaStream_t s);
// out0 = V(b0); b0 zero on the fixed DOFs; out0 must not alias b0 or mg buffers
int mg_vcycle_enqueue(bsp_mg* mg, const double* b0, double* out0, double omega, int nu,
                      const int* gate, cudaStream_t s);

// Preconditioned CG, `steps` iterations from x = 0 on K(a) x = b (b zero on
// the fixed DOFs), then out = base - beta * x (base nullable -> 0).
// mg == nullptr -> Jacobi preconditioner.  `R` may alias b (then b is
// consumed).  The workspace is owned by the grid (ensure_pcg).
struct PcgWork {
  double *X = nullptr, *R = nullptr, *P = nullptr, *Q = nullptr, *Z = nullptr, *D = nullptr;
  double* sc = nullptr;  // device scalars: [0] rz, [1..4] HK_STORE (p.Kp ...), [5] rz', [6] beta
  unsigned* cnt = nullptr;
  double* part = nullptr;
  long long n = 0;
};
int pcg_enqueue(bsp_grid* g, PcgWork& w, bsp_mg* mg, const double* a, const double* b, int steps,
                double omega, int nu, const double* base, double beta, double* out,
                const int* gate, cudaStream_t s, bool setup = true);
int pcg_alloc(PcgWork& w, bsp_grid* g, bool with_mg);
// PCG kernels (pcg.cu); `defer` (row slabs): store this rank's partial sum
// there instead of finalising sc[]
__global__ void k_pcg_init_jacobi(const double* b, double* R, double* P, const double* D,
                                  double* sc, RedBuf rb, long long n, const int* gate,
                                  double* defer);
cudaError_t launch_pcg_update(unsigned blocks, cudaStream_t s, double* X, double* R,
                              const double* P, const double* Q, const double* D, double* sc,
                              RedBuf rb, long long n, int first, int last, const double* base,
                              double beta, double* out, const int* gate, double* defer);
__global__ void k_pcg_dir(double* P, const double* R, const double* D, const double* Z,
                          const double* sc, long long n, const int* gate);
__global__ void k_pcg_init_z(const double* b, double* R, const double* Z, double* P, double* sc,
                             RedBuf rb, long long n, const int* gate, double* defer);
__global__ void k_pcg_rz(const double* R, const double* Z, double* sc, RedBuf rb, long long n,
                         const int* gate, double* defer);
__global__ void k_mask_copy(const double* x0, const uint32_t* fixbits, double* x, long long n);
void pcg_free(PcgWork& w);
}  // namespace bsp
