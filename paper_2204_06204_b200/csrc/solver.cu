// Device-resident outer loop of run() (reference solvers.py:416-475) and the
// Jacobi-PCG exact solve (fea.py:230-275 contract).
//
// One iteration k (parity p = (k-1)&1 selects the ping-pong buffers):
//   1 k_filter_fwd      v[p] -> v_phys, a = v_phys^eta            (solvers.py:442-443)
//   2 k_stiff RESIDUAL  r = K(a)u[p] - f, max|r|, u.Ku, |r|^2,
//                       energies*eta*v_phys^(eta-1) -> sens,
//                       + fused low-level epilogue (fbto: u[1-p] = u - beta r;
//                       pfbto: z = r/diag^2; cpfbto: q_0 = r)         (447-457)
//   3 k_filter_adj      sens -> g                                   (457)
//   4 low level         pfbto: u[1-p] = u - beta K z ; cpfbto: 21 power
//                       kernels + TSQR + combine                      (460)
//   5 k_highlevel       mean projection, projection, dv_inf, volume,
//                       record row, termination, k++                 (462-475)
// Each parity's sequence is captured once into a CUDA graph; a batch of
// iterations is a chain of graph launches with no host synchronisation.
// Divergence (non-finite residual) and convergence gate every later kernel.
#include <algorithm>
#include <cstring>
#include <vector>

#include "grid.cuh"
#include "highlevel.cuh"
#include "krylov.cuh"
#include "misc.cuh"

using namespace bsp;

namespace bsp {
int krylov_enqueue(bsp_grid* g, const double* d_a, const double* d_b, int dim, const double* d_base,
                   double beta, double* d_out, double* Q, bool b_in_Q0, const int* gate,
                   cudaStream_t s);
}

struct bsp_solver {
  bsp_grid* g = nullptr;
  bsp_solver_config cfg{};
  FilterTaps taps{};
  cudaStream_t s = nullptr;
  double* u[2] = {nullptr, nullptr};
  double* v[2] = {nullptr, nullptr};
  double* vp = nullptr;
  double* a = nullptr;
  double* sens = nullptr;
  double* gr = nullptr;
  double* z = nullptr;       // pfbto z = r/d^2
  double* Q = nullptr;       // Krylov basis (npow+1) x n, q_0 = r
  uint8_t* active = nullptr;
  double n_active = 0.0;
  double* alphas = nullptr;  // [max_batch]
  RecRow* rec = nullptr;     // [max_batch]
  double* h_alphas = nullptr;
  RecRow* h_rec = nullptr;
  DevState* h_st = nullptr;
  double* hl_part = nullptr;
  int hl_blocks = 0;
  cudaGraphExec_t exec[2] = {nullptr, nullptr};
  bool graphs = false;
  int kernels_per_iter = 0;
  long long last_k = 0;  // last completed iteration
};

static int enqueue_iteration(bsp_solver* S, int p, cudaStream_t s) {
  bsp_grid* g = S->g;
  const bsp_solver_config& c = S->cfg;
  const int* gate = &g->st->done;
  int nk = 0;
  int rc = launch_filter(S->v[p], S->vp, S->a, c.eta, g->nx, g->ny, S->taps, 0, gate, s);
  if (rc) return rc;
  ++nk;
  StiffArgs r = stiff_args(g);
  r.a = S->a;
  r.u = (const double2*)S->u[p];
  r.flags = SF_SUB_LOAD | SF_REDUCE | SF_ENERGY | SF_IN_MASKED;  // u is masked by construction
  r.vp = S->vp;
  r.eta = c.eta;
  r.sens = S->sens;
  r.hook = HK_RESIDUAL;
  r.gate0 = gate;
  switch (c.algorithm) {
    case BSP_ALGO_FBTO:
      r.flags |= SF_AXPY;
      r.base = (const double2*)S->u[p];
      r.beta = c.beta;
      r.out = (double2*)S->u[1 - p];
      break;
    case BSP_ALGO_PFBTO_JACOBI:
      r.flags |= SF_D2DIV;
      r.out = (double2*)S->z;
      break;
    case BSP_ALGO_CPFBTO_KRYLOV:
      r.out = (double2*)S->Q;
      break;
    default:
      return set_error(BSP_EINVAL, "solver algorithm %d not supported", c.algorithm);
  }
  BSP_CU(launch_stiff(g, r, s));
  ++nk;
  // adjoint filter + sum of g over active elements (mean projection)
  rc = launch_filter(S->sens, S->gr, nullptr, 1.0, g->nx, g->ny, S->taps, 1, gate, s, g->st,
                     S->active, RedBuf{g->part, g->counter});
  if (rc) return rc;
  ++nk;
  if (c.algorithm == BSP_ALGO_PFBTO_JACOBI) {
    StiffArgs q = stiff_args(g);
    q.a = S->a;
    q.u = (const double2*)S->z;
    q.out = (double2*)S->u[1 - p];
    q.base = (const double2*)S->u[p];
    q.beta = c.beta;
    q.flags = SF_AXPY | SF_IN_MASKED;  // z = r/d^2 is zero on fixed DOFs
    q.gate0 = gate;
    BSP_CU(launch_stiff(g, q, s));
    ++nk;
  } else if (c.algorithm == BSP_ALGO_CPFBTO_KRYLOV) {
    rc = krylov_enqueue(g, S->a, S->Q, c.krylov_dim, S->u[p], c.beta, S->u[1 - p], S->Q, true,
                        gate, s);
    if (rc) return rc;
    int levels = 0;
    for (int nin = tsqr_leaves(g->n); nin > 1 || levels == 0; nin = (nin + tsqr_fan_in() - 1) / tsqr_fan_in())
      ++levels;
    nk += (int)std::min<long long>((long long)c.krylov_dim + 1, g->n) + 2 + levels;
  }
  HLArgs h{};
  h.v = S->v[p];
  h.g = S->gr;
  h.v_next = S->v[1 - p];
  h.active = S->active;
  h.E = g->E;
  h.n_active = S->n_active;
  h.lo = c.v_lo;
  h.hi = c.v_hi;
  h.budget = c.budget;
  h.alphas = S->alphas;
  h.mean_projection = c.mean_projection;
  h.tol_dv = c.tol_dv;
  h.tol_res = c.tol_res;
  h.rb = RedBuf{g->part, g->counter};
  h.part = S->hl_part;
  h.st = g->st;
  h.rec = S->rec;
  BSP_CU(launch_highlevel(h, S->hl_blocks, g->nsm, s));
  nk += 2;
  S->kernels_per_iter = nk;
  return BSP_OK;
}

static void free_solver(bsp_solver* S) {
  if (!S) return;
  for (int i = 0; i < 2; ++i) {
    if (S->exec[i]) cudaGraphExecDestroy(S->exec[i]);
    cudaFree(S->u[i]);
    cudaFree(S->v[i]);
  }
  cudaFree(S->vp);
  cudaFree(S->a);
  cudaFree(S->sens);
  cudaFree(S->gr);
  cudaFree(S->z);
  cudaFree(S->Q);
  cudaFree(S->active);
  cudaFree(S->alphas);
  cudaFree(S->rec);
  cudaFree(S->hl_part);
  if (S->h_alphas) cudaFreeHost(S->h_alphas);
  if (S->h_rec) cudaFreeHost(S->h_rec);
  if (S->h_st) cudaFreeHost(S->h_st);
  if (S->s) cudaStreamDestroy(S->s);
  delete S;
}

extern "C" int bsp_solver_destroy(bsp_solver* S) {
  if (S) cudaStreamSynchronize(S->s);
  free_solver(S);
  return BSP_OK;
}

extern "C" int bsp_solver_create(bsp_grid* g, const bsp_solver_config* cfg,
                                 const uint8_t* h_active, const double* h_v0, bsp_solver** out) {
  if (!g || !cfg || !h_v0 || !out) return set_error(BSP_EINVAL, "null argument");
  const bsp_solver_config& c = *cfg;
  if (c.algorithm < BSP_ALGO_FBTO || c.algorithm > BSP_ALGO_CPFBTO_KRYLOV)
    return set_error(BSP_EINVAL, "solver algorithm %d not supported on the device loop",
                     c.algorithm);
  if (c.algorithm == BSP_ALGO_PFBTO_JACOBI && !g->uniform_diag)
    return set_error(BSP_EUNSUPPORTED, "PFBTO needs a uniform ke diagonal");
  if (c.algorithm == BSP_ALGO_CPFBTO_KRYLOV && c.krylov_dim < 1)
    return set_error(BSP_EINVAL, "Krylov dimension must be at least 1");
  if (c.max_batch < 1) return set_error(BSP_EINVAL, "max_batch must be >= 1");
  bsp_solver* S = new bsp_solver();
  S->g = g;
  S->cfg = c;
  int rc = make_taps(c.taps, c.n_taps, S->taps);
  if (rc) {
    delete S;
    return rc;
  }
  const size_t nb = g->n * sizeof(double), eb = g->E * sizeof(double);
  const int npow = (int)std::min<long long>((long long)std::max(c.krylov_dim, 1) + 1, g->n);
  bool ok = cudaStreamCreateWithFlags(&S->s, cudaStreamNonBlocking) == cudaSuccess;
  for (int i = 0; i < 2 && ok; ++i)
    ok = cudaMalloc(&S->u[i], nb) == cudaSuccess && cudaMalloc(&S->v[i], eb) == cudaSuccess;
  ok = ok && cudaMalloc(&S->vp, eb) == cudaSuccess && cudaMalloc(&S->a, eb) == cudaSuccess &&
       cudaMalloc(&S->sens, eb) == cudaSuccess && cudaMalloc(&S->gr, eb) == cudaSuccess;
  if (ok && c.algorithm == BSP_ALGO_PFBTO_JACOBI) ok = cudaMalloc(&S->z, nb) == cudaSuccess;
  if (ok && c.algorithm == BSP_ALGO_CPFBTO_KRYLOV)
    ok = cudaMalloc(&S->Q, (size_t)(npow + 1) * nb) == cudaSuccess;
  S->hl_blocks = highlevel_blocks(g->device);
  ok = ok && cudaMalloc(&S->hl_part, 4ull * S->hl_blocks * sizeof(double)) == cudaSuccess &&
       cudaMalloc(&S->alphas, c.max_batch * sizeof(double)) == cudaSuccess &&
       cudaMalloc(&S->rec, c.max_batch * sizeof(RecRow)) == cudaSuccess &&
       cudaMallocHost(&S->h_alphas, c.max_batch * sizeof(double)) == cudaSuccess &&
       cudaMallocHost(&S->h_rec, c.max_batch * sizeof(RecRow)) == cudaSuccess &&
       cudaMallocHost(&S->h_st, sizeof(DevState)) == cudaSuccess;
  long long n_active = g->E;
  if (ok && h_active) {
    n_active = 0;
    for (long long e = 0; e < g->E; ++e) n_active += h_active[e] ? 1 : 0;
    ok = cudaMalloc(&S->active, g->E) == cudaSuccess &&
         cudaMemcpy(S->active, h_active, g->E, cudaMemcpyHostToDevice) == cudaSuccess;
  }
  if (!ok) {
    cudaGetLastError();
    free_solver(S);
    return set_error(BSP_ENOMEM, "solver allocation failed (n=%lld E=%lld)", g->n, g->E);
  }
  S->n_active = (double)n_active;
  if (c.algorithm == BSP_ALGO_CPFBTO_KRYLOV) {
    rc = ensure_tsqr(g);
    if (rc) {
      free_solver(S);
      return rc;
    }
  }
  // initial state: u = 0, v = v0, k = 1
  cudaMemsetAsync(S->u[0], 0, nb, S->s);
  cudaMemsetAsync(S->u[1], 0, nb, S->s);
  cudaMemcpyAsync(S->v[0], h_v0, eb, cudaMemcpyHostToDevice, S->s);
  std::memset(S->h_st, 0, sizeof(DevState));
  S->h_st->k = 1;
  S->h_st->k_base = 1;
  cudaMemcpyAsync(g->st, S->h_st, sizeof(DevState), cudaMemcpyHostToDevice, S->s);
  // capture one graph per parity
  S->graphs = true;
  for (int p = 0; p < 2 && S->graphs; ++p) {
    cudaGraph_t graph = nullptr;
    if (cudaStreamBeginCapture(S->s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      S->graphs = false;
      break;
    }
    rc = enqueue_iteration(S, p, S->s);
    cudaError_t e = cudaStreamEndCapture(S->s, &graph);
    if (rc != BSP_OK || e != cudaSuccess || !graph) {
      S->graphs = false;
      cudaGetLastError();
      if (graph) cudaGraphDestroy(graph);
      break;
    }
    e = cudaGraphInstantiate(&S->exec[p], graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      S->graphs = false;
      S->exec[p] = nullptr;
      cudaGetLastError();
    }
  }
  if (!S->graphs) {
    for (int p = 0; p < 2; ++p)
      if (S->exec[p]) {
        cudaGraphExecDestroy(S->exec[p]);
        S->exec[p] = nullptr;
      }
  }
  cudaError_t e = cudaStreamSynchronize(S->s);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    free_solver(S);
    return set_error(BSP_ECUDA, "solver create: %s", cudaGetErrorString(e));
  }
  *out = S;
  return BSP_OK;
}

static int launch_iter(bsp_solver* S, long long k) {
  const int p = (int)((k - 1) & 1);
  if (S->graphs) {
    BSP_CU(cudaGraphLaunch(S->exec[p], S->s));
    return BSP_OK;
  }
  return enqueue_iteration(S, p, S->s);
}

extern "C" int bsp_solver_set_alphas(bsp_solver* S, long long k_base, int n,
                                     const double* h_alphas) {
  if (!S || (n > 0 && !h_alphas)) return set_error(BSP_EINVAL, "null argument");
  if (n < 0 || n > S->cfg.max_batch)
    return set_error(BSP_EINVAL, "n %d outside [0, %d]", n, S->cfg.max_batch);
  // the pinned staging buffer may still feed an in-flight copy of the last batch
  BSP_CU(cudaStreamSynchronize(S->s));
  std::memcpy(S->h_alphas, h_alphas, n * sizeof(double));
  BSP_CU(cudaMemcpyAsync(S->alphas, S->h_alphas, n * sizeof(double), cudaMemcpyHostToDevice,
                         S->s));
  S->h_st->k_base = k_base;
  BSP_CU(cudaMemcpyAsync(&S->g->st->k_base, &S->h_st->k_base, sizeof(long long),
                         cudaMemcpyHostToDevice, S->s));
  return BSP_OK;
}

extern "C" int bsp_solver_launch(bsp_solver* S, long long k) {
  if (!S || k < 1) return set_error(BSP_EINVAL, "bad argument");
  return launch_iter(S, k);
}

extern "C" int bsp_solver_finish(bsp_solver* S, long long k_first, int n_iters, double* h_rec,
                                 int* h_done, int* h_status) {
  if (!S) return set_error(BSP_EINVAL, "null argument");
  if (n_iters < 0 || n_iters > S->cfg.max_batch)
    return set_error(BSP_EINVAL, "n_iters %d outside [0, %d]", n_iters, S->cfg.max_batch);
  bsp_grid* g = S->g;
  BSP_CU(cudaMemcpyAsync(S->h_rec, S->rec, n_iters * sizeof(RecRow), cudaMemcpyDeviceToHost, S->s));
  BSP_CU(cudaMemcpyAsync(S->h_st, g->st, sizeof(DevState), cudaMemcpyDeviceToHost, S->s));
  BSP_CU(cudaStreamSynchronize(S->s));
  const DevState& st = *S->h_st;
  long long done = st.k - k_first;
  if (done < 0) done = 0;
  if (done > n_iters) done = n_iters;
  S->last_k = st.k - 1;
  const int status = st.done;
  if (h_rec) {
    for (long long i = 0; i < done; ++i) {
      h_rec[4 * i + 0] = S->h_rec[i].compliance;
      h_rec[4 * i + 1] = S->h_rec[i].res_inf;
      h_rec[4 * i + 2] = S->h_rec[i].dv_inf;
      h_rec[4 * i + 3] = S->h_rec[i].volume;
    }
    if (status == BSP_ST_DIVERGED && done < n_iters) {
      h_rec[4 * done + 0] = st.compliance;
      h_rec[4 * done + 1] = st.res_inf;
    }
  }
  if (h_done) *h_done = (int)done;
  if (h_status) *h_status = status;
  return BSP_OK;
}

extern "C" int bsp_solver_run(bsp_solver* S, long long k_first, int n_iters,
                              const double* h_alphas, double* h_rec, int* h_done, int* h_status) {
  if (!S || !h_alphas) return set_error(BSP_EINVAL, "null argument");
  if (k_first != S->last_k + 1)
    return set_error(BSP_EINVAL, "k_first %lld is not the next iteration %lld", k_first,
                     S->last_k + 1);
  int rc = bsp_solver_set_alphas(S, k_first, n_iters, h_alphas);
  if (rc) return rc;
  for (int i = 0; i < n_iters; ++i) {
    rc = launch_iter(S, k_first + i);
    if (rc) return rc;
  }
  return bsp_solver_finish(S, k_first, n_iters, h_rec, h_done, h_status);
}

extern "C" int bsp_solver_read(bsp_solver* S, int field, double* h_out) {
  if (!S || !h_out) return set_error(BSP_EINVAL, "null argument");
  bsp_grid* g = S->g;
  const long long k = S->last_k;
  const int p = (int)(((k < 1 ? 1 : k) - 1) & 1);
  const double* src = nullptr;
  size_t bytes = 0;
  switch (field) {
    case 0: src = k < 1 ? S->u[0] : S->u[p]; bytes = g->n * 8; break;
    case 1: src = k < 1 ? S->v[0] : S->v[p]; bytes = g->E * 8; break;
    case 2: src = S->vp; bytes = g->E * 8; break;
    case 3: src = S->a; bytes = g->E * 8; break;
    case 4: src = k < 1 ? S->u[0] : S->u[1 - p]; bytes = g->n * 8; break;
    case 5: src = k < 1 ? S->v[0] : S->v[1 - p]; bytes = g->E * 8; break;
    default: return set_error(BSP_EINVAL, "unknown field %d", field);
  }
  BSP_CU(cudaMemcpyAsync(h_out, src, bytes, cudaMemcpyDeviceToHost, S->s));
  BSP_CU(cudaStreamSynchronize(S->s));
  return BSP_OK;
}

extern "C" int bsp_solver_step_host(bsp_solver* S, long long k, double alpha, const double* h_v,
                                    const double* h_u, double* h_v_next, double* h_u_next,
                                    double* h_rec4) {
  if (!S || !h_v || !h_u || k < 1) return set_error(BSP_EINVAL, "bad argument");
  bsp_grid* g = S->g;
  const int p = (int)((k - 1) & 1);
  BSP_CU(cudaMemcpyAsync(S->v[p], h_v, g->E * 8, cudaMemcpyHostToDevice, S->s));
  BSP_CU(cudaMemcpyAsync(S->u[p], h_u, g->n * 8, cudaMemcpyHostToDevice, S->s));
  S->h_alphas[0] = alpha;
  BSP_CU(cudaMemcpyAsync(S->alphas, S->h_alphas, sizeof(double), cudaMemcpyHostToDevice, S->s));
  std::memset(S->h_st, 0, sizeof(DevState));
  S->h_st->k = k;
  S->h_st->k_base = k;
  BSP_CU(cudaMemcpyAsync(g->st, S->h_st, sizeof(DevState), cudaMemcpyHostToDevice, S->s));
  int rc = launch_iter(S, k);
  if (rc) return rc;
  if (h_v_next)
    BSP_CU(cudaMemcpyAsync(h_v_next, S->v[1 - p], g->E * 8, cudaMemcpyDeviceToHost, S->s));
  if (h_u_next)
    BSP_CU(cudaMemcpyAsync(h_u_next, S->u[1 - p], g->n * 8, cudaMemcpyDeviceToHost, S->s));
  BSP_CU(cudaMemcpyAsync(S->h_rec, S->rec, sizeof(RecRow), cudaMemcpyDeviceToHost, S->s));
  BSP_CU(cudaMemcpyAsync(S->h_st, g->st, sizeof(DevState), cudaMemcpyDeviceToHost, S->s));
  BSP_CU(cudaStreamSynchronize(S->s));
  S->last_k = S->h_st->k - 1;
  if (h_rec4) {
    h_rec4[0] = S->h_rec[0].compliance;
    h_rec4[1] = S->h_rec[0].res_inf;
    h_rec4[2] = S->h_rec[0].dv_inf;
    h_rec4[3] = S->h_rec[0].volume;
  }
  if (S->h_st->done == BSP_ST_DIVERGED)
    return set_error(BSP_ENONFINITE, "non-finite iterate at iteration %lld", k);
  return BSP_OK;
}

extern "C" int bsp_solver_info(bsp_solver* S, double* h_out) {
  if (!S || !h_out) return set_error(BSP_EINVAL, "null argument");
  h_out[0] = S->graphs ? 1.0 : 0.0;
  h_out[1] = S->kernels_per_iter;
  h_out[2] = S->h_st->lam_rounds;
  h_out[3] = S->h_st->kry_rank;
  return BSP_OK;
}

extern "C" void* bsp_solver_stream(bsp_solver* S) { return S ? (void*)S->s : nullptr; }

// ------------------------------------------------------- exact solve (CG) ---
namespace bsp {
struct CgArgs {
  double* x;
  double* r;
  double* p;
  const double* q;
  const double* d;
  long long n;
  double* cg;  // [0] rz, [3] max|r|, [4] p.q, [9] beta
  RedBuf rb;
};

// r = -(Kx - f) (input in r), p = r/d, rz, max|r|
__global__ void k_cg_init(CgArgs a) {
  double rz = 0.0, m = -INFINITY, z0 = 0.0, z1 = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.n;
       i += (long long)gridDim.x * blockDim.x) {
    double ri = -a.r[i];
    a.r[i] = ri;
    double zi = ri / a.d[i];
    a.p[i] = zi;
    rz += ri * zi;
    m = nanmax(m, fabs(ri));
  }
  __shared__ double tot[4];
  if (grid_reduce4(a.rb, rz, z0, z1, m, tot) && threadIdx.x == 0) {
    a.cg[0] = tot[0];
    a.cg[3] = tot[3];
  }
}

// x += alpha p; r -= alpha q; rz_new = r.(r/d); beta = rz_new/rz
__global__ void k_cg_step(CgArgs a) {
  const double alpha = a.cg[0] / a.cg[4];
  double rz = 0.0, m = -INFINITY, z0 = 0.0, z1 = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.n;
       i += (long long)gridDim.x * blockDim.x) {
    a.x[i] += alpha * a.p[i];
    double ri = a.r[i] - alpha * a.q[i];
    a.r[i] = ri;
    rz += ri * (ri / a.d[i]);
    m = nanmax(m, fabs(ri));
  }
  __shared__ double tot[4];
  if (grid_reduce4(a.rb, rz, z0, z1, m, tot) && threadIdx.x == 0) {
    a.cg[9] = tot[0] / a.cg[0];
    a.cg[0] = tot[0];
    a.cg[3] = tot[3];
  }
}

__global__ void k_cg_dir(CgArgs a) {
  const double beta = a.cg[9];
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.n;
       i += (long long)gridDim.x * blockDim.x)
    a.p[i] = a.r[i] / a.d[i] + beta * a.p[i];
}

__global__ void k_mask_copy(const double* x0, const uint32_t* fixbits, double* x, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    uint32_t b = fix_bits(fixbits, i >> 1);
    bool fixed = (i & 1) ? (b & 2u) : (b & 1u);
    x[i] = (x0 && !fixed) ? x0[i] : 0.0;
  }
}
}  // namespace bsp

extern "C" int bsp_exact_solve(bsp_grid* g, const double* d_a, double tol, const double* d_x0,
                               long long max_iters, double* d_u, void* stream) {
  if (!g || !d_a || !d_u) return set_error(BSP_EINVAL, "null argument");
  if (!(tol > 0)) return set_error(BSP_EINVAL, "tol must be positive");
  if (!g->uniform_diag) return set_error(BSP_EUNSUPPORTED, "Jacobi PCG needs a uniform ke diagonal");
  cudaStream_t s = (cudaStream_t)stream;
  int rc = ensure_wk(g, 4 * (size_t)g->n + 8);
  if (rc) return rc;
  double* r = g->wk;
  double* p = g->wk + g->n;
  double* q = g->wk + 2 * g->n;
  double* d = g->wk + 3 * g->n;
  double* cg = g->red + 16;
  const unsigned nb = (unsigned)std::min<long long>((g->n + 255) / 256, 4 * g->nsm);
  CgArgs A{d_u, r, p, q, d, g->n, cg, RedBuf{g->part, g->counter}};
  k_mask_copy<<<nb, 256, 0, s>>>(d_x0, g->fixbits, d_u, g->n);
  k_diag<<<(unsigned)((g->N + 255) / 256), 256, 0, s>>>(g->view(), g->km, d_a, (double2*)d);
  BSP_CU(cudaGetLastError());
  long long it = 0;
  const int check_every = 8;
  for (int restart = 0; restart < 64; ++restart) {
    // true residual t = Kx - f into r, then r = -t, p = r/d
    StiffArgs t = stiff_args(g);
    t.a = d_a;
    t.u = (const double2*)d_u;
    t.out = (double2*)r;
    t.flags = SF_SUB_LOAD | SF_IN_MASKED;  // x was masked by k_mask_copy
    BSP_CU(launch_stiff(g, t, s));
    k_cg_init<<<nb, 256, 0, s>>>(A);
    BSP_CU(cudaGetLastError());
    BSP_CU(cudaMemcpyAsync(g->hpin, cg + 3, sizeof(double), cudaMemcpyDeviceToHost, s));
    BSP_CU(cudaStreamSynchronize(s));
    double res = g->hpin[0];
    if (!(res == res)) return set_error(BSP_ESOLVE, "non-finite residual in exact_solve");
    if (res <= tol) return BSP_OK;
    if (it >= max_iters)
      return set_error(BSP_ESOLVE, "CG did not reach tol %g (residual %.3e)", tol, res);
    bool recheck = false;
    while (it < max_iters && !recheck) {
      for (int j = 0; j < check_every && it < max_iters; ++j, ++it) {
        StiffArgs m = stiff_args(g);
        m.a = d_a;
        m.u = (const double2*)p;
        m.out = (double2*)q;
        m.flags = SF_REDUCE | SF_IN_MASKED;  // CG directions stay masked
        m.hook = HK_STORE;
        m.red_out = cg + 4;  // [4] = p.Kp
        BSP_CU(launch_stiff(g, m, s));
        k_cg_step<<<nb, 256, 0, s>>>(A);
        k_cg_dir<<<nb, 256, 0, s>>>(A);
        BSP_CU(cudaGetLastError());
      }
      BSP_CU(cudaMemcpyAsync(g->hpin, cg + 3, sizeof(double), cudaMemcpyDeviceToHost, s));
      BSP_CU(cudaStreamSynchronize(s));
      double rr = g->hpin[0];
      if (!(rr == rr)) return set_error(BSP_ESOLVE, "non-finite residual in exact_solve");
      if (rr <= 0.5 * tol) recheck = true;  // confirm with the true residual
    }
  }
  return set_error(BSP_ESOLVE, "CG did not reach tol %g", tol);
}
