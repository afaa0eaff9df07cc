// Row-slab domain decomposition of the outer loop over several GPUs (SURVEY
// §8(e)), one process per GPU with NCCL, or all slabs in one process (local
// transport: the same kernels and exchange pattern with device copies, used
// for single-GPU parity tests).
//
// Geometry.  Rank r owns element rows [e0, e1) and node rows [e0, e1) (the last
// rank also owns node row ny).  It stores the window of element rows [w0, w1)
// = [e0 - H, e1 + H) clipped to the grid, with H = filter radius + 1, as a
// local nx x (w1 - w0) grid (node rows [w0, w1]).  Every kernel runs on the
// whole window; only owned rows are exact and only they enter reductions:
//   v     exact on [e0-H, e1+H) after the v halo exchange
//   a     exact on [e0-1, e1+1): 7-tap filter of the exact v rows
//   r, z  exact on owned node rows (elements e0-1 .. e1-1, u rows e0-1 .. e1)
//   sens  exact on owned element rows; the adjoint needs +-radius rows: halo
//   u     ghost node rows e0-1 and e1 by exchange
// Per pfbto iteration: 3 all-gathers of 8-double partial totals (residual,
// sum g, high-level), summed in rank order on every rank (bitwise identical
// scalars everywhere, run-to-run deterministic), and 2 grouped halo
// exchanges (sens + z; v + u).  An active budget (rare) ends the batch and the
// host runs the lambda search with one all-gather per round.
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "grid.cuh"
#include "highlevel.cuh"
#include "mg.cuh"
#include "krylov.cuh"

using namespace bsp;

namespace bsp {
constexpr int kSlot = 8;  // doubles per rank partial
}

namespace {

struct Slab {
  int rank = 0;
  int e0 = 0, e1 = 0, w0 = 0, w1 = 0;
  int nyl = 0;
  int own0 = 0, own1 = 0;    // local owned element rows
  int nown0 = 0, nown1 = 0;  // local owned node rows
  bsp_grid* g = nullptr;
  double *u[2] = {nullptr, nullptr}, *v[2] = {nullptr, nullptr};
  double *vp = nullptr, *a = nullptr, *sens = nullptr, *gr = nullptr, *z = nullptr;
  uint8_t* active = nullptr;
  // Jacobi-PCG low-level step (pcg_jacobi): window-sized vectors + scalars
  double *X = nullptr, *R = nullptr, *P = nullptr, *Q = nullptr, *D = nullptr, *sc = nullptr;
  // CPFBTO Krylov step: window-sized power basis (npow+1 columns), TSQR scratch,
  // every rank's local R factor (all-gathered)
  double *K = nullptr, *Rbuf = nullptr, *gathR = nullptr;
  int tsqr_blocks = 0;
  // MG-PCG (mg_pcg): block-Jacobi multigrid preconditioner.  The block is the
  // principal submatrix of K on this rank's owned node rows: a local grid of
  // window node rows [lb, hb] whose extra rows beyond the owned ones (one per
  // interior cut) are fixed, with its own V-cycle hierarchy.
  bsp_grid* gb = nullptr;
  bsp_mg* mg = nullptr;
  int lb = 0, hb = 0;
  double *Z = nullptr, *Rb = nullptr;
  double* alphas = nullptr;
  RecRow* rec = nullptr;
  // beta's power iteration on the slabs (bsp_dist_estimate_beta): x ping-pong, K x / d^2
  double *pb[2] = {nullptr, nullptr}, *pt = nullptr;
  double* slot = nullptr;  // [kSlot]
  double* gath = nullptr;  // [G * kSlot]
};

// sum the per-rank partials in rank order: slots [0, NS) add, the rest max
template <int N, int NS>
__device__ void gather_total(const double* gath, int G, double* tot) {
  for (int i = 0; i < N; ++i) tot[i] = i < NS ? 0.0 : -INFINITY;
  for (int r = 0; r < G; ++r)
    for (int i = 0; i < N; ++i) {
      const double x = gath[r * kSlot + i];
      tot[i] = i < NS ? tot[i] + x : nanmax(tot[i], x);
    }
}

__global__ void k_fin_residual(DevState* st, const double* gath, int G) {
  if (st->done) return;
  double tot[4];
  gather_total<4, 3>(gath, G, tot);
  residual_hook(st, tot);
}

__global__ void k_fin_gsum(DevState* st, const double* gath, int G) {
  if (st->done) return;
  double tot[1];
  gather_total<1, 1>(gath, G, tot);
  st->gsum = tot[0];
}

__global__ void k_fin_hl(HLArgs p, const double* gath, int G) {
  if (p.st->done) return;
  double tot[6];
  gather_total<6, 4>(gath, G, tot);
  hl_write_hook(p, tot);
}

// PCG scalars from the gathered partials: sc[idx] = sum (rz or p.Kp)
__global__ void k_fin_sc(double* sc, int idx, const double* gath, int G, const int* gate) {
  if (gate && *gate) return;
  double tot[1];
  gather_total<1, 1>(gath, G, tot);
  sc[idx] = tot[0];
}

// rz' = sum; beta = rz'/rz (pcg.cu k_pcg_update's finalisation)
__global__ void k_fin_beta(double* sc, const double* gath, int G, const int* gate) {
  if (gate && *gate) return;
  double tot[1];
  gather_total<1, 1>(gath, G, tot);
  sc[6] = (tot[0] > 0.0 && sc[0] > 0.0) ? tot[0] / sc[0] : 0.0;
  sc[0] = tot[0];
}

// beta's power iteration (fea.py:278-301 / solvers.py:348-364 on the slabs):
// i < 0: the start vector's norm (pw[1], the scale of iteration 0's input);
// else the HK_POWER / HK_POWER_DOT hook on the rank-order totals
__global__ void k_fin_power(DevState* st, const double* gath, int G, int dot, int i) {
  double tot[3];
  gather_total<3, 3>(gath, G, tot);
  const double n = sqrt(tot[1]);
  if (i < 0) {
    st->pw[1] = n;
    st->pow_stop = (n == 0.0) ? 1 : 0;
    st->rho = dot ? 1.0 : 0.0;
    return;
  }
  if (st->pow_stop) return;
  st->rho = dot ? tot[2] : tot[0];
  st->pw[i & 1] = n;
  if (n == 0.0) st->pow_stop = 1;
}

// slot[1] = sum of x^2 over local rows [r0, r1) (row = doubles per row)
__global__ void k_rows_sumsq(const double* x, long long r0, long long r1, long long row, RedBuf rb,
                             double* slot) {
  double s = 0.0;
  const long long n = (r1 - r0) * row;
  const double* p = x + r0 * row;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    s += p[i] * p[i];
  __shared__ double tot[4];
  if (grid_reduce4(rb, 0.0, s, 0.0, -INFINITY, tot) && threadIdx.x == 0) {
    slot[0] = 0.0;
    slot[1] = tot[1];
    slot[2] = 0.0;
    slot[3] = 0.0;
  }
}

// the activation field for the host reads (fbto / pfbto do not store it)
__global__ void k_act_from_vp(const double* vp, double* a, long long n, double eta) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    a[i] = act_pow(vp[i], eta);
}

__global__ void k_fill(double* x, long long n, double v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] = v;
}

// Krylov power i: m = |K q_i / |q_i|| over all ranks (the HK_KRYLOV hook)
__global__ void k_fin_krylov(DevState* st, const double* gath, int G, int i) {
  if (st->done || st->kry_stop) return;
  double tot[1];
  gather_total<1, 1>(gath + 1, G, tot);  // slot[1] = |t|^2 of the reducing k_stiff
  const double m = sqrt(tot[0]);
  if (m == 0.0) {
    st->kry_stop = 1;
  } else {
    st->norms[i + 1] = m;
    st->kry_count = i + 1;
  }
}

BSP_DEV double clampd(double x, double lo, double hi) { return fmin(fmax(x, lo), hi); }

BSP_DEV double trial(const HLArgs& p, long long e, double alpha, double mean) {
  const double step = p.mean_projection ? (p.g[e] - mean) : p.g[e];
  return p.v[e] + alpha * step;
}

// host lambda search: regime split at lam on the owned elements -> slot
__global__ void __launch_bounds__(256) k_lam_split(HLArgs p, double lam, double alpha) {
  const double mean = p.mean_projection ? p.st->gsum / p.n_active : 0.0;
  double smid = 0.0, nmid = 0.0, nlo = 0.0, nhi = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < p.E; e += stride) {
    if (p.active && !p.active[e]) continue;
    const double w = trial(p, e, alpha, mean);
    const double d = w - lam;
    if (d <= p.lo) nlo += 1.0;
    else if (d >= p.hi) nhi += 1.0;
    else { smid += w; nmid += 1.0; }
  }
  __shared__ double tot[4];
  double v4[4] = {smid, nmid, nlo, nhi};
  if (grid_reduce_nn<4, 4>(p.rb, v4, tot) && threadIdx.x == 0)
    for (int i = 0; i < 4; ++i) p.defer_out[i] = tot[i];
}

// final write v_next = clamp(w - lam) -> slot (volume, dv)
__global__ void __launch_bounds__(256) k_lam_write(HLArgs p, double lam, double alpha) {
  const double mean = p.mean_projection ? p.st->gsum / p.n_active : 0.0;
  double vol = 0.0, dv = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < p.E; e += stride) {
    const double v = p.v[e];
    double out = v;
    if (!p.active || p.active[e]) out = clampd(trial(p, e, alpha, mean) - lam, p.lo, p.hi);
    p.v_next[e] = out;
    dv = nanmax(dv, fabs(out - v));
    vol += v;
  }
  __shared__ double tot[2];
  double v2[2] = {vol, dv};
  if (grid_reduce_nn<2, 1>(p.rb, v2, tot) && threadIdx.x == 0) {
    p.defer_out[0] = tot[0];
    p.defer_out[1] = tot[1];
  }
}

__global__ void k_fin_lam(HLArgs p, const double* gath, int G, double lam, int rounds) {
  double tot[2];
  gather_total<2, 1>(gath, G, tot);
  p.st->lam_needed = 0;
  hl_finalize(p, tot[1], tot[0], lam, rounds);
}

}  // namespace

struct bsp_dist {
  int G = 1, nx = 0, ny = 0, H = 4;
  bool local = true;
  ncclComm_t comm = nullptr;
  std::vector<Slab> slabs;
  bsp_solver_config cfg{};
  FilterTaps taps{};
  double n_active = 0.0;
  cudaStream_t s = nullptr;
  cudaGraphExec_t exec[2] = {nullptr, nullptr};
  bool graphs = false;
  double* h_alphas = nullptr;
  RecRow* h_rec = nullptr;
  DevState* h_st = nullptr;
  double* h_gath = nullptr;
  long long last_k = 0;
  int lam_rounds_total = 0, host_lambda_iters = 0;
  // fbto / pfbto created without beta: bsp_dist_estimate_beta computes it on
  // the slabs, then the iteration graphs are captured
  bool need_beta = false;
  // fbto / pfbto: after the residual the iteration forks (as on one GPU,
  // solver.cu): the side branch exchanges the energies' halo, runs the
  // adjoint filter and the high-level write with their all-gathers and
  // exchanges v's halo on its own stream and communicator (comm2, split from
  // comm: the two branches' NCCL calls never share one); the main branch
  // exchanges z's row, runs the Jacobi step and exchanges u's row -- each
  // branch's exchanges overlap the other branch's kernels
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  ncclComm_t comm2 = nullptr;
  // cpfbto_krylov: powers requested (min(dim + 1, global DOFs)) and formed
  // (<= 63, krylov.cuh), TSQR columns and the R factor stride of its variant
  int npow_req = 0, npow = 0, nc = 0, rdim = 0;
  size_t kr() const { return (size_t)rdim * rdim; }  // doubles per R factor
};

namespace {

int fail_nccl(ncclResult_t r, const char* what) {
  return set_error(BSP_ECUDA, "%s: %s", what, ncclGetErrorString(r));
}
#define BSP_NCCL(call)                                  \
  do {                                                  \
    ncclResult_t r_ = (call);                           \
    if (r_ != ncclSuccess) return fail_nccl(r_, #call); \
  } while (0)

size_t erow(const bsp_dist* d) { return (size_t)d->nx; }             // doubles per element row
unsigned pcg_blocks(long long n, int nsm) {  // same as pcg.cu's vec_blocks
  long long b = (n / 2 + 255) / 256;
  return (unsigned)std::max<long long>(1, std::min<long long>(b, 16ll * nsm));
}
size_t nrow(const bsp_dist* d) { return 2 * (size_t)(d->nx + 1); }   // doubles per node row

// All-gather of every slab's slot into every slab's gath.
int allgather(bsp_dist* d, cudaStream_t s = nullptr, ncclComm_t comm = nullptr) {
  if (!s) s = d->s;
  if (!comm) comm = d->comm;
  if (d->local) {
    for (auto& dst : d->slabs)
      for (auto& src : d->slabs)
        BSP_CU(cudaMemcpyAsync(dst.gath + src.rank * kSlot, src.slot, kSlot * sizeof(double),
                               cudaMemcpyDeviceToDevice, s));
    return BSP_OK;
  }
  Slab& sl = d->slabs[0];
  BSP_NCCL(ncclAllGather(sl.slot, sl.gath, kSlot, ncclDouble, comm, s));
  return BSP_OK;
}

// All-gather of every rank's local R factor (d->kr() doubles at `src` of each
// slab) into every slab's gathR.
int allgather_R(bsp_dist* d, const std::vector<const double*>& src) {
  const size_t kr = d->kr();
  if (d->local) {
    for (auto& dst : d->slabs)
      for (size_t r = 0; r < d->slabs.size(); ++r)
        BSP_CU(cudaMemcpyAsync(dst.gathR + d->slabs[r].rank * kr, src[r], kr * sizeof(double),
                               cudaMemcpyDeviceToDevice, d->s));
    return BSP_OK;
  }
  BSP_NCCL(ncclAllGather(src[0], d->slabs[0].gathR, kr, ncclDouble, d->comm, d->s));
  return BSP_OK;
}

// One halo exchange item: field selector, depth (rows), element or node rows.
struct HaloItem {
  double* (*field)(Slab&, int p);
  int depth;
  bool node;
  int col = 0;  // column of a multi-column field (the Krylov basis), stride = window n
};

double* col_ptr(const HaloItem& h, Slab& s, int p) {
  return h.field(s, p) + (size_t)h.col * (size_t)s.g->n;
}

double* f_v_next(Slab& s, int p) { return s.v[1 - p]; }
double* f_u_next(Slab& s, int p) { return s.u[1 - p]; }
double* f_sens(Slab& s, int) { return s.sens; }
double* f_z(Slab& s, int) { return s.z; }
double* f_p(Slab& s, int) { return s.P; }
double* f_k(Slab& s, int) { return s.K; }
double* f_pb(Slab& s, int p) { return s.pb[p]; }
double* f_pt(Slab& s, int) { return s.pt; }

// rows this slab sends up (to rank-1) / down (to rank+1), and its halo rows
// filled from above / below
void halo_rows(const Slab& s, const HaloItem& h, int& send_up, int& send_dn, int& recv_up,
               int& recv_dn) {
  if (h.node) {
    send_up = s.nown0;      // first owned node row -> rank-1's bottom ghost
    send_dn = s.own1 - 1;   // last owned node row (global e1-1) -> rank+1's top ghost
    recv_up = s.nown0 - 1;  // ghost node row e0-1
    recv_dn = s.own1;       // ghost node row e1
  } else {
    send_up = s.own0;
    send_dn = s.own1 - h.depth;
    recv_up = s.own0 - h.depth;
    recv_dn = s.own1;
  }
}

int halo(bsp_dist* d, int p, const std::vector<HaloItem>& items, cudaStream_t st = nullptr,
         ncclComm_t comm = nullptr) {
  if (!st) st = d->s;
  if (!comm) comm = d->comm;
  const int G = d->G;
  if (G == 1) return BSP_OK;
  if (d->local) {
    for (int r = 0; r + 1 < G; ++r) {
      Slab& up = d->slabs[r];
      Slab& dn = d->slabs[r + 1];
      for (const HaloItem& h : items) {
        const size_t row = h.node ? nrow(d) : erow(d);
        const size_t bytes = row * h.depth * sizeof(double);
        int su, sd, ru, rd;
        int su2, sd2, ru2, rd2;
        halo_rows(up, h, su, sd, ru, rd);
        halo_rows(dn, h, su2, sd2, ru2, rd2);
        // up's bottom owned rows -> dn's top halo; dn's top owned rows -> up's bottom halo
        BSP_CU(cudaMemcpyAsync(col_ptr(h, dn, p) + ru2 * row, col_ptr(h, up, p) + sd * row, bytes,
                               cudaMemcpyDeviceToDevice, st));
        BSP_CU(cudaMemcpyAsync(col_ptr(h, up, p) + rd * row, col_ptr(h, dn, p) + su2 * row, bytes,
                               cudaMemcpyDeviceToDevice, st));
      }
    }
    return BSP_OK;
  }
  Slab& s = d->slabs[0];
  BSP_NCCL(ncclGroupStart());
  for (const HaloItem& h : items) {
    const size_t row = h.node ? nrow(d) : erow(d);
    const size_t cnt = row * h.depth;
    int su, sd, ru, rd;
    halo_rows(s, h, su, sd, ru, rd);
    double* f = col_ptr(h, s, p);
    if (s.rank > 0) {
      BSP_NCCL(ncclSend(f + su * row, cnt, ncclDouble, s.rank - 1, comm, st));
      BSP_NCCL(ncclRecv(f + ru * row, cnt, ncclDouble, s.rank - 1, comm, st));
    }
    if (s.rank + 1 < G) {
      BSP_NCCL(ncclSend(f + sd * row, cnt, ncclDouble, s.rank + 1, comm, st));
      BSP_NCCL(ncclRecv(f + rd * row, cnt, ncclDouble, s.rank + 1, comm, st));
    }
  }
  BSP_NCCL(ncclGroupEnd());
  return BSP_OK;
}

HLArgs hl_args(bsp_dist* d, Slab& s, int p) {
  const size_t off = (size_t)s.own0 * d->nx;
  HLArgs h{};
  h.v = s.v[p] + off;
  h.g = s.gr + off;
  h.v_next = s.v[1 - p] + off;
  h.active = s.active ? s.active + off : nullptr;
  h.E = (long long)(s.own1 - s.own0) * d->nx;
  h.n_active = d->n_active;
  h.lo = d->cfg.v_lo;
  h.hi = d->cfg.v_hi;
  h.budget = d->cfg.budget;
  h.alphas = s.alphas;
  h.mean_projection = d->cfg.mean_projection;
  h.tol_dv = d->cfg.tol_dv;
  h.tol_res = d->cfg.tol_res;
  h.rb = RedBuf{s.g->part, s.g->counter};
  h.st = s.g->st;
  h.rec = s.rec;
  h.defer_out = s.slot;
  h.host_lambda = 1;
  return h;
}

// Jacobi-preconditioned CG on the slabs: u_next = u - beta PCG_k(K(a), r) with
// the CG dot products (p.Kp, r.z) all-gathered per rank and summed in rank
// order, and the search direction p halo-exchanged (one node row each side)
// before every matvec.  Vector updates run on the owned node rows only.
// z = M^{-1} r on this slab's block: the local V-cycle of the owned rows
// (input masked to the block's fixed DOFs, which include the cut rows)
static int block_vcycle(bsp_dist* d, Slab& s, cudaStream_t st) {
  const size_t row = nrow(d);
  const long long nb = s.gb->n;
  k_mask_copy<<<pcg_blocks(2 * nb, s.g->nsm), 256, 0, st>>>(s.R + (size_t)s.lb * row,
                                                            s.gb->fixbits, s.Rb, nb);
  BSP_CU(cudaGetLastError());
  return mg_vcycle_enqueue(s.mg, s.Rb, s.Z + (size_t)s.lb * row, d->cfg.mg_omega, d->cfg.mg_nu,
                           &s.g->st->done, st);
}

int enqueue_pcg(bsp_dist* d, int p) {
  const bsp_solver_config& c = d->cfg;
  cudaStream_t st = d->s;
  const int steps = c.inner_steps;
  const size_t row = nrow(d);
  const bool mgp = c.algorithm == BSP_ALGO_MG_PCG;
  int rc;
  for (Slab& s : d->slabs) {
    const int* gate = &s.g->st->done;
    const size_t off = (size_t)s.nown0 * row;
    const long long n = (long long)(s.nown1 - s.nown0) * row;
    if (mgp) {
      if ((rc = mg_setup_enqueue(s.mg, s.a + (size_t)s.lb * d->nx, gate, st))) return rc;
      if ((rc = block_vcycle(d, s, st))) return rc;
      k_pcg_init_z<<<pcg_blocks(n, s.g->nsm), 256, 0, st>>>(
          s.R + off, s.R + off, s.Z + off, s.P + off, s.sc, RedBuf{s.g->part, s.g->counter}, n,
          gate, s.slot);
    } else {
      k_diag<<<node_grid(s.g->nx, s.g->ny, wave_blocks((const void*)k_diag, 256)), 256, 0, st>>>(s.g->view(), s.g->km, s.a,
                                                               (double2*)s.D);
      k_pcg_init_jacobi<<<pcg_blocks(n, s.g->nsm), 256, 0, st>>>(
          s.R + off, s.R + off, s.P + off, s.D + off, s.sc, RedBuf{s.g->part, s.g->counter}, n,
          gate, s.slot);
    }
    BSP_CU(cudaGetLastError());
  }
  if ((rc = allgather(d))) return rc;
  for (Slab& s : d->slabs) k_fin_sc<<<1, 1, 0, st>>>(s.sc, 0, s.gath, d->G, &s.g->st->done);
  BSP_CU(cudaGetLastError());
  for (int j = 0; j < steps; ++j) {
    if ((rc = halo(d, p, {{f_p, 1, true}}))) return rc;
    for (Slab& s : d->slabs) {
      StiffArgs q = stiff_args(s.g);
      q.a = s.a;
      q.u = (const double2*)s.P;
      q.out = (double2*)s.Q;
      q.flags = SF_REDUCE | SF_IN_MASKED;
      q.hook = HK_STORE;
      q.red_out = s.slot;  // slot[0] = this rank's p.Kp
      q.red_need = 1;
      q.red_y0 = s.nown0;
      q.red_y1 = s.nown1;
      q.gate0 = &s.g->st->done;
      BSP_CU(launch_stiff(s.g, q, st));
    }
    if ((rc = allgather(d))) return rc;
    const int last = j == steps - 1;
    for (Slab& s : d->slabs) {
      const int* gate = &s.g->st->done;
      k_fin_sc<<<1, 1, 0, st>>>(s.sc, 1, s.gath, d->G, gate);
      const size_t off = (size_t)s.nown0 * row;
      const long long n = (long long)(s.nown1 - s.nown0) * row;
      BSP_CU(launch_pcg_update(pcg_blocks(n, s.g->nsm), st, s.X + off, s.R + off, s.P + off,
                               s.Q + off, mgp ? nullptr : s.D + off, s.sc,
                               RedBuf{s.g->part, s.g->counter}, n, j == 0, last, s.u[p] + off,
                               c.beta, s.u[1 - p] + off, gate, s.slot));
    }
    if (last) break;
    if (mgp) {  // z = M^{-1} r, rz' = r.z over the owned rows
      for (Slab& s : d->slabs) {
        const size_t off = (size_t)s.nown0 * row;
        const long long n = (long long)(s.nown1 - s.nown0) * row;
        if ((rc = block_vcycle(d, s, st))) return rc;
        k_pcg_rz<<<pcg_blocks(n, s.g->nsm), 256, 0, st>>>(s.R + off, s.Z + off, s.sc,
                                                          RedBuf{s.g->part, s.g->counter}, n,
                                                          &s.g->st->done, s.slot);
        BSP_CU(cudaGetLastError());
      }
    }
    if ((rc = allgather(d))) return rc;
    for (Slab& s : d->slabs) {
      const int* gate = &s.g->st->done;
      k_fin_beta<<<1, 1, 0, st>>>(s.sc, s.gath, d->G, gate);
      const size_t off = (size_t)s.nown0 * row;
      const long long n = (long long)(s.nown1 - s.nown0) * row;
      k_pcg_dir<<<pcg_blocks(n, s.g->nsm), 256, 0, st>>>(s.P + off, s.R + off,
                                                         mgp ? nullptr : s.D + off,
                                                         mgp ? s.Z + off : nullptr, s.sc, n, gate);
      BSP_CU(cudaGetLastError());
    }
  }
  return BSP_OK;
}

// CPFBTO Krylov step on the slabs (solvers.py:222-255): the power basis
// q_{i+1} = K q_i / |q_i| with q_i halo-exchanged and |K q_i| all-gathered per
// power; TSQR of each rank's owned rows down to one local R; the local R
// factors all-gathered and merged by every rank in rank order (identical
// coefficients everywhere); the combination on the owned rows.
int enqueue_krylov(bsp_dist* d, int p) {
  const bsp_solver_config& c = d->cfg;
  cudaStream_t st = d->s;
  const size_t row = nrow(d);
  int rc;
  const int npow = d->npow, nc = d->nc;
  const size_t kr = d->kr();
  for (int i = 0; i < npow; ++i) {
    if ((rc = halo(d, p, {{f_k, 1, true, i}}))) return rc;
    for (Slab& s : d->slabs) {
      const long long ldq = s.g->n;
      StiffArgs q = stiff_args(s.g);
      q.a = s.a;
      q.u = (const double2*)(s.K + i * ldq);
      q.in_div = &s.g->st->norms[i];
      q.out = (double2*)(s.K + (i + 1) * ldq);
      q.flags = SF_REDUCE | SF_IN_MASKED;
      q.hook = HK_STORE;
      q.red_out = s.slot;  // slot[1] = this rank's |K q_i / |q_i||^2
      q.red_need = 2;
      q.red_y0 = s.nown0;
      q.red_y1 = s.nown1;
      q.gate0 = &s.g->st->done;
      q.gate1 = &s.g->st->kry_stop;
      BSP_CU(launch_stiff(s.g, q, st));
    }
    if ((rc = allgather(d))) return rc;
    for (Slab& s : d->slabs) k_fin_krylov<<<1, 1, 0, st>>>(s.g->st, s.gath, d->G, i);
    BSP_CU(cudaGetLastError());
  }
  // local TSQR of the owned rows (no solve at the last local level)
  std::vector<const double*> localR;
  for (Slab& s : d->slabs) {
    const size_t off = (size_t)s.nown0 * row;
    KryArgs ka{};
    ka.Q = s.K + off;
    ka.ldq = s.g->n;
    ka.n = (long long)(s.nown1 - s.nown0) * row;
    ka.Rbuf = s.Rbuf;
    ka.st = s.g->st;
    ka.no_solve = 1;
    BSP_CU(launch_tsqr_leaf(nc, s.tsqr_blocks, ka, st));
    const int fan = tsqr_fan_in(nc);
    const size_t half = (size_t)s.tsqr_blocks * kr;
    int nin = s.tsqr_blocks, lvl = 0;
    const double* last = s.Rbuf;
    while (nin > 1) {
      const int nout = (nin + fan - 1) / fan;
      const double* rin = s.Rbuf + ((lvl & 1) ? half : 0);
      double* rout = s.Rbuf + ((lvl & 1) ? 0 : half);
      BSP_CU(launch_tsqr_merge(nc, nout, ka, rin, nin, rout, st));
      last = rout;
      nin = nout;
      ++lvl;
    }
    localR.push_back(last);
  }
  if ((rc = allgather_R(d, localR))) return rc;
  for (Slab& s : d->slabs) {
    // merge the G local factors in rank order; the single-CTA level solves
    KryArgs ka{};
    ka.st = s.g->st;
    ka.npow_req = d->npow_req;  // a truncated basis is refused by the solve (kry_trunc)
    const int fan = tsqr_fan_in(nc);
    int nin = d->G, lvl = 0;
    const double* rin = s.gathR;
    double* bufs[2] = {s.Rbuf, s.Rbuf + (size_t)std::max(s.tsqr_blocks, d->G) * kr};
    do {
      const int nout = (nin + fan - 1) / fan;
      double* rout = bufs[lvl & 1];
      BSP_CU(launch_tsqr_merge(nc, nout, ka, rin, nin, rout, st));
      rin = rout;
      nin = nout;
      ++lvl;
    } while (nin > 1);
    // u_next = u - beta sum_i coef_i q_i on the owned rows
    const size_t off = (size_t)s.nown0 * row;
    KryArgs kc{};
    kc.Q = s.K + off;
    kc.ldq = s.g->n;
    kc.n = (long long)(s.nown1 - s.nown0) * row;
    kc.st = s.g->st;
    kc.u = s.u[p] + off;
    kc.out = s.u[1 - p] + off;
    kc.beta = c.beta;
    k_kry_combine<<<pcg_blocks(kc.n, s.g->nsm), 256, 0, st>>>(kc);
    BSP_CU(cudaGetLastError());
  }
  return BSP_OK;
}

int enqueue_iteration(bsp_dist* d, int p) {
  const bsp_solver_config& c = d->cfg;
  cudaStream_t st = d->s;
  const bool pf = c.algorithm == BSP_ALGO_PFBTO_JACOBI;
  const bool pcg = c.algorithm == BSP_ALGO_PCG_JACOBI || c.algorithm == BSP_ALGO_MG_PCG;
  const bool kry = c.algorithm == BSP_ALGO_CPFBTO_KRYLOV;
  // fbto / pfbto: the stiffness kernels raise v_phys to eta themselves
  // (SF_A_POW, as on one GPU): the filter writes no activation array
  const bool apow = c.algorithm == BSP_ALGO_FBTO || pf;
  int rc;
  // A: filter + residual/energies (+ fused low-level epilogue)
  for (Slab& s : d->slabs) {
    bsp_grid* g = s.g;
    const int* gate = &g->st->done;
    FilterArgs fa = filter_args(s.v[p], s.vp, apow ? nullptr : s.a, c.eta, d->nx, s.nyl, d->taps, gate, nullptr,
                                nullptr, RedBuf{nullptr, nullptr});
    fa.gy0 = s.w0;
    fa.gny = d->ny;
    rc = launch_filter_fa(fa, 0, st);
    if (rc) return rc;
    StiffArgs r = stiff_args(g);
    r.a = apow ? s.vp : s.a;
    r.u = (const double2*)s.u[p];
    r.flags = SF_SUB_LOAD | SF_REDUCE | SF_ENERGY | SF_IN_MASKED | (apow ? SF_A_POW : 0);
    r.vp = s.vp;
    r.eta = c.eta;
    r.sens = s.sens;
    r.hook = HK_STORE;
    r.red_out = s.slot;
    r.red_y0 = s.nown0;
    r.red_y1 = s.nown1;
    r.gate0 = gate;
    if (pf) {
      r.flags |= SF_D2DIV;
      r.out = (double2*)s.z;
    } else if (pcg) {
      r.out = (double2*)s.R;  // the CG right-hand side
    } else if (kry) {
      r.out = (double2*)s.K;  // basis column 0 = r
    } else {
      r.flags |= SF_AXPY;
      r.base = (const double2*)s.u[p];
      r.beta = c.beta;
      r.out = (double2*)s.u[1 - p];
    }
    BSP_CU(launch_stiff(g, r, st));
  }
  if ((rc = allgather(d))) return rc;
  for (Slab& s : d->slabs) {
    k_fin_residual<<<1, 1, 0, st>>>(s.g->st, s.gath, d->G);
    BSP_CU(cudaGetLastError());
  }
  const bool fork = d->side != nullptr;
  cudaStream_t t = st;
  ncclComm_t ct = d->comm;
  if (fork) {
    BSP_CU(cudaEventRecord(d->ev_fork, st));
    BSP_CU(cudaStreamWaitEvent(d->side, d->ev_fork, 0));
    t = d->side;
    ct = d->comm2;
    if ((rc = halo(d, p, {{f_sens, d->taps.r, false}}, t, ct))) return rc;
  } else {
    std::vector<HaloItem> mid = {{f_sens, d->taps.r, false}};
    if (pf) mid.push_back({f_z, 1, true});
    if ((rc = halo(d, p, mid))) return rc;
  }
  // C: adjoint filter, sum of g over owned active elements
  for (Slab& s : d->slabs) {
    FilterArgs fa = filter_args(s.sens, s.gr, nullptr, 1.0, d->nx, s.nyl, d->taps, &s.g->st->done,
                                s.g->st, s.active, RedBuf{s.g->part, s.g->counter});
    fa.gy0 = s.w0;
    fa.gny = d->ny;
    fa.red_y0 = s.own0;
    fa.red_y1 = s.own1;
    fa.defer_out = s.slot;
    if ((rc = launch_filter_fa(fa, 1, t))) return rc;
  }
  if ((rc = allgather(d, t, ct))) return rc;
  for (Slab& s : d->slabs) {
    k_fin_gsum<<<1, 1, 0, t>>>(s.g->st, s.gath, d->G);
    BSP_CU(cudaGetLastError());
  }
  if (fork) {
    // side branch: the high-level write, its all-gather, v's halo
    for (Slab& s : d->slabs) {
      HLArgs h = hl_args(d, s, p);
      k_hl_write<<<write_blocks(h.E, s.g->nsm), 256, 0, t>>>(h);
      BSP_CU(cudaGetLastError());
    }
    if ((rc = allgather(d, t, ct))) return rc;
    for (Slab& s : d->slabs) {
      k_fin_hl<<<1, 1, 0, t>>>(hl_args(d, s, p), s.gath, d->G);
      BSP_CU(cudaGetLastError());
    }
    if ((rc = halo(d, p, {{f_v_next, d->H, false}}, t, ct))) return rc;
    BSP_CU(cudaEventRecord(d->ev_join, t));
    // main branch: z's row, the Jacobi step (pfbto; fbto's update was the
    // residual's epilogue), u's row
    if (pf) {
      if ((rc = halo(d, p, {{f_z, 1, true}}))) return rc;
      for (Slab& s : d->slabs) {
        StiffArgs q = stiff_args(s.g);
        q.a = s.vp;  // v_phys; SF_A_POW raises it to eta
        q.eta = c.eta;
        q.u = (const double2*)s.z;
        q.out = (double2*)s.u[1 - p];
        q.base = (const double2*)s.u[p];
        q.beta = c.beta;
        q.flags = SF_AXPY | SF_IN_MASKED | SF_A_POW;
        q.gate0 = &s.g->st->done;
        BSP_CU(launch_stiff(s.g, q, st));
      }
    }
    if ((rc = halo(d, p, {{f_u_next, 1, true}}))) return rc;
    BSP_CU(cudaStreamWaitEvent(st, d->ev_join, 0));
    return BSP_OK;
  }
  if (pcg && (rc = enqueue_pcg(d, p))) return rc;
  if (kry && (rc = enqueue_krylov(d, p))) return rc;
  // D: Jacobi-squared low-level step, optimistic high-level write
  for (Slab& s : d->slabs) {
    if (pf) {
      StiffArgs q = stiff_args(s.g);
      q.a = s.vp;  // v_phys; SF_A_POW raises it to eta
      q.eta = c.eta;
      q.u = (const double2*)s.z;
      q.out = (double2*)s.u[1 - p];
      q.base = (const double2*)s.u[p];
      q.beta = c.beta;
      q.flags = SF_AXPY | SF_IN_MASKED | SF_A_POW;
      q.gate0 = &s.g->st->done;
      BSP_CU(launch_stiff(s.g, q, st));
    }
    HLArgs h = hl_args(d, s, p);
    k_hl_write<<<write_blocks(h.E, s.g->nsm), 256, 0, st>>>(h);
    BSP_CU(cudaGetLastError());
  }
  if ((rc = allgather(d))) return rc;
  for (Slab& s : d->slabs) {
    k_fin_hl<<<1, 1, 0, st>>>(hl_args(d, s, p), s.gath, d->G);
    BSP_CU(cudaGetLastError());
  }
  return halo(d, p, {{f_v_next, d->H, false}, {f_u_next, 1, true}});
}

// one graph per parity (NCCL operations are captured with the kernels);
// without graphs the iterations are enqueued one by one
void capture_graphs(bsp_dist* d) {
  d->graphs = true;
  for (int p = 0; p < 2 && d->graphs; ++p) {
    cudaGraph_t graph = nullptr;
    if (cudaStreamBeginCapture(d->s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      d->graphs = false;
      break;
    }
    const int rc = enqueue_iteration(d, p);
    cudaError_t e = cudaStreamEndCapture(d->s, &graph);
    if (rc != BSP_OK || e != cudaSuccess || !graph) {
      d->graphs = false;
      cudaGetLastError();
      if (graph) cudaGraphDestroy(graph);
      break;
    }
    e = cudaGraphInstantiate(&d->exec[p], graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      d->graphs = false;
      d->exec[p] = nullptr;
      cudaGetLastError();
    }
  }
  if (!d->graphs)
    for (int p = 0; p < 2; ++p)
      if (d->exec[p]) {
        cudaGraphExecDestroy(d->exec[p]);
        d->exec[p] = nullptr;
      }
}

void free_dist(bsp_dist* d) {
  if (!d) return;
  for (int i = 0; i < 2; ++i)
    if (d->exec[i]) cudaGraphExecDestroy(d->exec[i]);
  for (Slab& s : d->slabs) {
    for (int i = 0; i < 2; ++i) {
      cudaFree(s.u[i]);
      cudaFree(s.v[i]);
    }
    cudaFree(s.vp);
    cudaFree(s.a);
    cudaFree(s.sens);
    cudaFree(s.gr);
    cudaFree(s.z);
    cudaFree(s.X);
    cudaFree(s.R);
    cudaFree(s.P);
    cudaFree(s.Q);
    cudaFree(s.D);
    cudaFree(s.sc);
    cudaFree(s.K);
    cudaFree(s.Rbuf);
    cudaFree(s.gathR);
    cudaFree(s.active);
    cudaFree(s.alphas);
    cudaFree(s.rec);
    cudaFree(s.slot);
    cudaFree(s.gath);
    if (s.g) bsp_grid_destroy(s.g);
    if (s.mg) bsp_mg_destroy(s.mg);
    if (s.gb) bsp_grid_destroy(s.gb);
    cudaFree(s.Z);
    cudaFree(s.Rb);
  }
  if (d->comm2) ncclCommDestroy(d->comm2);
  if (d->comm) ncclCommDestroy(d->comm);
  if (d->side) cudaStreamDestroy(d->side);
  if (d->ev_fork) cudaEventDestroy(d->ev_fork);
  if (d->ev_join) cudaEventDestroy(d->ev_join);
  if (d->h_alphas) cudaFreeHost(d->h_alphas);
  if (d->h_rec) cudaFreeHost(d->h_rec);
  if (d->h_st) cudaFreeHost(d->h_st);
  if (d->h_gath) cudaFreeHost(d->h_gath);
  if (d->s) cudaStreamDestroy(d->s);
  delete d;
}

int launch_iter(bsp_dist* d, long long k) {
  const int p = (int)((k - 1) & 1);
  if (d->graphs) {
    BSP_CU(cudaGraphLaunch(d->exec[p], d->s));
    return BSP_OK;
  }
  return enqueue_iteration(d, p);
}

int set_alphas(bsp_dist* d, long long k_base, int n, const double* h_alphas) {
  BSP_CU(cudaStreamSynchronize(d->s));
  std::memcpy(d->h_alphas, h_alphas, n * sizeof(double));
  d->h_st->k_base = k_base;
  for (Slab& s : d->slabs) {
    BSP_CU(cudaMemcpyAsync(s.alphas, d->h_alphas, n * sizeof(double), cudaMemcpyHostToDevice, d->s));
    BSP_CU(cudaMemcpyAsync(&s.g->st->k_base, &d->h_st->k_base, sizeof(long long),
                           cudaMemcpyHostToDevice, d->s));
  }
  return BSP_OK;
}

// The lambda search of an iteration whose box sum exceeded the budget
// (projection.py:65-91), host-driven: one all-gather per regime-Newton round.
int host_lambda(bsp_dist* d, long long k) {
  const int p = (int)((k - 1) & 1);
  cudaStream_t st = d->s;
  const DevState& hs = *d->h_st;  // read by the caller after the batch
  const double alpha = d->h_alphas[k - hs.k_base];
  const double lo = d->cfg.v_lo, hi = d->cfg.v_hi, budget = d->cfg.budget;
  const int zero = 0;
  for (Slab& s : d->slabs)
    BSP_CU(cudaMemcpyAsync(&s.g->st->done, &zero, sizeof(int), cudaMemcpyHostToDevice, st));
  double L = 0.0, U = hs.scratch[3] - lo;
  const double guess = hs.scratch[4];
  double lam = (guess > L && guess < U) ? guess : 0.5 * (L + U);
  int rounds;
  int rc;
  for (rounds = 1; rounds <= 200; ++rounds) {
    for (Slab& s : d->slabs) {
      HLArgs h = hl_args(d, s, p);
      k_lam_split<<<write_blocks(h.E, s.g->nsm), 256, 0, st>>>(h, lam, alpha);
      BSP_CU(cudaGetLastError());
    }
    if ((rc = allgather(d))) return rc;
    Slab& s0 = d->slabs[0];
    BSP_CU(cudaMemcpyAsync(d->h_gath, s0.gath, d->G * kSlot * sizeof(double),
                           cudaMemcpyDeviceToHost, st));
    BSP_CU(cudaStreamSynchronize(st));
    double smid = 0.0, nmid = 0.0, nlo = 0.0, nhi = 0.0;
    for (int r = 0; r < d->G; ++r) {
      smid += d->h_gath[r * kSlot + 0];
      nmid += d->h_gath[r * kSlot + 1];
      nlo += d->h_gath[r * kSlot + 2];
      nhi += d->h_gath[r * kSlot + 3];
    }
    const double f = smid - nmid * lam + nlo * lo + nhi * hi;
    if (f > budget) L = lam; else U = lam;
    double next;
    if (nmid > 0.0) {
      const double root = (smid + nlo * lo + nhi * hi - budget) / nmid;
      if (std::fabs(root - lam) <= 1e-15 * std::max(1.0, std::fabs(lam))) {
        lam = (root > L && root < U) ? root : lam;
        break;
      }
      next = (root > L && root < U) ? root : 0.5 * (L + U);
    } else {
      next = 0.5 * (L + U);
    }
    // a bracket below the sums' rounding noise (a few ulps of the budget,
    // e.g. a box sum over the budget by ulps that the re-summed split no
    // longer exceeds): bisecting on would only walk lam into denormals
    if (!(U - L > 1e-15 * std::fmax(1.0, std::fabs(U))) || next == lam) {
      lam = (f > budget) ? U : lam;
      break;
    }
    lam = next;
  }
  if (lam < 0.0) lam = 0.0;
  for (Slab& s : d->slabs) {
    HLArgs h = hl_args(d, s, p);
    k_lam_write<<<write_blocks(h.E, s.g->nsm), 256, 0, st>>>(h, lam, alpha);
    BSP_CU(cudaGetLastError());
  }
  if ((rc = allgather(d))) return rc;
  for (Slab& s : d->slabs) {
    k_fin_lam<<<1, 1, 0, st>>>(hl_args(d, s, p), s.gath, d->G, lam, rounds);
    BSP_CU(cudaGetLastError());
  }
  if ((rc = halo(d, p, {{f_v_next, d->H, false}}))) return rc;
  d->lam_rounds_total += rounds;
  d->host_lambda_iters += 1;
  return BSP_OK;
}

}  // namespace

// BSP_DIST_FORK=0: the slab iteration as one chain (A/B switch)
static bool dist_fork_enabled() {
  static const bool on = [] {
    const char* e = getenv("BSP_DIST_FORK");
    return !(e && e[0] == '0');
  }();
  return on;
}

// ------------------------------------------------------------------ C ABI ---
extern "C" int bsp_nccl_unique_id(uint8_t* out, int* nbytes) {
  if (!out) return set_error(BSP_EINVAL, "null argument");
  ncclUniqueId id;
  BSP_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  if (nbytes) *nbytes = (int)sizeof(id);
  return BSP_OK;
}

extern "C" int bsp_dist_slab_rows(int ny, int world, int rank, int halo, int* e0, int* e1,
                                  int* w0, int* w1) {
  if (world < 1 || rank < 0 || rank >= world || ny < 1)
    return set_error(BSP_EINVAL, "bad slab request (ny=%d world=%d rank=%d)", ny, world, rank);
  const int a = (int)((long long)ny * rank / world), b = (int)((long long)ny * (rank + 1) / world);
  if (e0) *e0 = a;
  if (e1) *e1 = b;
  if (w0) *w0 = std::max(0, a - halo);
  if (w1) *w1 = std::min(ny, b + halo);
  return BSP_OK;
}

extern "C" int bsp_dist_destroy(bsp_dist* d) {
  if (d) cudaStreamSynchronize(d->s);
  free_dist(d);
  return BSP_OK;
}

// h_fixed/h_load/h_active/h_v0 cover the slabs' windows: in local mode the
// GLOBAL arrays (all slabs are built here); in NCCL mode this rank's window
// only (node rows [w0, w1], element rows [w0, w1)).
extern "C" int bsp_dist_create(int nx, int ny, int world, int rank, const uint8_t* nccl_id,
                               const double* h_ke, const uint8_t* h_fixed, const double* h_load,
                               const bsp_solver_config* cfg, const uint8_t* h_active,
                               double n_active, const double* h_v0, bsp_dist** out) {
  if (!h_ke || !h_fixed || !h_load || !cfg || !h_v0 || !out)
    return set_error(BSP_EINVAL, "null argument");
  bsp_solver_config c;
  {
    const int rc = normalize_config(cfg, c);
    if (rc) return rc;
  }
  if (c.algorithm != BSP_ALGO_FBTO && c.algorithm != BSP_ALGO_PFBTO_JACOBI &&
      c.algorithm != BSP_ALGO_PCG_JACOBI && c.algorithm != BSP_ALGO_CPFBTO_KRYLOV &&
      c.algorithm != BSP_ALGO_MG_PCG)
    return set_error(BSP_EUNSUPPORTED,
                     "row slabs support fbto, pfbto_jacobi, cpfbto_krylov, pcg_jacobi and mg_pcg "
                     "(algorithm %d)", c.algorithm);
  if (c.algorithm == BSP_ALGO_MG_PCG && (c.inner_steps < 1 || c.mg_nu < 1 || !(c.mg_omega > 0.0)))
    return set_error(BSP_EINVAL, "mg_pcg on row slabs needs inner_steps >= 1, nu >= 1, omega > 0");
  if (c.algorithm == BSP_ALGO_CPFBTO_KRYLOV && c.krylov_dim < 1)
    return set_error(BSP_EINVAL, "krylov_dim must be >= 1, got %d", c.krylov_dim);
  if (c.algorithm == BSP_ALGO_PCG_JACOBI && c.inner_steps < 1)
    return set_error(BSP_EINVAL, "inner_steps must be >= 1, got %d", c.inner_steps);
  if (c.max_batch < 1) return set_error(BSP_EINVAL, "max_batch must be >= 1");
  bsp_dist* d = new bsp_dist();
  d->G = world;
  d->nx = nx;
  d->ny = ny;
  d->local = nccl_id == nullptr;
  d->cfg = c;
  d->cfg.taps = nullptr;  // copied into d->taps
  d->n_active = n_active;
  if (c.algorithm == BSP_ALGO_CPFBTO_KRYLOV) {
    // as krylov_enqueue (capi.cu): the global DOF count caps the powers
    const long long n_glob = 2ll * (nx + 1) * (ny + 1);
    d->npow_req = (int)std::min<long long>((long long)c.krylov_dim + 1, n_glob);
    d->npow = krylov_formed(d->npow_req);
    d->nc = d->npow + 1;
    d->rdim = tsqr_rdim(d->nc);
  }
  int rc = make_taps(c.taps, c.n_taps, d->taps);
  if (rc || d->taps.size > kMaxTaps) {
    delete d;
    return rc ? rc
              : set_error(BSP_EUNSUPPORTED, "row slabs: filter size %d > %d (halo rows)",
                          c.n_taps, kMaxTaps);
  }
  d->H = d->taps.r + 1;
  if ((long long)ny < (long long)world * d->H) {
    delete d;
    return set_error(BSP_EINVAL, "%d ranks need >= %d element rows each (ny=%d)", world, d->H, ny);
  }
  bool ok = cudaStreamCreateWithFlags(&d->s, cudaStreamNonBlocking) == cudaSuccess &&
            cudaMallocHost(&d->h_alphas, c.max_batch * sizeof(double)) == cudaSuccess &&
            cudaMallocHost(&d->h_rec, c.max_batch * sizeof(RecRow)) == cudaSuccess &&
            cudaMallocHost(&d->h_st, sizeof(DevState)) == cudaSuccess &&
            cudaMallocHost(&d->h_gath, (size_t)world * kSlot * sizeof(double)) == cudaSuccess;
  if (!ok) {
    free_dist(d);
    return set_error(BSP_ENOMEM, "host staging allocation failed");
  }
  const size_t NX1 = (size_t)nx + 1;
  const int first = d->local ? 0 : rank, last = d->local ? world : rank + 1;
  for (int r = first; r < last && rc == BSP_OK; ++r) {
    Slab s;
    s.rank = r;
    bsp_dist_slab_rows(ny, world, r, d->H, &s.e0, &s.e1, &s.w0, &s.w1);
    s.nyl = s.w1 - s.w0;
    s.own0 = s.e0 - s.w0;
    s.own1 = s.e1 - s.w0;
    s.nown0 = s.own0;
    s.nown1 = (r == world - 1) ? s.own1 + 1 : s.own1;
    // window slices of the host arrays (global in local mode)
    const size_t nb0 = d->local ? (size_t)s.w0 * NX1 * 2 : 0;
    const size_t eb0 = d->local ? (size_t)s.w0 * nx : 0;
    rc = bsp_grid_create(nx, s.nyl, h_ke, h_fixed + nb0, h_load + nb0, &s.g);
    if (rc) break;
    const size_t nb = s.g->n * sizeof(double), eb = s.g->E * sizeof(double);
    ok = true;
    for (int i = 0; i < 2 && ok; ++i)
      ok = cudaMalloc(&s.u[i], nb) == cudaSuccess && cudaMalloc(&s.v[i], eb) == cudaSuccess;
    ok = ok && cudaMalloc(&s.vp, eb) == cudaSuccess && cudaMalloc(&s.a, eb) == cudaSuccess &&
         cudaMalloc(&s.sens, eb) == cudaSuccess && cudaMalloc(&s.gr, eb) == cudaSuccess &&
         cudaMalloc(&s.alphas, c.max_batch * sizeof(double)) == cudaSuccess &&
         cudaMalloc(&s.rec, c.max_batch * sizeof(RecRow)) == cudaSuccess &&
         cudaMalloc(&s.slot, kSlot * sizeof(double)) == cudaSuccess &&
         cudaMalloc(&s.gath, (size_t)world * kSlot * sizeof(double)) == cudaSuccess;
    if (ok && c.algorithm == BSP_ALGO_PFBTO_JACOBI) ok = cudaMalloc(&s.z, nb) == cudaSuccess;
    if (ok && (c.algorithm == BSP_ALGO_PCG_JACOBI || c.algorithm == BSP_ALGO_MG_PCG))
      ok = cudaMalloc(&s.X, nb) == cudaSuccess && cudaMalloc(&s.R, nb) == cudaSuccess &&
           cudaMalloc(&s.P, nb) == cudaSuccess && cudaMalloc(&s.Q, nb) == cudaSuccess &&
           cudaMalloc(&s.D, nb) == cudaSuccess &&
           cudaMalloc(&s.sc, 16 * sizeof(double)) == cudaSuccess;
    if (ok && c.algorithm == BSP_ALGO_MG_PCG) {
      // the block grid: owned node rows plus one fixed row beyond each cut
      s.lb = s.nown0 - (r > 0 ? 1 : 0);
      s.hb = s.nown1 - 1 + (r < world - 1 ? 1 : 0);
      const size_t rowb = NX1 * 2;
      std::vector<uint8_t> fb((size_t)(s.hb - s.lb + 1) * rowb);
      std::memcpy(fb.data(), h_fixed + nb0 + (size_t)s.lb * rowb, fb.size());
      if (r > 0) std::fill(fb.begin(), fb.begin() + rowb, (uint8_t)1);
      if (r < world - 1) std::fill(fb.end() - rowb, fb.end(), (uint8_t)1);
      std::vector<double> zl(fb.size(), 0.0);
      rc = bsp_grid_create(nx, s.hb - s.lb, h_ke, fb.data(), zl.data(), &s.gb);
      if (rc == BSP_OK) rc = bsp_mg_create(s.gb, c.mg_levels, &s.mg);
      if (rc) {
        d->slabs.push_back(s);
        break;
      }
      ok = cudaMalloc(&s.Z, nb) == cudaSuccess && cudaMalloc(&s.Rb, s.gb->n * sizeof(double)) == cudaSuccess;
      if (ok) cudaMemset(s.Z, 0, nb);
    }
    if (ok && c.algorithm == BSP_ALGO_CPFBTO_KRYLOV) {
      ok = tsqr_prepare() == cudaSuccess;
      const long long owned = (long long)(s.nown1 - s.nown0) * 2 * (nx + 1);
      s.tsqr_blocks = tsqr_leaves(owned, d->nc);
      ok = ok && cudaMalloc(&s.K, (size_t)(d->npow + 1) * nb) == cudaSuccess &&
           cudaMalloc(&s.Rbuf, 2ull * std::max(s.tsqr_blocks, world) * d->kr() * sizeof(double)) == cudaSuccess &&
           cudaMalloc(&s.gathR, (size_t)world * d->kr() * sizeof(double)) == cudaSuccess;
      if (ok) cudaMemset(s.K, 0, (size_t)(d->npow + 1) * nb);
    }
    if (ok && h_active)
      ok = cudaMalloc(&s.active, s.g->E) == cudaSuccess &&
           cudaMemcpy(s.active, h_active + eb0, s.g->E, cudaMemcpyHostToDevice) == cudaSuccess;
    if (!ok) {
      cudaGetLastError();
      d->slabs.push_back(s);
      rc = set_error(BSP_ENOMEM, "slab %d allocation failed", r);
      break;
    }
    // zero everything (ghost rows never hold stale NaNs), then the initial state
    for (int i = 0; i < 2; ++i) {
      cudaMemset(s.u[i], 0, nb);
      cudaMemset(s.v[i], 0, eb);
    }
    cudaMemset(s.vp, 0, eb);
    cudaMemset(s.a, 0, eb);
    cudaMemset(s.sens, 0, eb);
    cudaMemset(s.gr, 0, eb);
    if (s.z) cudaMemset(s.z, 0, nb);
    for (double* b : {s.X, s.R, s.P, s.Q, s.D})
      if (b) cudaMemset(b, 0, nb);
    if (s.sc) cudaMemset(s.sc, 0, 16 * sizeof(double));
    cudaMemset(s.slot, 0, kSlot * sizeof(double));
    cudaMemset(s.gath, 0, (size_t)world * kSlot * sizeof(double));
    cudaMemcpy(s.v[0], h_v0 + eb0, eb, cudaMemcpyHostToDevice);
    DevState init{};
    init.k = 1;
    init.k_base = 1;
    cudaMemcpy(s.g->st, &init, sizeof(DevState), cudaMemcpyHostToDevice);
    d->slabs.push_back(s);
  }
  if (rc == BSP_OK && !d->local) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t nr = ncclCommInitRank(&d->comm, world, id, rank);
    if (nr != ncclSuccess) rc = fail_nccl(nr, "ncclCommInitRank");
  }
  // one slab has no exchanges to overlap (measured: C5 on one NCCL rank
  // 4.32 ms/iter chained, 4.37 forked)
  if (rc == BSP_OK && world > 1 &&
      (c.algorithm == BSP_ALGO_FBTO || c.algorithm == BSP_ALGO_PFBTO_JACOBI) &&
      dist_fork_enabled()) {
    if (cudaStreamCreateWithFlags(&d->side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&d->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&d->ev_join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      rc = set_error(BSP_ENOMEM, "slab stream allocation failed");
    } else if (!d->local) {
      ncclResult_t nr = ncclCommSplit(d->comm, 0, rank, &d->comm2, nullptr);
      if (nr != ncclSuccess) rc = fail_nccl(nr, "ncclCommSplit");
    }
  }
  if (rc == BSP_OK) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) rc = set_error(BSP_ECUDA, "dist create: %s", cudaGetErrorString(e));
  }
  if (rc) {
    free_dist(d);
    return rc;
  }
  d->need_beta = (c.algorithm == BSP_ALGO_FBTO || c.algorithm == BSP_ALGO_PFBTO_JACOBI) &&
                 !(c.beta > 0.0);
  if (!d->need_beta) capture_graphs(d);
  *out = d;
  return BSP_OK;
}

// Iterations k_first .. k_first+n-1 (same contract as bsp_solver_run).
extern "C" int bsp_dist_run(bsp_dist* d, long long k_first, int n, const double* h_alphas,
                            double* h_rec, int* h_done, int* h_status) {
  if (!d || !h_alphas) return set_error(BSP_EINVAL, "null argument");
  if (d->need_beta)
    return set_error(BSP_EINVAL, "beta not set: call bsp_dist_estimate_beta first");
  if (n < 0 || n > d->cfg.max_batch)
    return set_error(BSP_EINVAL, "n %d outside [0, %d]", n, d->cfg.max_batch);
  if (k_first != d->last_k + 1)
    return set_error(BSP_EINVAL, "k_first %lld is not the next iteration %lld", k_first,
                     d->last_k + 1);
  int rc = set_alphas(d, k_first, n, h_alphas);
  if (rc) return rc;
  long long k = k_first;
  const long long k_end = k_first + n;
  int status = 0;
  while (k < k_end) {
    for (long long j = k; j < k_end; ++j)
      if ((rc = launch_iter(d, j))) return rc;
    Slab& s0 = d->slabs[0];
    BSP_CU(cudaMemcpyAsync(d->h_st, s0.g->st, sizeof(DevState), cudaMemcpyDeviceToHost, d->s));
    BSP_CU(cudaStreamSynchronize(d->s));
    d->h_st->k_base = k_first;
    status = d->h_st->done;
    k = d->h_st->k;
    if (status != 3) break;
    // an active budget at iteration k: lambda search on the host, then resume
    if ((rc = host_lambda(d, k))) return rc;
    BSP_CU(cudaMemcpyAsync(d->h_st, s0.g->st, sizeof(DevState), cudaMemcpyDeviceToHost, d->s));
    BSP_CU(cudaStreamSynchronize(d->s));
    d->h_st->k_base = k_first;
    status = d->h_st->done;
    k = d->h_st->k;
    if (status) break;
  }
  Slab& s0 = d->slabs[0];
  BSP_CU(cudaMemcpyAsync(d->h_rec, s0.rec, n * sizeof(RecRow), cudaMemcpyDeviceToHost, d->s));
  BSP_CU(cudaStreamSynchronize(d->s));
  long long done = std::min<long long>(std::max<long long>(k - k_first, 0), n);
  d->last_k = k - 1;
  for (long long i = 0; i < done; ++i) {
    h_rec[4 * i + 0] = d->h_rec[i].compliance;
    h_rec[4 * i + 1] = d->h_rec[i].res_inf;
    h_rec[4 * i + 2] = d->h_rec[i].dv_inf;
    h_rec[4 * i + 3] = d->h_rec[i].volume;
  }
  if (status == BSP_ST_DIVERGED && done < n) {
    h_rec[4 * done + 0] = d->h_st->compliance;
    h_rec[4 * done + 1] = d->h_st->res_inf;
  }
  if (h_done) *h_done = (int)done;
  if (h_status) *h_status = status;
  return BSP_OK;
}

// beta = 1 / rho of the power iteration the single-GPU set-up runs
// (solvers.py:334-364): fbto rho(K(1)), pfbto rho(K M^-2 K) at the initial
// design -- on the slabs: each iteration halo-exchanges its input node rows,
// reduces x.Kx (or x.K M^-2 K x) and |.|^2 over the owned rows and
// all-gathers the partials (rank-order sums: the same value on every rank).
// d_normals: the seeded standard normals of the GLOBAL grid on this rank's
// device (the start vector before masking and normalisation, fea.py:289-292).
extern "C" int bsp_dist_estimate_beta(bsp_dist* d, const double* d_normals, int iters,
                                      double* h_rho) {
  if (!d || !d_normals || !h_rho) return set_error(BSP_EINVAL, "null argument");
  if (iters < 1) return set_error(BSP_EINVAL, "iters must be >= 1");
  const bsp_solver_config& c = d->cfg;
  if (c.algorithm != BSP_ALGO_FBTO && c.algorithm != BSP_ALGO_PFBTO_JACOBI)
    return set_error(BSP_EINVAL, "the slab beta estimate is for fbto / pfbto_jacobi");
  const int dot = c.algorithm == BSP_ALGO_PFBTO_JACOBI;
  cudaStream_t st = d->s;
  const size_t row = nrow(d);
  int rc;
  for (Slab& s : d->slabs) {
    const size_t nb = s.g->n * sizeof(double);
    for (double** b : {&s.pb[0], &s.pb[1], &s.pt}) {
      BSP_CU(cudaMallocAsync(b, nb, st));
      BSP_CU(cudaMemsetAsync(*b, 0, nb, st));
    }
    // x0 = masked window rows [w0, w1] of the global normals (iteration 0's
    // input: pb[1], scaled by its global norm pw[1])
    k_mask_copy<<<pcg_blocks(2 * s.g->n, s.g->nsm), 256, 0, st>>>(
        d_normals + (size_t)s.w0 * row, s.g->fixbits, s.pb[1], s.g->n);
    k_rows_sumsq<<<pcg_blocks(2 * s.g->n, s.g->nsm), 256, 0, st>>>(
        s.pb[1], s.nown0, s.nown1, (long long)row, RedBuf{s.g->part, s.g->counter}, s.slot);
    BSP_CU(cudaGetLastError());
    // the activation at the initial design: fbto ones, pfbto filter(v0)^eta
    if (!dot) {
      k_fill<<<pcg_blocks(2 * s.g->E, s.g->nsm), 256, 0, st>>>(s.a, s.g->E, 1.0);
      BSP_CU(cudaGetLastError());
    } else {
      FilterArgs fa = filter_args(s.v[0], s.vp, s.a, c.eta, d->nx, s.nyl, d->taps, nullptr,
                                  nullptr, nullptr, RedBuf{nullptr, nullptr});
      fa.gy0 = s.w0;
      fa.gny = d->ny;
      if ((rc = launch_filter_fa(fa, 0, st))) return rc;
    }
  }
  if ((rc = allgather(d))) return rc;
  for (Slab& s : d->slabs) k_fin_power<<<1, 1, 0, st>>>(s.g->st, s.gath, d->G, dot, -1);
  BSP_CU(cudaGetLastError());
  for (int i = 0; i < iters; ++i) {
    const int pin = (i - 1) & 1;
    if ((rc = halo(d, pin, {{f_pb, 1, true}}))) return rc;
    for (Slab& s : d->slabs) {
      const int* stop = &s.g->st->pow_stop;
      const double* xdiv = &s.g->st->pw[pin];
      StiffArgs q = stiff_args(s.g);
      q.a = s.a;
      q.u = (const double2*)s.pb[pin];
      q.in_div = xdiv;
      q.gate0 = stop;
      q.flags = SF_IN_MASKED;
      if (dot) {
        q.out = (double2*)s.pt;
        q.flags |= SF_D2DIV;
        BSP_CU(launch_stiff(s.g, q, st));
      } else {
        q.out = (double2*)s.pb[i & 1];
        q.flags |= SF_REDUCE;
        q.hook = HK_STORE;
        q.red_need = 3;  // x.Kx, |Kx|^2
        q.red_out = s.slot;
        q.red_y0 = s.nown0;
        q.red_y1 = s.nown1;
        BSP_CU(launch_stiff(s.g, q, st));
      }
    }
    if (dot) {
      if ((rc = halo(d, 0, {{f_pt, 1, true}}))) return rc;
      for (Slab& s : d->slabs) {
        StiffArgs q = stiff_args(s.g);
        q.a = s.a;
        q.u = (const double2*)s.pt;
        q.out = (double2*)s.pb[i & 1];
        q.dotv = (const double2*)s.pb[pin];
        q.dot_div = &s.g->st->pw[pin];
        q.gate0 = &s.g->st->pow_stop;
        q.flags = SF_REDUCE | SF_IN_MASKED;
        q.hook = HK_STORE;
        q.red_need = 6;  // |t|^2, dot
        q.red_out = s.slot;
        q.red_y0 = s.nown0;
        q.red_y1 = s.nown1;
        BSP_CU(launch_stiff(s.g, q, st));
      }
    }
    if ((rc = allgather(d))) return rc;
    for (Slab& s : d->slabs) k_fin_power<<<1, 1, 0, st>>>(s.g->st, s.gath, d->G, dot, i);
    BSP_CU(cudaGetLastError());
  }
  Slab& s0 = d->slabs[0];
  BSP_CU(cudaMemcpyAsync(d->h_st, s0.g->st, sizeof(DevState), cudaMemcpyDeviceToHost, st));
  BSP_CU(cudaStreamSynchronize(st));
  const double rho = d->h_st->rho;
  for (Slab& s : d->slabs)
    for (double** b : {&s.pb[0], &s.pb[1], &s.pt}) {
      cudaFreeAsync(*b, st);
      *b = nullptr;
    }
  // the iteration state the power iteration borrowed: pow fields only; the
  // activation / v_phys are recomputed by every iteration's filter
  BSP_CU(cudaStreamSynchronize(st));
  *h_rho = rho;
  if (!(rho > 0.0) || !std::isfinite(rho))
    return set_error(BSP_ECUDA, "slab power iteration gave rho = %g", rho);
  d->cfg.beta = 1.0 / rho;
  if (d->need_beta) {
    d->need_beta = false;
    capture_graphs(d);
  }
  return BSP_OK;
}

// Owned rows of a state field of the LAST COMPLETED iteration: 0 u, 1 v,
// 2 v_phys, 3 activation.  Local mode: the global array; NCCL mode: this
// rank's owned element rows (u: owned node rows).
extern "C" int bsp_dist_read(bsp_dist* d, int field, double* h_out) {
  if (!d || !h_out) return set_error(BSP_EINVAL, "null argument");
  const long long k = d->last_k;
  const int p = (int)(((k < 1 ? 1 : k) - 1) & 1);
  size_t off = 0;
  for (Slab& s : d->slabs) {
    const double* src = nullptr;
    size_t row = 0;
    int r0 = s.own0, r1 = s.own1;
    switch (field) {
      case 0: src = s.u[p]; row = nrow(d); r0 = s.nown0; r1 = s.nown1; break;
      case 1: src = s.v[p]; row = erow(d); break;
      case 2: src = s.vp; row = erow(d); break;
      case 3:
        if (d->cfg.algorithm == BSP_ALGO_FBTO || d->cfg.algorithm == BSP_ALGO_PFBTO_JACOBI) {
          k_act_from_vp<<<pcg_blocks(2 * s.g->E, s.g->nsm), 256, 0, d->s>>>(s.vp, s.a, s.g->E,
                                                                            d->cfg.eta);
          BSP_CU(cudaGetLastError());
        }
        src = s.a;
        row = erow(d);
        break;
      default: return set_error(BSP_EINVAL, "unknown field %d", field);
    }
    const size_t cnt = (size_t)(r1 - r0) * row;
    BSP_CU(cudaMemcpyAsync(h_out + off, src + (size_t)r0 * row, cnt * sizeof(double),
                           cudaMemcpyDeviceToHost, d->s));
    off += cnt;
  }
  BSP_CU(cudaStreamSynchronize(d->s));
  return BSP_OK;
}

// h_out[0] graphs, [1] host lambda iterations, [2] total lambda rounds,
// [3] halo rows H, [4] slabs in this process
extern "C" int bsp_dist_info(bsp_dist* d, double* h_out) {
  if (!d || !h_out) return set_error(BSP_EINVAL, "null argument");
  h_out[0] = d->graphs ? 1.0 : 0.0;
  h_out[1] = d->host_lambda_iters;
  h_out[2] = d->lam_rounds_total;
  h_out[3] = d->H;
  h_out[4] = (double)d->slabs.size();
  return BSP_OK;
}

// Device time of the communication alone: `iters` end-of-iteration halo
// exchanges (v: H rows, u: 1 node row) and `iters` all-gathers of the 8-double
// partials, each bracketed by CUDA events on the solver stream.
extern "C" int bsp_dist_comm_bench(bsp_dist* d, int iters, double* h_ms) {
  if (!d || !h_ms || iters < 1) return set_error(BSP_EINVAL, "bad argument");
  cudaEvent_t e[3];
  for (auto& x : e) BSP_CU(cudaEventCreate(&x));
  int rc;
  BSP_CU(cudaEventRecord(e[0], d->s));
  for (int i = 0; i < iters; ++i)
    if ((rc = halo(d, 0, {{f_v_next, d->H, false}, {f_u_next, 1, true}}))) return rc;
  BSP_CU(cudaEventRecord(e[1], d->s));
  for (int i = 0; i < iters; ++i)
    if ((rc = allgather(d))) return rc;
  BSP_CU(cudaEventRecord(e[2], d->s));
  BSP_CU(cudaEventSynchronize(e[2]));
  float a = 0.f, b = 0.f;
  cudaEventElapsedTime(&a, e[0], e[1]);
  cudaEventElapsedTime(&b, e[1], e[2]);
  h_ms[0] = a / iters;
  h_ms[1] = b / iters;
  for (auto& x : e) cudaEventDestroy(x);
  return BSP_OK;
}

extern "C" void* bsp_dist_stream(bsp_dist* d) { return d ? (void*)d->s : nullptr; }
