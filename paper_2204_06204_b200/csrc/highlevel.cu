// Projected design update: mean projection + bounded-simplex projection +
// termination measurements, as ONE cooperative (grid-synchronised) kernel.
// Restates reference solvers.py:193-197 (mean_project), solvers.py:284-302
// (high_level_step), projection.py:50-91 (project_simplex) and the record /
// termination lines solvers.py:464-475.
//
// Projection: the box early exit (projection.py:59-61) decides almost every
// iteration.  When the budget is active we solve
//   f(lam) = sum clamp(w - lam, lo, hi) = budget
// by a safeguarded regime-Newton iteration: at a trial lam one grid reduction
// yields the regime split (n_lo, n_mid, n_hi, S_mid); the root of the linear
// piece for that split, (S_mid + n_lo lo + n_hi hi - budget)/n_mid, is exact
// as soon as the split is right (the reference's sorted-breakpoint sweep finds
// the same piece).  A [L,U] bracket with bisection fallback guarantees
// termination.  Every reduction is a fixed-order tree -> deterministic.
#include <cooperative_groups.h>

#include "highlevel.cuh"
#include "solver_state.cuh"

namespace cg = cooperative_groups;

namespace bsp {

namespace {

// all blocks compute the same totals in the same order (deterministic)
template <bool MAX3>
BSP_DEV void grid_total(cg::grid_group& G, double* part, double v0, double v1, double v2,
                        double v3, double* out /* shared [4] */) {
  block_reduce4<MAX3>(v0, v1, v2, v3);
  const int tid = threadIdx.x;
  if (tid == 0) {
    double* p = part + 4ull * blockIdx.x;
    p[0] = v0; p[1] = v1; p[2] = v2; p[3] = v3;
  }
  G.sync();
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = MAX3 ? -INFINITY : 0.0;
  for (unsigned b = tid; b < gridDim.x; b += blockDim.x) {
    const double* p = part + 4ull * b;
    a0 += __ldcg(p);
    a1 += __ldcg(p + 1);
    a2 += __ldcg(p + 2);
    a3 = MAX3 ? nanmax(a3, __ldcg(p + 3)) : a3 + __ldcg(p + 3);
  }
  block_reduce4<MAX3>(a0, a1, a2, a3);
  if (tid == 0) { out[0] = a0; out[1] = a1; out[2] = a2; out[3] = a3; }
  // every block must finish reading `part` before it is reused
  G.sync();
}

BSP_DEV double clampd(double x, double lo, double hi) { return fmin(fmax(x, lo), hi); }

}  // namespace

__global__ void __launch_bounds__(256) k_highlevel(HLArgs p) {
  cg::grid_group G = cg::this_grid();
  DevState* st = p.st;
  if (st && st->done) return;  // uniform across the grid
  __shared__ double tot[4];
  const long long E = p.E;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const double lo = p.lo, hi = p.hi, budget = p.budget;
  const double alpha = st ? p.alphas[st->k - st->k_base] : p.alpha;
  const bool has_g = p.g != nullptr;

  // phase A: mean of g over active elements (solvers.py:195-197, 297-299)
  double mean = 0.0;
  if (has_g && p.mean_projection) {
    double s = 0.0;
    for (long long e = t0; e < E; e += stride)
      if (!p.active || p.active[e]) s += p.g[e];
    grid_total<false>(G, p.part, s, 0.0, 0.0, 0.0, tot);
    mean = tot[0] / (double)p.n_active;
  }
  auto trial = [&](long long e) -> double {
    double v = p.v[e];
    if (!has_g) return v;
    double step = p.mean_projection ? (p.g[e] - mean) : p.g[e];
    return v + alpha * step;
  };

  // phase B: box projection sum and max(w) (projection.py:59-61, 40)
  double bs = 0.0, wmax = -INFINITY;
  for (long long e = t0; e < E; e += stride) {
    if (p.active && !p.active[e]) continue;
    double w = trial(e);
    bs += clampd(w, lo, hi);
    wmax = nanmax(wmax, w);
  }
  grid_total<true>(G, p.part, bs, 0.0, 0.0, wmax, tot);
  const double boxsum = tot[0];
  wmax = tot[3];

  // phase C: lambda (rare branch)
  double lam = 0.0;
  int rounds = 0;
  if (boxsum > budget) {
    double L = 0.0, U = wmax - lo;
    lam = 0.5 * (L + U);
    for (rounds = 1; rounds <= 200; ++rounds) {
      double smid = 0.0, nmid = 0.0, nlo = 0.0, nhi = 0.0;
      for (long long e = t0; e < E; e += stride) {
        if (p.active && !p.active[e]) continue;
        double w = trial(e);
        double d = w - lam;
        if (d <= lo) nlo += 1.0;
        else if (d >= hi) nhi += 1.0;
        else { smid += w; nmid += 1.0; }
      }
      grid_total<false>(G, p.part, smid, nmid, nlo, nhi, tot);
      smid = tot[0]; nmid = tot[1]; nlo = tot[2]; nhi = tot[3];
      double f = smid - nmid * lam + nlo * lo + nhi * hi;
      if (f > budget) L = lam; else U = lam;
      double next;
      if (nmid > 0.0) {
        double root = (smid + nlo * lo + nhi * hi - budget) / nmid;
        if (root == lam) break;            // split consistent: exact root
        next = (root > L && root < U) ? root : 0.5 * (L + U);
      } else {
        next = 0.5 * (L + U);
      }
      if (!(U - L > 0.0) || next == lam) { lam = (f > budget) ? U : lam; break; }
      lam = next;
    }
    if (lam < 0.0) lam = 0.0;
  }

  // phase D: write v_next, measure dv_inf and volume (solvers.py:464-466)
  double dv = 0.0, vol = 0.0;
  for (long long e = t0; e < E; e += stride) {
    double v = p.v[e];
    double out = v;
    if (!p.active || p.active[e]) out = clampd(trial(e) - lam, lo, hi);
    p.v_next[e] = out;
    dv = nanmax(dv, fabs(out - v));
    vol += v;
  }
  grid_total<true>(G, p.part, vol, 0.0, 0.0, dv, tot);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (p.diag) {
      p.diag[0] = mean; p.diag[1] = boxsum; p.diag[2] = lam; p.diag[3] = (double)rounds;
      p.diag[4] = tot[3]; p.diag[5] = tot[0];
    }
    if (st) {
      const long long k = st->k;
      RecRow& row = p.rec[k - st->k_base];
      row.compliance = st->compliance;
      row.res_inf = st->res_inf;
      row.dv_inf = tot[3];
      row.volume = tot[0];
      st->dv_inf = tot[3];
      st->volume = tot[0];
      st->lambda = lam;
      st->lam_rounds = rounds;
      if (tot[3] < p.tol_dv && st->res_inf < p.tol_res) {
        st->done = 1;
        st->conv_k = k;
      }
      st->k = k + 1;
    }
  }
}

int highlevel_blocks(int device) {
  int nsm = 0, per = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_highlevel, 256, 0);
  if (per < 1) per = 1;
  if (per > 4) per = 4;
  return nsm * per;
}

cudaError_t launch_highlevel(const HLArgs& a, int blocks, cudaStream_t s) {
  HLArgs args = a;
  void* kp[] = {&args};
  return cudaLaunchCooperativeKernel((const void*)k_highlevel, dim3(blocks), dim3(256), kp, 0, s);
}

}  // namespace bsp
