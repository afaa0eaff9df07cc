// Device pieces of the projected design update shared by highlevel.cu and the
// fused small-grid iteration (fused.cu): deterministic grid totals of a
// cooperative grid, the trial point, and the safeguarded regime-Newton lambda
// search of k_hl_fix (projection.py:65-91) as a device function.
#pragma once
#include <cooperative_groups.h>

#include "highlevel.cuh"
#include "solver_state.cuh"

namespace bsp {
namespace cg = cooperative_groups;

namespace {

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
  G.sync();  // all blocks read `part` before it is reused
}

BSP_DEV double clampd(double x, double lo, double hi) { return fmin(fmax(x, lo), hi); }

BSP_DEV double step_alpha(const HLArgs& p) {
  const DevState* st = p.st;
  return p.alphas ? p.alphas[st->k - st->k_base] : p.alpha;
}

BSP_DEV double g_mean(const HLArgs& p) {
  return (p.g && p.mean_projection) ? p.st->gsum / p.n_active : 0.0;
}


// Calls f(e, v[e], g[e], active[e]) for this thread's elements: 4 consecutive
// elements per trip with 16-byte loads when the arrays allow it.
template <class F>
BSP_DEV void for_each_element(const HLArgs& p, F&& f) {
  const long long E = p.E;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nthr = (long long)gridDim.x * blockDim.x;
  const bool has_g = p.g != nullptr;
  const bool vec = ((reinterpret_cast<uintptr_t>(p.v) | reinterpret_cast<uintptr_t>(p.v_next) |
                     (has_g ? reinterpret_cast<uintptr_t>(p.g) : 0)) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(p.active) & 3) == 0;
  long long e0 = 0;
  if (vec) {
    const long long E4 = E & ~3ll;
    for (long long e = 4 * tid; e < E4; e += 4 * nthr) {
      const double2 va = __ldcg(reinterpret_cast<const double2*>(p.v + e));
      const double2 vb = __ldcg(reinterpret_cast<const double2*>(p.v + e + 2));
      double2 ga = make_double2(0.0, 0.0), gb = ga;
      if (has_g) {
        ga = __ldcg(reinterpret_cast<const double2*>(p.g + e));
        gb = __ldcg(reinterpret_cast<const double2*>(p.g + e + 2));
      }
      uchar4 m = make_uchar4(1, 1, 1, 1);
      if (p.active) m = *reinterpret_cast<const uchar4*>(p.active + e);
      f(e, va.x, ga.x, m.x != 0);
      f(e + 1, va.y, ga.y, m.y != 0);
      f(e + 2, vb.x, gb.x, m.z != 0);
      f(e + 3, vb.y, gb.y, m.w != 0);
    }
    e0 = E4;
  }
  for (long long e = e0 + tid; e < E; e += nthr)
    f(e, p.v[e], has_g ? p.g[e] : 0.0, !p.active || p.active[e]);
}

BSP_DEV double trial_w(const HLArgs& p, double v, double g, double alpha, double mean) {
  if (!p.g) return v;
  return v + alpha * (p.mean_projection ? g - mean : g);
}

// k_hl_fix's body on a cooperative grid G (all blocks call it together):
// the lambda search, the rewrite of v_next and the record row.
// The lambda search of k_hl_fix run by ONE block (the last block of
// k_hl_write or k_hl_adj4) over all elements: for small grids (E <= kSmallFix) a few
// passes over L2-resident data cost less than launching k_hl_fix every
// iteration.  Same safeguarded regime-Newton, block reductions instead of
// grid syncs; then the rewrite and the record row.
BSP_DEV void block_lambda(const HLArgs& p, const double* tot6, double alpha, double mean) {
  const double lo = p.lo, hi = p.hi, budget = p.budget;
  const long long E = p.E;
  __shared__ double bt[4];
  double L = 0.0, U = tot6[5] - lo;
  const double guess = tot6[2] > 0.0 ? (tot6[0] - budget) / tot6[2] : -1.0;
  double lam = (guess > L && guess < U) ? guess : 0.5 * (L + U);
  int rounds;
  for (rounds = 1; rounds <= 200; ++rounds) {
    double v4[4] = {0.0, 0.0, 0.0, 0.0};  // S_mid, n_mid, n_lo, n_hi
    for (long long e = threadIdx.x; e < E; e += blockDim.x) {
      if (p.active && !p.active[e]) continue;
      const double w = trial_w(p, p.v[e], p.g ? p.g[e] : 0.0, alpha, mean);
      const double d = w - lam;
      if (d <= lo) v4[2] += 1.0;
      else if (d >= hi) v4[3] += 1.0;
      else { v4[0] += w; v4[1] += 1.0; }
    }
    block_reduce_nn<4, 4>(v4);
    if (threadIdx.x == 0)
      for (int i = 0; i < 4; ++i) bt[i] = v4[i];
    __syncthreads();
    const double smid = bt[0], nmid = bt[1], nlo = bt[2], nhi = bt[3];
    __syncthreads();
    const double f = smid - nmid * lam + nlo * lo + nhi * hi;
    if (f > budget) L = lam; else U = lam;
    double next;
    if (nmid > 0.0) {
      const double root = (smid + nlo * lo + nhi * hi - budget) / nmid;
      if (fabs(root - lam) <= 1e-15 * fmax(1.0, fabs(lam))) {
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
    if (!(U - L > 1e-15 * fmax(1.0, fabs(U))) || next == lam) {
      lam = (f > budget) ? U : lam;
      break;
    }
    lam = next;
  }
  if (lam < 0.0) lam = 0.0;
  double v4[4] = {0.0, 0.0, 0.0, -INFINITY};  // volume, -, -, max dv
  for (long long e = threadIdx.x; e < E; e += blockDim.x) {
    const double v = p.v[e];
    const bool act = !p.active || p.active[e];
    const double out = act ? clampd(trial_w(p, v, p.g ? p.g[e] : 0.0, alpha, mean) - lam, lo, hi) : v;
    p.v_next[e] = out;
    v4[3] = nanmax(v4[3], fabs(out - v));
    v4[0] += v;
  }
  block_reduce_nn<4, 3>(v4);
  if (threadIdx.x == 0) hl_finalize(p, fmax(v4[3], 0.0), v4[0], lam, rounds);
}


BSP_DEV void hl_fix_body(const HLArgs& p, cg::grid_group& G) {
  DevState* st = p.st;
  __shared__ double tot[4];
  const double lo = p.lo, hi = p.hi, budget = p.budget;
  const double alpha = step_alpha(p), mean = g_mean(p);
  double L = 0.0, U = st->scratch[3] - lo;
  const double guess = st->scratch[4];
  double lam = (guess > L && guess < U) ? guess : 0.5 * (L + U);
  int rounds;
  for (rounds = 1; rounds <= 200; ++rounds) {
    double smid = 0.0, nmid = 0.0, nlo = 0.0, nhi = 0.0;
    for_each_element(p, [&](long long, double v, double g, bool act) {
      if (!act) return;
      const double w = trial_w(p, v, g, alpha, mean);
      const double d = w - lam;
      if (d <= lo) nlo += 1.0;
      else if (d >= hi) nhi += 1.0;
      else { smid += w; nmid += 1.0; }
    });
    grid_total<false>(G, p.part, smid, nmid, nlo, nhi, tot);
    smid = tot[0]; nmid = tot[1]; nlo = tot[2]; nhi = tot[3];
    const double f = smid - nmid * lam + nlo * lo + nhi * hi;
    if (f > budget) L = lam; else U = lam;
    double next;
    if (nmid > 0.0) {
      const double root = (smid + nlo * lo + nhi * hi - budget) / nmid;
      // split consistent: root of this piece.  The sums are only exact to a
      // few ulps of the budget, so once the Newton step is below 1e-15 (in
      // density units) the remaining wobble is rounding noise -- stop rather
      // than bisect the noise down to adjacent floats (up to 200 grid syncs).
      if (fabs(root - lam) <= 1e-15 * fmax(1.0, fabs(lam))) {
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
    if (!(U - L > 1e-15 * fmax(1.0, fabs(U))) || next == lam) {
      lam = (f > budget) ? U : lam;
      break;
    }
    lam = next;
  }
  if (lam < 0.0) lam = 0.0;
  double dv = 0.0, vol = 0.0;
  for_each_element(p, [&](long long e, double v, double g, bool act) {
    const double out = act ? clampd(trial_w(p, v, g, alpha, mean) - lam, lo, hi) : v;
    p.v_next[e] = out;
    dv = nanmax(dv, fabs(out - v));
    vol += v;
  });
  grid_total<true>(G, p.part, vol, 0.0, 0.0, dv, tot);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->lam_needed = 0;
    hl_finalize(p, tot[3], tot[0], lam, rounds);
  }
}

}  // namespace
}  // namespace bsp
