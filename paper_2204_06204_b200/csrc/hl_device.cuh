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
// g = C^T s for the fused path (k_hl_adj4 stores no g): the y pass of
// s / sy, / sx, the x pass -- the sums of k_filter_adj4 / k_hl_adj4 in their
// order.  v_next is the scratch (the rewrite below overwrites it).
BSP_DEV double fix_mass(const FilterTaps& w, int i, int len) {
  const int k0 = max(0, w.r - i);
  const int k1 = min(w.size, len - i + w.r);
  return w.cum[k1] - w.cum[k0];
}

BSP_DEV void fix_regather_g(const HLArgs& p, cg::grid_group& G) {
  constexpr int K = 7, R = 3;  // the fused path runs radius-3 filters only
  const FilterTaps& w = p.taps;
  const int nx = p.nx, ny = p.ny;
  double* tmp = p.v_next;
  double* g = const_cast<double*>(p.g);
  double wk[K];
#pragma unroll
  for (int k = 0; k < K; ++k) wk[k] = w.w[k];
  const double is_in = 1.0 / (w.cum[w.size] - w.cum[0]);  // interior 1 / mass
  // rows over blocks, columns over threads (no index division)
  for (int y = blockIdx.x; y < ny; y += gridDim.x) {
    double isy[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int yy = y + k - R;
      isy[k] = (yy < 0 || yy >= ny) ? 0.0
               : ((yy >= R && yy < ny - R) ? is_in : 1.0 / fix_mass(w, yy, ny));
    }
    const double* src = p.g_src + (long long)y * nx;
    for (int x = threadIdx.x; x < nx; x += blockDim.x) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int yy = y + k - R;
        acc += wk[k] * (((yy >= 0 && yy < ny) ? src[(long long)(k - R) * nx + x] : 0.0) * isy[k]);
      }
      const double isx = (x >= R && x < nx - R) ? is_in : 1.0 / fix_mass(w, x, nx);
      tmp[(long long)y * nx + x] = acc * isx;
    }
  }
  G.sync();
  for (int y = blockIdx.x; y < ny; y += gridDim.x) {
    const double* row = tmp + (long long)y * nx;
    for (int x = threadIdx.x; x < nx; x += blockDim.x) {
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int xx = x + k - R;
        acc += wk[k] * ((xx >= 0 && xx < nx) ? row[xx] : 0.0);
      }
      g[(long long)y * nx + x] = acc;
    }
  }
  G.sync();
}

BSP_DEV void hl_fix_body(const HLArgs& p, cg::grid_group& G) {
  DevState* st = p.st;
  __shared__ double tot[4];
  if (p.g_src) fix_regather_g(p, G);
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
    if (!(U - L > 0.0) || next == lam) {
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
