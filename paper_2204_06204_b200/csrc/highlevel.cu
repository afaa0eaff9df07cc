// Projected design update: mean projection + bounded-simplex projection +
// termination measurements.  Restates reference solvers.py:193-197
// (mean_project), solvers.py:284-302 (high_level_step), projection.py:50-91
// (project_simplex) and the record / termination lines solvers.py:464-475.
//
// Common path (box early exit, projection.py:59-61 -- SURVEY §0.1-4 measured
// 99.6% of iterations): ONE streaming kernel, k_hl_write.  It forms
// w = v + alpha (g - mean) (mean of g over active elements was reduced by the
// adjoint-filter epilogue), writes clamp(w) optimistically and reduces
// (box sum, max w, max |dv|, sum v) with a deterministic last-block
// finalisation that writes the ConvergenceRecord row and the termination flag.
// If the box sum exceeds the budget the finaliser raises `lam_needed` instead
// and the cooperative k_hl_fix kernel -- which otherwise exits at once --
// solves  sum clamp(w - lam, lo, hi) = budget  by a safeguarded regime-Newton
// iteration: at a trial lam one grid reduction yields the regime split
// (n_lo, n_mid, n_hi, S_mid); the root of that linear piece,
// (S_mid + n_lo lo + n_hi hi - budget)/n_mid, is exact once the split is
// right (the same piece the reference's sorted-breakpoint sweep selects), and
// an [L,U] bracket with bisection guarantees termination.  All reductions are
// fixed-order trees -> bitwise deterministic.
#include <cooperative_groups.h>

#include <cstdlib>

#include "highlevel.cuh"
#include "hl_device.cuh"
#include "solver_state.cuh"

namespace bsp {

namespace {

}  // namespace

// optimistic box projection + measurements (common path).  Streaming: each
// thread takes 4 consecutive elements per trip (two 16-byte loads per array
// when aligned) so that enough bytes are in flight per SM to reach HBM rate.
__global__ void __launch_bounds__(256) k_hl_write(HLArgs p) {
  pdl_begin();
  DevState* st = p.st;
  if (st->done) return;
  const double alpha = step_alpha(p), mean = g_mean(p);
  const double lo = p.lo, hi = p.hi;
  // sums: box sum, volume, interior count, interior sum of w; maxima: dv, w
  double bs = 0.0, vol = 0.0, nmid = 0.0, smid = 0.0, dv = 0.0, wmax = -INFINITY;
  const bool has_g = p.g != nullptr;
  auto one = [&](double v, double g, bool act, double& out) {
    out = v;
    if (act) {
      const double w = has_g ? v + alpha * (p.mean_projection ? g - mean : g) : v;
      out = clampd(w, lo, hi);
      bs += out;
      wmax = nanmax(wmax, w);
      if (w > lo && w < hi) { nmid += 1.0; smid += w; }
    }
    dv = nanmax(dv, fabs(out - v));
    vol += v;
  };
  const long long E = p.E;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nthr = (long long)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(p.v) | reinterpret_cast<uintptr_t>(p.v_next) |
                     (has_g ? reinterpret_cast<uintptr_t>(p.g) : 0)) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(p.active) & 3) == 0;
  long long e0 = 0;
  if (vec) {
    const long long E4 = E & ~3ll;
    for (long long e = 4 * tid; e < E4; e += 4 * nthr) {
      const double2 va = __ldcs(reinterpret_cast<const double2*>(p.v + e));
      const double2 vb = __ldcs(reinterpret_cast<const double2*>(p.v + e + 2));
      double2 ga = make_double2(0.0, 0.0), gb = ga;
      if (has_g) {
        ga = __ldcs(reinterpret_cast<const double2*>(p.g + e));
        gb = __ldcs(reinterpret_cast<const double2*>(p.g + e + 2));
      }
      bool a0 = true, a1 = true, a2 = true, a3 = true;
      if (p.active) {
        const uchar4 m = *reinterpret_cast<const uchar4*>(p.active + e);  // E4 aligned by 4
        a0 = m.x; a1 = m.y; a2 = m.z; a3 = m.w;
      }
      double2 oa, ob;
      one(va.x, ga.x, a0, oa.x);
      one(va.y, ga.y, a1, oa.y);
      one(vb.x, gb.x, a2, ob.x);
      one(vb.y, gb.y, a3, ob.y);
      __stcs(reinterpret_cast<double2*>(p.v_next + e), oa);
      __stcs(reinterpret_cast<double2*>(p.v_next + e + 2), ob);
    }
    e0 = E4;
  }
  for (long long e = e0 + tid; e < E; e += nthr) {
    double out;
    one(p.v[e], has_g ? p.g[e] : 0.0, !p.active || p.active[e], out);
    p.v_next[e] = out;
  }
  pdl_trigger();
  __shared__ double tot[6];
  double v6[6] = {bs, vol, nmid, smid, dv, wmax};
  if (grid_reduce_nn<6, 4>(p.rb, v6, tot)) {  // last block, all its threads
    if (p.defer_out) {
      if (threadIdx.x == 0)
        for (int i = 0; i < 6; ++i) p.defer_out[i] = tot[i];
    } else if (tot[0] > p.budget && p.E <= p.small_fix && !p.host_lambda) {
      block_lambda(p, tot, alpha, mean);  // small grids: no separate k_hl_fix launch
    } else if (threadIdx.x == 0) {
      hl_write_hook(p, tot);
    }
  }
}

// rare branch: the budget is active -> lambda search, rewrite, finalize
__global__ void __launch_bounds__(256) k_hl_fix(HLArgs p) {
  pdl_begin();  // launched early under PDL: wait for the predecessor's writes
  DevState* st = p.st;
  if (st->done || !st->lam_needed) return;  // uniform across the grid
  cg::grid_group G = cg::this_grid();
  hl_fix_body(p, G);
}

// sum of g over active elements -> st->gsum (standalone high_level_step)
__global__ void __launch_bounds__(256) k_masked_sum(const double* g, const uint8_t* active,
                                                    long long n, RedBuf rb, DevState* st) {
  double s = 0.0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += stride)
    if (!active || active[e]) s += g[e];
  __shared__ double tot[4];
  if (grid_reduce4(rb, s, 0.0, 0.0, -INFINITY, tot) && threadIdx.x == 0) st->gsum = tot[0];
}

int highlevel_blocks(int device) {
  int nsm = 0, per = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_hl_fix, 256, 0);
  if (per < 1) per = 1;
  if (per > 4) per = 4;
  return nsm * per;
}

int write_blocks(long long E, int nsm) {
  long long b = (E + 1023) / 1024;  // 4 elements per thread per trip
  if (b > 8ll * nsm) b = 8ll * nsm;
  if (b < 1) b = 1;
  return (int)b;
}

long long small_fix_limit() {
  static const long long v = [] {
    const char* e = getenv("BSP_SMALL_FIX");
    return e ? atoll(e) : kSmallFix;
  }();
  return v;
}

cudaError_t launch_hl_write(const HLArgs& a0, int nsm, cudaStream_t s) {
  HLArgs a = a0;
  a.small_fix = 0;
  return launch_k(k_hl_write, dim3(write_blocks(a.E, nsm)), dim3(256), 0, s, a);
}

cudaError_t launch_hl_fix(const HLArgs& a, int fix_blocks, cudaStream_t s) {
  // cooperative (grid syncs in the lambda search), and under PDL launched
  // while its predecessor finishes (pdl_begin at the top waits for it)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(fix_blocks);
  cfg.blockDim = dim3(256);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, k_hl_fix, a);
}

cudaError_t launch_highlevel(const HLArgs& a0, int fix_blocks, int nsm, cudaStream_t s) {
  HLArgs a = a0;
  a.small_fix = small_fix_limit();
  cudaError_t e = launch_k(k_hl_write, dim3(write_blocks(a.E, nsm)), dim3(256), 0, s, a);
  if (e != cudaSuccess || a.E <= a.small_fix) return e;  // small grids: k_hl_write's last block
  return launch_hl_fix(a, fix_blocks, s);
}

}  // namespace bsp
