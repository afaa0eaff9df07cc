// Q4 stiffness strip kernel (see stiffness.cuh for the design summary).
//
// v2: cp.async-pipelined.  Every warp owns 32 element columns (31 emitted
// node columns) and a strip of R element rows.  The warp streams the rows it
// needs -- u (33 nodes), a (32 elements), the fixed-DOF words and, per mode,
// the load f, SIMP density v_phys, axpy base and dot vector -- through a
// private S-stage shared-memory ring with 16/8/4-byte cp.async copies.
// Out-of-grid nodes/elements are zero-filled by the copy (src-size 0), so the
// inner loop has no bounds checks: a zero activation outside the grid makes
// virtual elements contribute nothing.  S-1 rows are in flight per warp while
// the element algebra of the current row runs out of registers/shared memory.
#include "grid.cuh"
#include "solver_state.cuh"
#include "stiffness.cuh"
#include "q4.cuh"

namespace bsp {

namespace {

BSP_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

BSP_DEV void cp16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0));
}
BSP_DEV void cp8(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src),
               "r"(valid ? 8 : 0));
}
BSP_DEV void cp4(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src),
               "r"(valid ? 4 : 0));
}
BSP_DEV void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
BSP_DEV void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// shared-memory stage layout (bytes, per warp and stage)
struct StageLayout {
  int u, a, m, f, vp, base, dotv, size;
};

__host__ __device__ inline StageLayout stage_layout(int flags) {
  StageLayout L{};
  int o = 0;
  L.u = o; o += 33 * 16;
  L.a = o; o += 32 * 8;
  L.m = o; o += 16;
  L.f = -1; L.vp = -1; L.base = -1; L.dotv = -1;
  if (flags & SF_SUB_LOAD) { L.f = o; o += 32 * 16; }
  if (flags & SF_STAGE_VP) { L.vp = o; o += 32 * 8; }
  if (flags & SF_AXPY) { L.base = o; o += 32 * 16; }
  if (flags & SF_REDUCE_DOT) { L.dotv = o; o += 32 * 16; }
  L.size = o;
  return L;
}

}  // namespace

constexpr int kWarpsPerBlock = 4;
constexpr int kStages = 8;  // power of two (ring index masking)

// 2-bit fixed flags of window node k (0..32) from the staged word group:
// node (rowj + base - 1 + k) sits at bit 2*k + off of words[0..2]
BSP_DEV uint32_t win_bits(const uint32_t* words, int off, int k) {
  const int pos = off + 2 * k;
  return (words[pos >> 5] >> (pos & 31)) & 3u;
}

// F >= 0: the complete flag set is a compile-time constant (hot launch
// shapes, dead paths removed); F == -1: flags read at run time (fallback).
// SF_IN_MASKED: the input vector is zero on fixed DOFs (every vector the
// solver produces is), so the per-node input masking is skipped.
template <bool GENERIC, int F>
__global__ void __launch_bounds__(128) k_stiff(StiffArgs p, KeModes km) {
  constexpr int S = kStages;
  pdl_begin();
  if ((p.gate0 && *p.gate0) || (p.gate1 && *p.gate1)) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const int flags = F >= 0 ? F : p.flags;
  const bool inmask = (flags & SF_IN_MASKED) != 0;
  const StageLayout L = stage_layout(flags);
  const int nx = p.g.nx, ny = p.g.ny;
  const long long NX1 = nx + 1;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int warp = blockIdx.x * kWarpsPerBlock + wib;
  const int base = warp * 31;
  const int ex = base + lane - 1;   // this lane's element column / window node lane
  const int xr = ex + 1;            // right node column (emitted by lanes 0..30)
  const int y0 = blockIdx.y * p.R;
  const int y1 = min(y0 + p.R, ny);
  const bool emit_col = (lane < 31) && (xr <= nx);
  const bool own_el = (lane >= 1) && (ex >= 0) && (ex < nx);
  const bool v_node = (ex >= 0) && (ex <= nx);
  const bool v_node31 = (xr <= nx);   // lane 31's extra window node base+31
  const bool v_el = (ex >= 0) && (ex < nx);
  const bool v_emit = (xr <= nx);
  const double rinv = p.in_div ? 1.0 / *p.in_div : 1.0;
  const double dinv = p.dot_div ? 1.0 / *p.dot_div : 1.0;
  const long long nwords = (p.g.n_nodes + 15) >> 4;
  // reduction window in window-slot-0 node ids: row y's slot 0 is y*NX1+base-1
  const long long red_n0 = (long long)p.red_y0 * NX1 + base - 1;
  const long long red_n1 = (long long)p.red_y1 * NX1 + base - 1;

  unsigned char* ring = smem + (size_t)wib * S * L.size;
  const uint32_t ring_s = smem_u32(ring);

  // producer cursors: per-lane global pointers of row r_iss.  A lane whose
  // column is outside the grid keeps a fixed in-bounds pointer (stride 0) and
  // copies with src-size 0 (zero fill).
  int r_iss = y0 - 1;
  const long long r0 = y0 - 1;
  const long long rs = r0 < 0 ? 0 : r0;  // first real row; row -1 is zero-filled
  const double2* pu = v_node ? p.u + rs * NX1 + ex : p.u;
  const long long su = v_node ? NX1 : 0;
  const double2* pu31 = v_node31 ? p.u + rs * NX1 + xr : p.u;
  const long long su31 = v_node31 ? NX1 : 0;
  const double* pa = v_el ? p.a + rs * nx + ex : p.a;
  const double* pv = (v_el && L.vp >= 0) ? p.vp + rs * nx + ex : p.vp;
  const long long se = v_el ? nx : 0;
  const long long jo0 = rs * NX1 + xr;
  const long long so = v_emit ? NX1 : 0;
  const double2* pf = (L.f >= 0 && v_emit) ? p.g.load + jo0 : p.g.load;
  const double2* pb = (L.base >= 0 && v_emit) ? p.base + jo0 : p.base;
  const double2* pd = (L.dotv >= 0 && v_emit) ? p.dotv + jo0 : p.dotv;
  long long wrow = r0 * NX1 + base - 1;  // node id of window slot 0

  auto issue = [&](int st) {
    const uint32_t d = ring_s + st * L.size;
    const bool nrow = (r_iss >= 0);        // rows issued never exceed ny
    const bool er = nrow && (r_iss < ny);
    const bool vu = nrow && v_node;
    cp16(d + L.u + lane * 16, vu ? (const void*)pu : (const void*)p.u, vu);
    if (lane == 31) {
      const bool v31 = nrow && v_node31;
      cp16(d + L.u + 32 * 16, v31 ? (const void*)pu31 : (const void*)p.u, v31);
    }
    cp8(d + L.a + lane * 8, er ? (const void*)pa : (const void*)p.a, er && v_el);
    if (L.vp >= 0) cp8(d + L.vp + lane * 8, er ? (const void*)pv : (const void*)p.vp, er && v_el);
    if (lane < 4) {
      const long long w = (wrow >> 4) + lane;
      const bool vw = nrow && w >= 0 && w < nwords;
      cp4(d + L.m + lane * 4, vw ? (const void*)(p.g.fixbits + w) : (const void*)p.g.fixbits, vw);
    }
    const bool ve = nrow && v_emit;
    if (L.f >= 0) cp16(d + L.f + lane * 16, ve ? (const void*)pf : (const void*)p.g.load, ve);
    if (L.base >= 0) cp16(d + L.base + lane * 16, ve ? (const void*)pb : (const void*)p.base, ve);
    if (L.dotv >= 0) cp16(d + L.dotv + lane * 16, ve ? (const void*)pd : (const void*)p.dotv, ve);
    if (nrow) {  // the cursors start at row max(y0-1, 0)
      pu += su; pu31 += su31; pa += se; pv += se;
      pf += so; pb += so; pd += so;
    }
    ++r_iss;
    wrow += NX1;
  };

  // window nodes lane, lane+1 of a staged row (masked unless inmask)
  auto nodes = [&](const unsigned char* sp, long long w0, double2& N0, double2& N1) {
    const double2* U = reinterpret_cast<const double2*>(sp + L.u);
    N0 = U[lane];
    N1 = U[lane + 1];
    if (!inmask) {
      const uint32_t* words = reinterpret_cast<const uint32_t*>(sp + L.m);
      const int off = 2 * (int)(w0 & 15);
      N0 = apply_mask(N0, win_bits(words, off, lane));
      N1 = apply_mask(N1, win_bits(words, off, lane + 1));
    }
  };

  double s0 = 0.0, s1 = 0.0, s2 = 0.0, m3 = -INFINITY;
  const int nrows = y1 - y0 + 2;  // node rows y0-1 .. y1
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < nrows) issue(s);
    cp_commit();
  }
  cp_wait<S - 2>();
  __syncwarp();
  long long wT = r0 * NX1 + base - 1;  // window slot 0 node id of the top row
  double2 uTL, uTR;
  nodes(ring, wT, uTL, uTR);
  double accLx = 0.0, accLy = 0.0, accRx = 0.0, accRy = 0.0;
  double aPrev = 0.0;
  // output cursors start at the first emitted row y0 (advanced per emit)
  double2* po = p.out ? p.out + (long long)y0 * NX1 + xr : nullptr;
  double* ps = (flags & SF_ENERGY) ? p.sens + (long long)y0 * nx + ex : nullptr;

  auto emit = [&](long long w0, const unsigned char* sp, double asum_mine) {
    double lx = __shfl_down_sync(0xffffffffu, accLx, 1);
    double ly = __shfl_down_sync(0xffffffffu, accLy, 1);
    double as = 0.0;
    if (flags & (SF_D2DIV | SF_D1DIV)) as = asum_mine + __shfl_down_sync(0xffffffffu, asum_mine, 1);
    if (!emit_col) return;
    const uint32_t* words = reinterpret_cast<const uint32_t*>(sp + L.m);
    const uint32_t bits = win_bits(words, 2 * (int)(w0 & 15), lane + 1);
    double2 ku = apply_mask(make_double2((accRx + lx) * rinv, (accRy + ly) * rinv), bits);
    double2 t = ku;
    if (flags & SF_SUB_LOAD) {
      const double2 f = reinterpret_cast<const double2*>(sp + L.f)[lane];
      t.x -= f.x;
      t.y -= f.y;
    }
    if ((flags & SF_REDUCE) && w0 >= red_n0 && w0 < red_n1) {
      s0 += rinv * (uTR.x * ku.x + uTR.y * ku.y);
      s1 += t.x * t.x + t.y * t.y;
      // plain max (3 instructions, not 7): a NaN reaches s1 = sum t^2 and the
      // finaliser turns the max into NaN (stiff_hook), as np.max would be
      m3 = fmax(m3, fabs(t.x));
      m3 = fmax(m3, fabs(t.y));
      if (flags & SF_REDUCE_DOT) {
        const double2 dv = apply_mask(reinterpret_cast<const double2*>(sp + L.dotv)[lane], bits);
        s2 += dinv * (dv.x * ku.x + dv.y * ku.y);
      }
    }
    if (flags & (SF_D2DIV | SF_D1DIV)) {
      // d = kd * as on free DOFs (t is zero on fixed ones): one division per
      // node, the per-component constants 1/kd (1/kd^2) are kernel parameters
      const double ias = rcp_pos(as);
      if (flags & SF_D2DIV) {
        const double i2 = ias * ias;
        t.x = (bits & 1u) ? t.x : t.x * (km.ikdx2 * i2);
        t.y = (bits & 2u) ? t.y : t.y * (km.ikdy2 * i2);
      } else {
        t.x = (bits & 1u) ? t.x : t.x * (km.ikdx * ias);
        t.y = (bits & 2u) ? t.y : t.y * (km.ikdy * ias);
      }
    }
    if (flags & SF_AXPY) {
      const double2 b = reinterpret_cast<const double2*>(sp + L.base)[lane];
      t.x = b.x - p.beta * t.x;
      t.y = b.y - p.beta * t.y;
    }
    if (po) *po = t;
  };

  // step t processes element row ey = y0-1+t (stages of rows t and t+1)
  for (int t = 0; t < nrows - 1; ++t) {
    const int ey = y0 - 1 + t;
    __syncwarp();  // every lane is done with stage (t-1)%S
    if (t + S - 1 < nrows) issue((t + S - 1) & (S - 1));
    cp_commit();
    cp_wait<S - 2>();
    __syncwarp();
    const unsigned char* spT = ring + (t & (S - 1)) * L.size;
    const unsigned char* spB = ring + ((t + 1) & (S - 1)) * L.size;
    const long long wB = wT + NX1;
    double2 uBL, uBR;
    nodes(spB, wB, uBL, uBR);
    double ae = reinterpret_cast<const double*>(spT + L.a)[lane];
    if (flags & SF_A_POW) ae = act_pow(ae, p.eta);
    double2 o0, o1, o2, o3;
    double energy = 0.0;
    if (flags & SF_ENERGY) {
      element<GENERIC, true>(km, ae, uTL, uTR, uBR, uBL, o0, o1, o2, o3, energy);
      if (own_el && ey >= y0) {
        double pre = 1.0;
        if (L.vp >= 0) {
          const double vpe = reinterpret_cast<const double*>(spT + L.vp)[lane];
          const double e1 = p.eta - 1.0;  // numpy squares for **2.0
          pre = p.eta * (e1 == 2.0 ? vpe * vpe : (e1 == 1.0 ? vpe : pow(vpe, e1)));
        }
        *ps = pre * energy;
      }
      if (ey >= y0) ps += nx;
    } else {
      element<GENERIC, false>(km, ae, uTL, uTR, uBR, uBL, o0, o1, o2, o3, energy);
    }
    accLx += o0.x; accLy += o0.y;
    accRx += o1.x; accRy += o1.y;
    if (ey >= y0) {
      emit(wT, spT, aPrev + ae);
      if (po) po += NX1;
    }
    accLx = o3.x; accLy = o3.y;
    accRx = o2.x; accRy = o2.y;
    aPrev = ae;
    uTL = uBL;
    uTR = uBR;
    wT = wB;
  }
  if (y1 == ny) emit(wT, ring + ((nrows - 1) & (S - 1)) * L.size, aPrev);
  cp_wait<0>();
  pdl_trigger();

  if (flags & SF_REDUCE) {
    __shared__ double tot[4];
    if (grid_reduce4(p.rb, s0, s1, s2, m3, tot)) {
      if (threadIdx.x == 0) stiff_hook(p, tot);
    }
  }
}

template <bool GENERIC, int F>
static cudaError_t launch_t(bsp_grid* g, const StiffArgs& p, cudaStream_t s) {
  const StageLayout L = stage_layout(p.flags);
  const size_t sm = (size_t)kWarpsPerBlock * kStages * L.size;
  cudaError_t e = smem_optin((const void*)k_stiff<GENERIC, F>, 160 * 1024);
  if (e != cudaSuccess) return e;
  return launch_k(k_stiff<GENERIC, F>, g->sgrid, dim3(32 * kWarpsPerBlock), sm, s, p, g->km);
}

template <bool GENERIC>
static cudaError_t dispatch(bsp_grid* g, const StiffArgs& p, cudaStream_t s) {
  switch (p.flags) {
#define BSP_CASE(f) \
  case (f):         \
    return launch_t<GENERIC, (f)>(g, p, s);
    BSP_STIFF_SHAPES(BSP_CASE)
#undef BSP_CASE
    default:
      return launch_t<GENERIC, -1>(g, p, s);
  }
}

bool launch_stiff_tma(bsp_grid* g, const StiffArgs& p, cudaStream_t s, cudaError_t* err);

cudaError_t launch_stiff(bsp_grid* g, const StiffArgs& p0, cudaStream_t s) {
  StiffArgs p = p0;
  if (p.rhs) p.g.load = p.rhs;
  if (p.dotv) p.flags |= SF_REDUCE_DOT;
  if ((p.flags & SF_ENERGY) && p.vp) p.flags |= SF_STAGE_VP;
  if ((p.flags & SF_SUB_LOAD) && (p.in_div || p.dot_div))
    return cudaErrorInvalidValue;  // residual shapes do not scale their input (stiffness_tma.cu)
  if ((p.flags & SF_REDUCE) && p.red_need) {  // drop the totals nobody reads
    if (!(p.red_need & 8)) p.flags |= SF_RED_NOMAX;
    if (!(p.red_need & 1)) p.flags |= SF_RED_NOS0;
  }
  cudaError_t e = cudaSuccess;
  if (g->use_tma && launch_stiff_tma(g, p, s, &e)) return e;
  if (p.flags & SF_SUM_SENS) return cudaErrorNotSupported;  // TMA-only epilogue
  p.flags &= ~(SF_RED_NOMAX | SF_RED_NOS0);  // the cp.async kernel computes all totals
  return g->generic ? dispatch<true>(g, p, s) : dispatch<false>(g, p, s);
}

// diag(K(a)) with ones at fixed DOFs (fea.py:184-189), node-centric
__global__ void k_diag(GridView g, KeModes km, const double* __restrict__ a, double2* d) {
  BSP_NODE_LOOP(x, y, j, g.nx, g.ny) {
    double s = 0.0;
    if (x > 0 && y > 0) s += a[(long long)(y - 1) * g.nx + x - 1];
    if (x < g.nx && y > 0) s += a[(long long)(y - 1) * g.nx + x];
    if (x > 0 && y < g.ny) s += a[(long long)y * g.nx + x - 1];
    if (x < g.nx && y < g.ny) s += a[(long long)y * g.nx + x];
    uint32_t bits = fix_bits(g.fixbits, j);
    d[j] = make_double2((bits & 1u) ? 1.0 : km.kdx * s, (bits & 2u) ? 1.0 : km.kdy * s);
  }
}

}  // namespace bsp
