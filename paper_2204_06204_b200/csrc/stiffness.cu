// Q4 stiffness strip kernel (see stiffness.cuh for the design summary).
#include "grid.cuh"
#include "solver_state.cuh"
#include "stiffness.cuh"

namespace bsp {

namespace {

BSP_DEV double2 ld_node(const GridView& g, const double2* __restrict__ u, int col, int row,
                        double rinv) {
  double2 v = make_double2(0.0, 0.0);
  if (col >= 0 && col <= g.nx && row >= 0 && row <= g.ny) {
    long long j = (long long)row * (g.nx + 1) + col;
    v = __ldg(u + j);
    v = apply_mask(v, fix_bits(g.fixbits, j));
    v.x *= rinv;
    v.y *= rinv;
  }
  return v;
}

// left/right nodes of this lane's element at node row `row`
BSP_DEV void ld_pair(const GridView& g, const double2* __restrict__ u, int lane, int ex, int row,
                     double rinv, double2& L, double2& R) {
  R = ld_node(g, u, ex + 1, row, rinv);
  double lx = __shfl_up_sync(0xffffffffu, R.x, 1);
  double ly = __shfl_up_sync(0xffffffffu, R.y, 1);
  if (lane == 0) {
    double2 t = ld_node(g, u, ex, row, rinv);
    lx = t.x;
    ly = t.y;
  }
  L = make_double2(lx, ly);
}

BSP_DEV double ld_a(const GridView& g, const double* __restrict__ a, int ex, int ey) {
  return (ex >= 0 && ex < g.nx && ey >= 0 && ey < g.ny) ? __ldg(a + (long long)ey * g.nx + ex)
                                                        : 0.0;
}

// Element response in the Hadamard mode basis.
// nodes: 0=(ex,ey) TL, 1=(ex+1,ey) TR, 2=(ex+1,ey+1) BR, 3=(ex,ey+1) BL
template <bool GENERIC>
BSP_DEV void element(const KeModes& km, double ae, double2 n0, double2 n1, double2 n2, double2 n3,
                     double2& o0, double2& o1, double2& o2, double2& o3, double& energy) {
  // forward transform per component
  double px = n2.x - n0.x, qx = n1.x - n3.x;
  double dxx = px + qx, dyx = px - qx;
  double hgx = (n0.x + n2.x) - (n1.x + n3.x);
  double py = n2.y - n0.y, qy = n1.y - n3.y;
  double dxy = py + qy, dyy = py - qy;
  double hgy = (n0.y + n2.y) - (n1.y + n3.y);
  double fTx = 0.0, fTy = 0.0, fdxx, fdyx, fhgx, fdxy, fdyy, fhgy;
  if (!GENERIC) {
    fdxx = km.m11 * dxx + km.m16 * dyy;
    fdyy = km.m16 * dxx + km.m66 * dyy;
    fdyx = km.m22 * dyx + km.m25 * dxy;
    fdxy = km.m25 * dyx + km.m55 * dxy;
    fhgx = km.m33 * hgx;
    fhgy = km.m77 * hgy;
    energy = 0.5 * (dxx * fdxx + dyy * fdyy + dyx * fdyx + dxy * fdxy + hgx * fhgx + hgy * fhgy);
  } else {
    double Tx = (n0.x + n1.x) + (n2.x + n3.x);
    double Ty = (n0.y + n1.y) + (n2.y + n3.y);
    double m[8] = {Tx, dxx, dyx, hgx, Ty, dxy, dyy, hgy};
    double f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) s += km.M[i * 8 + j] * m[j];
      f[i] = s;
    }
    double en = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) en += m[i] * f[i];
    energy = 0.5 * en;
    fTx = f[0]; fdxx = f[1]; fdyx = f[2]; fhgx = f[3];
    fTy = f[4]; fdxy = f[5]; fdyy = f[6]; fhgy = f[7];
    fTx *= ae;
    fTy *= ae;
  }
  fdxx *= ae; fdyx *= ae; fhgx *= ae;
  fdxy *= ae; fdyy *= ae; fhgy *= ae;
  // back transform: out_i = fT + H1[i] fdx + H2[i] fdy + H3[i] fhg
  double Px = fdxx + fdyx, Qx = fdxx - fdyx;
  double Py = fdxy + fdyy, Qy = fdxy - fdyy;
  o0 = make_double2(fTx + (fhgx - Px), fTy + (fhgy - Py));
  o1 = make_double2(fTx + (Qx - fhgx), fTy + (Qy - fhgy));
  o2 = make_double2(fTx + (Px + fhgx), fTy + (Py + fhgy));
  o3 = make_double2(fTx - (Qx + fhgx), fTy - (Qy + fhgy));
}

}  // namespace

template <bool GENERIC>
__global__ void __launch_bounds__(128) k_stiff(StiffArgs p, KeModes km) {
  if ((p.gate0 && *p.gate0) || (p.gate1 && *p.gate1)) return;
  const GridView g = p.g;
  const int nx = g.nx, ny = g.ny;
  const int lane = threadIdx.x & 31;
  const int warp = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int base = warp * 31;
  const int ex = base + lane - 1;
  const int xr = ex + 1;
  const int y0 = blockIdx.y * p.R;
  const int y1 = min(y0 + p.R, ny);
  const long long NX1 = nx + 1;
  const int flags = p.flags;
  const double rinv = p.in_div ? 1.0 / *p.in_div : 1.0;
  const double dinv = p.dot_div ? 1.0 / *p.dot_div : 1.0;
  const bool emit_col = (lane < 31) && (xr <= nx);
  const bool own_el = (lane >= 1) && (ex >= 0) && (ex < nx);

  double s0 = 0.0, s1 = 0.0, s2 = 0.0, m3 = -INFINITY;

  double2 uTL, uTR, uBL, uBR;
  ld_pair(g, p.u, lane, ex, y0 - 1, rinv, uTL, uTR);
  ld_pair(g, p.u, lane, ex, y0, rinv, uBL, uBR);
  double accLx = 0.0, accLy = 0.0, accRx = 0.0, accRy = 0.0;
  double aPrev = ld_a(g, p.a, ex, y0 - 1);
  double aCur = aPrev;

  auto emit = [&](int row, double asum_mine) {
    // node (xr,row) = my right partial + right neighbour's left partial
    double lx = __shfl_down_sync(0xffffffffu, accLx, 1);
    double ly = __shfl_down_sync(0xffffffffu, accLy, 1);
    double as = 0.0;
    if (flags & SF_D2DIV) as = asum_mine + __shfl_down_sync(0xffffffffu, asum_mine, 1);
    if (!emit_col) return;
    const long long j = (long long)row * NX1 + xr;
    const uint32_t bits = fix_bits(g.fixbits, j);
    double2 ku = make_double2(accRx + lx, accRy + ly);
    ku = apply_mask(ku, bits);
    double2 t = ku;
    if (flags & SF_SUB_LOAD) {
      double2 f = __ldg(g.load + j);
      t.x -= f.x;
      t.y -= f.y;
    }
    if (flags & SF_REDUCE) {
      s0 += uTR.x * ku.x + uTR.y * ku.y;
      s1 += t.x * t.x + t.y * t.y;
      m3 = nanmax(m3, fabs(t.x));
      m3 = nanmax(m3, fabs(t.y));
      if (p.dotv) {
        double2 dv = apply_mask(__ldg(p.dotv + j), bits);
        s2 += dinv * (dv.x * ku.x + dv.y * ku.y);
      }
    }
    if (flags & SF_D2DIV) {
      double dx = (bits & 1u) ? 1.0 : km.kdx * as;
      double dy = (bits & 2u) ? 1.0 : km.kdy * as;
      t.x = t.x / (dx * dx);
      t.y = t.y / (dy * dy);
    }
    if (flags & SF_AXPY) {
      double2 b = __ldg(p.base + j);
      t.x = b.x - p.beta * t.x;
      t.y = b.y - p.beta * t.y;
    }
    if (p.out) p.out[j] = t;
  };

  for (int ey = y0 - 1; ey < y1; ++ey) {
    aCur = ld_a(g, p.a, ex, ey);
    double2 nL = make_double2(0.0, 0.0), nR = nL;
    if (ey + 1 < y1) ld_pair(g, p.u, lane, ex, ey + 2, rinv, nL, nR);
    double2 o0, o1, o2, o3;
    double energy;
    element<GENERIC>(km, aCur, uTL, uTR, uBR, uBL, o0, o1, o2, o3, energy);
    if ((flags & SF_ENERGY) && own_el && ey >= y0) {
      double pre = 1.0;
      if (p.vp) {
        double vpe = __ldg(p.vp + (long long)ey * nx + ex);
        const double e1 = p.eta - 1.0;  // numpy squares for **2.0
        pre = p.eta * (e1 == 2.0 ? vpe * vpe : (e1 == 1.0 ? vpe : pow(vpe, e1)));
      }
      p.sens[(long long)ey * nx + ex] = pre * energy;
    }
    accLx += o0.x; accLy += o0.y;
    accRx += o1.x; accRy += o1.y;
    if (ey >= y0) emit(ey, aPrev + aCur);
    accLx = o3.x; accLy = o3.y;
    accRx = o2.x; accRy = o2.y;
    aPrev = aCur;
    uTL = uBL; uTR = uBR;
    uBL = nL; uBR = nR;
  }
  if (y1 == ny) emit(ny, aPrev);

  if (flags & SF_REDUCE) {
    __shared__ double tot[4];
    if (grid_reduce4(p.rb, s0, s1, s2, m3, tot)) {
      if (threadIdx.x == 0) {
        DevState* st = p.st;
        switch (p.hook) {
          case HK_STORE:
            p.red_out[0] = tot[0]; p.red_out[1] = tot[1];
            p.red_out[2] = tot[2]; p.red_out[3] = tot[3];
            break;
          case HK_RESIDUAL: {
            double comp = 0.5 * tot[0];
            double rinf = tot[3];
            st->compliance = comp;
            st->res_inf = rinf;
            double nb = sqrt(tot[1]);
            st->rnorm = nb;
            st->norms[0] = nb;
            st->kry_count = 0;
            st->kry_stop = (nb == 0.0) ? 1 : 0;
            if (!(isfinite(rinf) && isfinite(comp))) {
              st->done = 2;
              st->div_k = st->k;
            }
          } break;
          case HK_KRYLOV: {
            double m = sqrt(tot[1]);
            if (m == 0.0) {
              st->kry_stop = 1;
            } else {
              st->norms[p.hook_i + 1] = m;
              st->kry_count = p.hook_i + 1;
            }
          } break;
          case HK_POWER:
          case HK_POWER_DOT: {
            double n = sqrt(tot[1]);
            st->rho = (p.hook == HK_POWER) ? tot[0] : tot[2];
            st->pw[p.hook_i] = n;
            if (n == 0.0) st->pow_stop = 1;
          } break;
        }
      }
    }
  }
}

cudaError_t launch_stiff(bsp_grid* g, const StiffArgs& p, cudaStream_t s) {
  if (g->generic)
    k_stiff<true><<<g->sgrid, 128, 0, s>>>(p, g->km);
  else
    k_stiff<false><<<g->sgrid, 128, 0, s>>>(p, g->km);
  return cudaGetLastError();
}

// diag(K(a)) with ones at fixed DOFs (fea.py:184-189), node-centric
__global__ void k_diag(GridView g, KeModes km, const double* __restrict__ a, double2* d) {
  long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (j >= g.n_nodes) return;
  int x = (int)(j % (g.nx + 1)), y = (int)(j / (g.nx + 1));
  double s = 0.0;
  // incident elements in reference scatter order is irrelevant at 1e-16
  if (x > 0 && y > 0) s += a[(long long)(y - 1) * g.nx + x - 1];
  if (x < g.nx && y > 0) s += a[(long long)(y - 1) * g.nx + x];
  if (x > 0 && y < g.ny) s += a[(long long)y * g.nx + x - 1];
  if (x < g.nx && y < g.ny) s += a[(long long)y * g.nx + x];
  uint32_t bits = fix_bits(g.fixbits, j);
  d[j] = make_double2((bits & 1u) ? 1.0 : km.kdx * s, (bits & 2u) ? 1.0 : km.kdy * s);
}

}  // namespace bsp
