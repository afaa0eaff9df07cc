// Shared device pieces of the Q4 stiffness kernels (stiffness.cu: cp.async
// strip kernel; stiffness_tma.cu: TMA strip kernel).
#pragma once
#include "solver_state.cuh"
#include "stiffness.cuh"

namespace bsp {

// Element response in the per-component Hadamard mode basis (common.cuh).
// nodes: 0=(ex,ey) TL, 1=(ex+1,ey) TR, 2=(ex+1,ey+1) BR, 3=(ex,ey+1) BL
template <bool GENERIC, bool ENERGY>
BSP_DEV void element(const KeModes& km, double ae, double2 n0, double2 n1, double2 n2, double2 n3,
                     double2& o0, double2& o1, double2& o2, double2& o3, double& energy) {
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
    if (ENERGY)
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
    if (ENERGY) {
      double en = 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) en += m[i] * f[i];
      energy = 0.5 * en;
    }
    fTx = f[0] * ae; fdxx = f[1]; fdyx = f[2]; fhgx = f[3];
    fTy = f[4] * ae; fdxy = f[5]; fdyy = f[6]; fhgy = f[7];
  }
  fdxx *= ae; fdyx *= ae; fhgx *= ae;
  fdxy *= ae; fdyy *= ae; fhgy *= ae;
  double Px = fdxx + fdyx, Qx = fdxx - fdyx;
  double Py = fdxy + fdyy, Qy = fdxy - fdyy;
  if (!GENERIC) {
    // the isotropic Ke has no translation mode (fT = 0): the generic form's
    // 0 + x would cost 8 DADDs per element (the compiler must keep them: they
    // turn -0 into +0); only the sign of an exact zero differs
    o0 = make_double2(fhgx - Px, fhgy - Py);
    o1 = make_double2(Qx - fhgx, Qy - fhgy);
    o2 = make_double2(Px + fhgx, Py + fhgy);
    o3 = make_double2(-(Qx + fhgx), -(Qy + fhgy));
    return;
  }
  o0 = make_double2(fTx + (fhgx - Px), fTy + (fhgy - Py));
  o1 = make_double2(fTx + (Qx - fhgx), fTy + (Qy - fhgy));
  o2 = make_double2(fTx + (Px + fhgx), fTy + (Py + fhgy));
  o3 = make_double2(fTx - (Qx + fhgx), fTy - (Qy + fhgy));
}


// Finalisation of a reducing launch in the last block (tot = (u.Ku, |t|^2,
// dot, max|t|)): store, or one of the solver hooks.
BSP_DEV void stiff_hook(const StiffArgs& p, const double* tot_in) {
  DevState* st = p.st;
  // the per-thread maxima skip NaNs (fmax); a NaN anywhere made |t|^2 NaN
  const double tot[4] = {tot_in[0], tot_in[1], tot_in[2],
                         tot_in[1] != tot_in[1] ? tot_in[1] : tot_in[3]};
  switch (p.hook) {
    case HK_STORE:
      p.red_out[0] = tot[0]; p.red_out[1] = tot[1];
      p.red_out[2] = tot[2]; p.red_out[3] = tot[3];
      break;
    case HK_RESIDUAL:
      residual_hook(st, tot);
      if (p.flags & SF_SUM_SENS) st->gsum = tot[2];
      break;
    case HK_KRYLOV: {
      const double m = sqrt(tot[1]);
      if (m == 0.0) {
        st->kry_stop = 1;
      } else {
        st->norms[p.hook_i + 1] = m;
        st->kry_count = p.hook_i + 1;
      }
    } break;
    case HK_POWER:
    case HK_POWER_DOT: {
      const double n = sqrt(tot[1]);
      st->rho = (p.hook == HK_POWER) ? tot[0] : tot[2];
      st->pw[p.hook_i & 1] = n;
      if (n == 0.0) st->pow_stop = 1;
    } break;
  }
}

}  // namespace bsp
