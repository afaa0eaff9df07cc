// Geometric multigrid hierarchy and V-cycle (see mg.cuh for the algorithm).
//
// B200 mapping: every smoother / residual sweep is the same strip kernel as
// the matvec (k_stiff, stiffness.cu) with the SF_SUB_LOAD (rhs) + SF_D1DIV +
// SF_AXPY epilogue, so a Jacobi sweep costs one matvec of HBM traffic
// (u, b read, x written, a read).  Restriction fuses the next level's first
// (from-zero) Jacobi sweep; prolongation adds in place.  The coarsest level
// (<= 82 DOFs) is one CTA: assembly + in-shared-memory Gauss-Jordan inverse
// once per activation, a dense matvec per V-cycle.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "mg.cuh"
#include "q4.cuh"

using namespace bsp;

#ifndef BSP_PROLONG_U
#define BSP_PROLONG_U 2
#endif
#ifndef BSP_PROLONG_MINB
#define BSP_PROLONG_MINB 6
#endif

namespace bsp {

namespace {

BSP_DEV double act_at(const double* a, int nx, int ny, int x, int y) {
  return (x >= 0 && x < nx && y >= 0 && y < ny) ? a[(long long)y * nx + x] : 0.0;
}

// sum of the activations of the (<= 4) elements around node (x, y)
BSP_DEV double node_asum(const double* a, int nx, int ny, int x, int y) {
  return (act_at(a, nx, ny, x - 1, y - 1) + act_at(a, nx, ny, x, y - 1)) +
         (act_at(a, nx, ny, x - 1, y) + act_at(a, nx, ny, x, y));
}

BSP_DEV double2 jacobi_start(double2 b, uint32_t bits, double asum, const KeModes& km,
                             double omega) {
  // one reciprocal per node, in the smoother's form t * (1/kd * 1/asum)
  // (stiffness_tma.cu SF_D1DIV) instead of two divisions
  const double ia = asum == 0.0 ? 0.0 : 1.0 / asum;
  double2 x;
  x.x = (bits & 1u) ? 0.0 : (omega * b.x) * (km.ikdx * ia);
  x.y = (bits & 2u) ? 0.0 : (omega * b.y) * (km.ikdy * ia);
  return x;
}

}  // namespace

// a_c = mean of the 4 children (virtual children outside the fine grid = 0)
__global__ void k_mg_coarsen(const double* __restrict__ a, int nx, int ny, double* __restrict__ ac,
                             int nxc, int nyc, const int* gate) {
  if (gate && *gate) return;
  const long long E = (long long)nxc * nyc;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < E;
       e += (long long)gridDim.x * blockDim.x) {
    const int X = (int)(e % nxc), Y = (int)(e / nxc);
    const int x = 2 * X, y = 2 * Y;
    ac[e] = 0.25 * ((act_at(a, nx, ny, x, y) + act_at(a, nx, ny, x + 1, y)) +
                    (act_at(a, nx, ny, x, y + 1) + act_at(a, nx, ny, x + 1, y + 1)));
  }
}

// b_c = -M_c P~^T t (t: fine residual K x - b, zero on fine fixed DOFs);
// x_c = omega D_c^{-1} b_c (the coarse level's first Jacobi sweep from zero)
BSP_DEV void restrict_xy(int X, int Y, long long J, const double2* __restrict__ t, int nx, int ny,
                         double2* __restrict__ bc, double2* __restrict__ xc,
                         const double* __restrict__ ac, int nxc, int nyc,
                         const uint32_t* __restrict__ fixc, const KeModes& km, double omega) {
  double sx = 0.0, sy = 0.0;
  for (int dy = -1; dy <= 1; ++dy) {
    const int y = 2 * Y + dy;
    if (y < 0 || y > ny) continue;
    const double wy = dy == 0 ? 1.0 : 0.5;
    for (int dx = -1; dx <= 1; ++dx) {
      const int x = 2 * X + dx;
      if (x < 0 || x > nx) continue;
      const double w = wy * (dx == 0 ? 1.0 : 0.5);
      const double2 v = t[(long long)y * (nx + 1) + x];
      sx += w * v.x;
      sy += w * v.y;
    }
  }
  const uint32_t bits = fix_bits_gen(fixc, J);
  const double2 b = apply_mask(make_double2(-sx, -sy), bits);
  bc[J] = b;
  xc[J] = jacobi_start(b, bits, node_asum(ac, nxc, nyc, X, Y), km, omega);
}

BSP_DEV void restrict_node(long long J, const double2* __restrict__ t, int nx, int ny,
                           double2* __restrict__ bc, double2* __restrict__ xc,
                           const double* __restrict__ ac, int nxc, int nyc,
                           const uint32_t* __restrict__ fixc, const KeModes& km, double omega) {
  restrict_xy((int)(J % (nxc + 1)), (int)(J / (nxc + 1)), J, t, nx, ny, bc, xc, ac, nxc, nyc, fixc,
              km, omega);
}


__global__ void k_mg_restrict(const double2* __restrict__ t, int nx, int ny, double2* __restrict__ bc,
                              double2* __restrict__ xc, const double* __restrict__ ac, int nxc,
                              int nyc, const uint32_t* __restrict__ fixc, KeModes km, double omega,
                              const int* gate) {
  if (gate && *gate) return;
  // columns across the block, rows strided by the grid, 4 rows per trip so
  // that the loads of four nodes are in flight together (restrict pointers:
  // the compiler may hoist them above the stores)
  for (int X = blockIdx.x * blockDim.x + threadIdx.x; X <= nxc; X += gridDim.x * blockDim.x) {
#pragma unroll 4
    for (int Y = blockIdx.y; Y <= nyc; Y += gridDim.y)
      restrict_xy(X, Y, (long long)Y * (nxc + 1) + X, t, nx, ny, bc, xc, ac, nxc, nyc, fixc, km,
                  omega);
  }
}

// x += M_f P~ x_c  (in place; each fine node reads only coarse values)
// M_f P~ x_c at fine node (xx, yy), before the fine mask
BSP_DEV double2 prolong_sum(int xx, int yy, const double2* __restrict__ xc, int nxc) {
  const int X0 = xx >> 1, Y0 = yy >> 1, ox = xx & 1, oy = yy & 1;
  const double w = (ox ? 0.5 : 1.0) * (oy ? 0.5 : 1.0);
  // the coarse parents (Y0, X0), (Y0, X0+1), (Y0+1, X0), (Y0+1, X0+1) in this
  // summation order, the absent ones predicated off (no data-dependent loops:
  // odd and even columns alternate within a warp)
  const double2* r0 = xc + (long long)Y0 * (nxc + 1) + X0;
  const double2* r1 = r0 + (nxc + 1);
  const double2 v00 = r0[0];
  const double2 v01 = ox ? r0[1] : make_double2(0.0, 0.0);
  const double2 v10 = oy ? r1[0] : make_double2(0.0, 0.0);
  const double2 v11 = (ox && oy) ? r1[1] : make_double2(0.0, 0.0);
  double sx = w * v00.x, sy = w * v00.y;
  if (ox) {
    sx += w * v01.x;
    sy += w * v01.y;
  }
  if (oy) {
    sx += w * v10.x;
    sy += w * v10.y;
    if (ox) {
      sx += w * v11.x;
      sy += w * v11.y;
    }
  }
  return make_double2(sx, sy);
}

BSP_DEV void prolong_xy(int xx, int yy, long long j, double2* __restrict__ x,
                        const uint32_t* __restrict__ fixf, const double2* __restrict__ xc,
                        int nxc) {
  const double2 s = prolong_sum(xx, yy, xc, nxc);
  const uint32_t bits = fix_bits_gen(fixf, j);
  double2 o = x[j];
  if (!(bits & 1u)) o.x += s.x;
  if (!(bits & 2u)) o.y += s.y;
  x[j] = o;
}

BSP_DEV void prolong_node(long long j, double2* __restrict__ x, int nx,
                          const uint32_t* __restrict__ fixf, const double2* __restrict__ xc,
                          int nxc) {
  prolong_xy((int)(j % (nx + 1)), (int)(j / (nx + 1)), j, x, fixf, xc, nxc);
}

__global__ void __launch_bounds__(256, BSP_PROLONG_MINB) k_mg_prolong(double2* __restrict__ x, int nx, int ny, const uint32_t* __restrict__ fixf,
                             const double2* __restrict__ xc, int nxc, const int* gate) {
  if (gate && *gate) return;
  // x is updated in place, so the four rows of a trip are loaded first and
  // stored after (the loads of all four nodes in flight together)
  constexpr int U = BSP_PROLONG_U;
  const int dy = gridDim.y;
  for (int xx = blockIdx.x * blockDim.x + threadIdx.x; xx <= nx; xx += gridDim.x * blockDim.x) {
    for (int y0 = blockIdx.y; y0 <= ny; y0 += U * dy) {
      double2 o[U], add[U];
      uint32_t bits[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int yy = y0 + u * dy;
        if (yy > ny) break;
        const long long j = (long long)yy * (nx + 1) + xx;
        o[u] = x[j];
        bits[u] = fix_bits_gen(fixf, j);
        add[u] = prolong_sum(xx, yy, xc, nxc);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int yy = y0 + u * dy;
        if (yy > ny) break;
        if (!(bits[u] & 1u)) o[u].x += add[u].x;
        if (!(bits[u] & 2u)) o[u].y += add[u].y;
        x[(long long)yy * (nx + 1) + xx] = o[u];
      }
    }
  }
}

// level 0 first sweep from zero: x = omega D^{-1} b
__global__ void k_mg_jacobi0(const double2* __restrict__ b, double2* __restrict__ x,
                             const double* __restrict__ a, int nx, int ny,
                             const uint32_t* __restrict__ fix, KeModes km, double omega,
                             const int* gate) {
  if (gate && *gate) return;
  for (int xx = blockIdx.x * blockDim.x + threadIdx.x; xx <= nx; xx += gridDim.x * blockDim.x) {
#pragma unroll 4
    for (int yy = blockIdx.y; yy <= ny; yy += gridDim.y) {
      const long long j = (long long)yy * (nx + 1) + xx;
      x[j] = jacobi_start(b[j], fix_bits(fix, j), node_asum(a, nx, ny, xx, yy), km, omega);
    }
  }
}

// coarsest level: assemble K(a) densely (fixed DOFs -> identity rows/cols)
// and invert it by in-place Gauss-Jordan (SPD: no pivoting).  The matrix
// lives in registers: warp w owns columns [3w, 3w+3), lane l owns rows
// l, l+32, l+64 (9 entries per thread, up to 28 warps).  Pivot k reads the old
// row k, column k and 1/A_kk from a double-buffered shared copy that their
// owners refresh after each update, so a pivot costs one barrier.  The
// update is branch-free:
//   A' = A*s - c*(A_kj/A_kk)   with (s, c) = (1, A_ik), or (0, -1) on row k,
// and column k (warp-uniform) becomes -c/A_kk.  Bit-identical to the textbook
// order A_ij - A_ik (A_kj / A_kk), A_kj / A_kk, -A_ik / A_kk, 1 / A_kk.
constexpr int kFactorMax = 2 * kCoarseNodes + 2;           // DOFs
constexpr int kFactorCols = 3;                             // columns per warp
constexpr int kFactorWarps = (kFactorMax + kFactorCols - 1) / kFactorCols;
constexpr int kFactorThreads = 32 * kFactorWarps;
constexpr int kFactorRows = (kFactorMax + 31) / 32;        // rows per lane
constexpr int kFactorPad = 32 * kFactorRows;               // >= kFactorWarps * kFactorCols

// a, fix, ke: shared-memory copies (the assembly is latency-bound otherwise)
BSP_DEV double coarse_entry(const double* a, int nx, int ny, const uint32_t* fix,
                            const double* ke, int I, int J) {
  const int NX1 = nx + 1;
  const int nI = I >> 1, cI = I & 1, nJ = J >> 1, cJ = J & 1;
  const bool fI = (fix_bits_gen(fix, nI) >> cI) & 1u, fJ = (fix_bits_gen(fix, nJ) >> cJ) & 1u;
  if (fI || fJ) return (I == J) ? 1.0 : 0.0;
  double v = 0.0;
  const int xI = nI % NX1, yI = nI / NX1, xJ = nJ % NX1, yJ = nJ / NX1;
  // elements around node I in fixed order; local node index of (dx, dy)
  // relative to the element origin: (0,0)->0 (1,0)->1 (1,1)->2 (0,1)->3
  for (int k = 0; k < 4; ++k) {
    const int ex = xI - 1 + (k & 1), ey = yI - 1 + (k >> 1);
    if (ex < 0 || ex >= nx || ey < 0 || ey >= ny) continue;
    const int dxI = xI - ex, dyI = yI - ey, dxJ = xJ - ex, dyJ = yJ - ey;
    if (dxJ < 0 || dxJ > 1 || dyJ < 0 || dyJ > 1) continue;
    const int li = dyI ? (dxI ? 2 : 3) : dxI;
    const int lj = dyJ ? (dxJ ? 2 : 3) : dxJ;
    v += a[(long long)ey * nx + ex] * ke[(2 * li + cI) * 8 + 2 * lj + cJ];
  }
  return v;
}

__global__ void __launch_bounds__(kFactorThreads) k_mg_coarse_factor(
    const double* __restrict__ a, int nx, int ny, const uint32_t* __restrict__ fix,
    const double* __restrict__ ke, double* __restrict__ Ainv, int nc, const int* gate) {
  if (gate && *gate) return;
  constexpr int CW = kFactorCols, RL = kFactorRows;
  __shared__ double row[2][kFactorPad], col[2][kFactorPad], ipiv[2];
  __shared__ double ske[64], sa[kFactorMax];  // coarsest E <= nodes <= kFactorMax / 2
  __shared__ uint32_t sfix[(kFactorMax / 2 + 15) / 16 + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, j0 = CW * w;
  for (int t = threadIdx.x; t < 2 * kFactorPad; t += blockDim.x) {
    (&row[0][0])[t] = 0.0;
    (&col[0][0])[t] = 0.0;
  }
  for (int t = threadIdx.x; t < 64; t += blockDim.x) ske[t] = ke[t];
  for (int t = threadIdx.x; t < nx * ny; t += blockDim.x) sa[t] = a[t];
  for (int t = threadIdx.x; t < ((nx + 1) * (ny + 1) + 15) / 16; t += blockDim.x) sfix[t] = fix[t];
  __syncthreads();
  double A[RL][CW];
#pragma unroll
  for (int m = 0; m < RL; ++m) {
    const int i = lane + 32 * m;
#pragma unroll
    for (int q = 0; q < CW; ++q) {
      const int j = j0 + q;
      const double v = (i < nc && j < nc) ? coarse_entry(sa, nx, ny, sfix, ske, i, j) : 0.0;
      A[m][q] = v;
      if (i < nc && j == 0) col[0][i] = v;
      if (i == 0 && j < nc) row[0][j] = v;
      if (i == 0 && j == 0) ipiv[0] = v != 0.0 ? 1.0 / v : 0.0;
    }
  }
  __syncthreads();
  for (int k = 0; k < nc; ++k) {
    const int b = k & 1;
    const double ip = ipiv[b];
    double rs[CW];
#pragma unroll
    for (int q = 0; q < CW; ++q) rs[q] = row[b][j0 + q] * ip;
    double c[RL];
#pragma unroll
    for (int m = 0; m < RL; ++m) {
      const bool pr = lane + 32 * m == k;
      const double s = pr ? 0.0 : 1.0;
      c[m] = pr ? -1.0 : col[b][lane + 32 * m];
#pragma unroll
      for (int q = 0; q < CW; ++q) A[m][q] = __fma_rn(-c[m], rs[q], A[m][q] * s);
    }
    const int wk = k / CW;
    if (w == wk) {  // warp-uniform: this warp holds pivot column k
      const int qk = k - CW * wk;
#pragma unroll
      for (int m = 0; m < RL; ++m)
#pragma unroll
        for (int q = 0; q < CW; ++q)
          if (q == qk) A[m][q] = -c[m] * ip;
    }
    // publish column / row / pivot k+1 for the next step
    const int k1 = k + 1;
    const int wk1 = k1 / CW;
    if (w == wk1) {
      const int q1 = k1 - CW * wk1;
#pragma unroll
      for (int m = 0; m < RL; ++m) {
        double v = 0.0;
#pragma unroll
        for (int q = 0; q < CW; ++q)
          if (q == q1) v = A[m][q];
        col[b ^ 1][lane + 32 * m] = v;
        if (lane + 32 * m == k1) ipiv[b ^ 1] = v != 0.0 ? 1.0 / v : 0.0;
      }
    }
    if (lane == (k1 & 31)) {
      const int m1 = k1 >> 5;
#pragma unroll
      for (int m = 0; m < RL; ++m)
        if (m == m1) {
#pragma unroll
          for (int q = 0; q < CW; ++q) row[b ^ 1][j0 + q] = A[m][q];
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int m = 0; m < RL; ++m) {
    const int i = lane + 32 * m;
#pragma unroll
    for (int q = 0; q < CW; ++q)
      if (i < nc && j0 + q < nc) Ainv[i * nc + j0 + q] = A[m][q];
  }
}

// x = Ainv b on the coarsest level
__global__ void __launch_bounds__(128) k_mg_coarse_solve(const double* __restrict__ Ainv, int nc,
                                                         const double* __restrict__ b,
                                                         double* __restrict__ x, const int* gate) {
  if (gate && *gate) return;
  __shared__ double sb[2 * kCoarseNodes + 2];
  for (int i = threadIdx.x; i < nc; i += blockDim.x) sb[i] = b[i];
  __syncthreads();
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < nc; ++j) s += Ainv[i * nc + j] * sb[j];
    x[i] = s;
  }
}

// ---------------------------------------------------------------------------
// Coarse tail of the V-cycle in ONE CTA.  Levels with <= tail_nodes nodes run
// as a list of node-parallel ops separated by __syncthreads instead of one
// kernel launch each: below ~2k nodes a launch costs more than the sweep.
// The ops are those of the multi-kernel V-cycle (mg_vcycle_enqueue builds
// both from the same schedule); the smoother / residual node sum follows the
// strip kernel's order ((o2' + o1) of the left element column + (o3' + o0) of
// the right one, virtual elements contribute +0), so both paths agree.
enum TailOpType : int8_t { TO_JACOBI0, TO_SMOOTH, TO_RESID, TO_RESTRICT, TO_COARSE, TO_PROLONG,
                           TO_PROSMOOTH };
enum TailBuf : int8_t { TB_B, TB_X, TB_Y, TB_T, TB_IN, TB_OUT };
struct TailOp {
  int8_t type, level, src, dst, rhs;
  int8_t aux;  // TO_PROSMOOTH: the coarse source (level + 1)
};
struct TailLevel {
  int nx, ny;
  const double* a;      // global activation / fixed mask / vectors
  const uint32_t* fix;
  double *B, *X, *Y, *T;
  int oB, oX, oY, oT, oA, oF;  // shared-memory offsets (bytes) of the same
};
constexpr int kTailLevels = 12, kTailOps = 96;
constexpr int kTailSmem = 200 * 1024;
struct TailArgs {
  TailLevel lv[kTailLevels];
  TailOp op[kTailOps];
  int nops;
  int lt, L;         // levels lt..L live in shared memory
  int res_id;        // level-lt buffer copied back to global at the end (-1: none)
  const double* in;  // level-0 right-hand side (TB_IN, global)
  double* out;       // level-0 result (TB_OUT, global)
  const double* Ainv;
  int nc;
  double omega;
};

BSP_DEV double* tail_buf(const TailArgs& p, unsigned char* sm, int l, int id) {
  const TailLevel& L = p.lv[l];
  switch (id) {
    case TB_B: return (double*)(sm + L.oB);
    case TB_X: return (double*)(sm + L.oX);
    case TB_Y: return (double*)(sm + L.oY);
    case TB_T: return (double*)(sm + L.oT);
    case TB_IN: return const_cast<double*>(p.in);
    default: return p.out;
  }
}

// K(a) x at node (X, Y) in the strip kernel's summation order (unmasked)
// contribution k of the 4 elements around node (X, Y) to (K(a) x)_node:
// k = 0: o2 of (X-1,Y-1), 1: o1 of (X-1,Y), 2: o3 of (X,Y-1), 3: o0 of (X,Y);
// virtual elements contribute +0 (as the strip kernel's zero-filled ones)
BSP_DEV double2 elem_contrib(int nx, int ny, const double* a, const double2* x, const KeModes& km,
                             int X, int Y, int k, double& ae) {
  const int ex = X - 1 + (k >> 1), ey = Y - 1 + (k & 1);
  ae = 0.0;
  if (k > 3 || ex < 0 || ex >= nx || ey < 0 || ey >= ny) return make_double2(0.0, 0.0);
  ae = a[ey * nx + ex];
  const int NX1 = nx + 1;
  const int j = ey * NX1 + ex;
  double2 o0, o1, o2, o3;
  double en;
  element<false, false>(km, ae, x[j], x[j + 1], x[j + NX1 + 1], x[j + NX1], o0, o1, o2, o3, en);
  return k == 0 ? o2 : (k == 1 ? o1 : (k == 2 ? o3 : o0));
}

__global__ void __launch_bounds__(1024) k_mg_tail(TailArgs p, KeModes km, const int* gate) {
  if (gate && *gate) return;
  extern __shared__ __align__(16) unsigned char sm[];
  __shared__ double sb[2 * kCoarseNodes + 2];
  // stage the activations and fixed masks of the tail levels, and the
  // first level's right-hand side and first sweep (written by the restriction
  // kernel of level lt-1)
  for (int l = p.lt; l <= p.L; ++l) {
    const TailLevel& L = p.lv[l];
    const int E = L.nx * L.ny, N = (L.nx + 1) * (L.ny + 1), W = (N + 15) >> 4;
    double* a = (double*)(sm + L.oA);
    uint32_t* f = (uint32_t*)(sm + L.oF);
    for (int e = threadIdx.x; e < E; e += blockDim.x) a[e] = L.a[e];
    for (int w = threadIdx.x; w < W; w += blockDim.x) f[w] = L.fix[w];
    if (l == p.lt && l > 0) {
      double2* B = (double2*)(sm + L.oB);
      double2* X = (double2*)(sm + L.oX);
      for (int j = threadIdx.x; j < N; j += blockDim.x) {
        B[j] = ((const double2*)L.B)[j];
        X[j] = ((const double2*)L.X)[j];
      }
    }
  }
  __syncthreads();
  for (int o = 0; o < p.nops; ++o) {
    const TailOp op = p.op[o];
    const int l = op.level;
    const TailLevel& L = p.lv[l];
    const double* la = (const double*)(sm + L.oA);
    const uint32_t* lf = (const uint32_t*)(sm + L.oF);
    const int N = (L.nx + 1) * (L.ny + 1);
    switch (op.type) {
      case TO_JACOBI0: {
        const double2* b = (const double2*)tail_buf(p, sm, l, op.src);
        double2* x = (double2*)tail_buf(p, sm, l, op.dst);
        for (int j = threadIdx.x; j < N; j += blockDim.x) {
          const int xx = j % (L.nx + 1), yy = j / (L.nx + 1);
          x[j] = jacobi_start(b[j], fix_bits_gen(lf, j), node_asum(la, L.nx, L.ny, xx, yy), km,
                              p.omega);
        }
      } break;
      case TO_SMOOTH:
      case TO_RESID: {
        // 4 lanes per node (one per adjacent element), combined by shuffles
        // in the strip kernel's order (c0 + c1) + (c2 + c3)
        const double2* x = (const double2*)tail_buf(p, sm, l, op.src);
        const double2* b = (const double2*)tail_buf(p, sm, l, op.rhs);
        double2* out = (double2*)tail_buf(p, sm, l, op.dst);
        const int k = threadIdx.x & 3;
        for (int base = 0; base < 4 * N; base += blockDim.x) {
          const int j = (base + threadIdx.x) >> 2;
          const bool valid = j < N;
          const int X = valid ? j % (L.nx + 1) : 0, Y = valid ? j / (L.nx + 1) : 0;
          double ae;
          double2 c = elem_contrib(L.nx, L.ny, la, x, km, X, Y, valid ? k : 4, ae);
          c.x += __shfl_xor_sync(0xffffffffu, c.x, 1);
          c.y += __shfl_xor_sync(0xffffffffu, c.y, 1);
          ae += __shfl_xor_sync(0xffffffffu, ae, 1);
          c.x += __shfl_xor_sync(0xffffffffu, c.x, 2);
          c.y += __shfl_xor_sync(0xffffffffu, c.y, 2);
          const double as = ae + __shfl_xor_sync(0xffffffffu, ae, 2);
          if (!valid || k != 0) continue;
          const uint32_t bits = fix_bits_gen(lf, j);
          const double2 ku = apply_mask(c, bits);
          const double2 f = b[j];
          double2 t = make_double2(ku.x - f.x, ku.y - f.y);
          if (op.type == TO_SMOOTH) {
            const double ias = 1.0 / as;
            t.x = (bits & 1u) ? t.x : t.x * (km.ikdx * ias);
            t.y = (bits & 2u) ? t.y : t.y * (km.ikdy * ias);
            const double2 base_x = x[j];
            t.x = base_x.x - p.omega * t.x;
            t.y = base_x.y - p.omega * t.y;
          }
          out[j] = t;
        }
      } break;
      case TO_RESTRICT: {
        const TailLevel& C = p.lv[l + 1];
        const int Nc = (C.nx + 1) * (C.ny + 1);
        for (int J = threadIdx.x; J < Nc; J += blockDim.x)
          restrict_node(J, (const double2*)(sm + L.oT), L.nx, L.ny, (double2*)(sm + C.oB),
                        (double2*)(sm + C.oX), (const double*)(sm + C.oA), C.nx, C.ny,
                        (const uint32_t*)(sm + C.oF), km, p.omega);
      } break;
      case TO_COARSE: {
        const double* Bc = (const double*)(sm + L.oB);
        double* Yc = (double*)(sm + L.oY);
        for (int i = threadIdx.x; i < p.nc; i += blockDim.x) sb[i] = Bc[i];
        __syncthreads();
        for (int i = threadIdx.x; i < p.nc; i += blockDim.x) {
          double s = 0.0;
          for (int j = 0; j < p.nc; ++j) s += p.Ainv[i * p.nc + j] * sb[j];
          Yc[i] = s;
        }
      } break;
      case TO_PROLONG: {
        const TailLevel& C = p.lv[l + 1];
        double2* x = (double2*)tail_buf(p, sm, l, op.dst);
        const double2* xc = (const double2*)tail_buf(p, sm, l + 1, op.src);
        for (int j = threadIdx.x; j < N; j += blockDim.x) prolong_node(j, x, L.nx, lf, xc, C.nx);
      } break;
    }
    __syncthreads();
  }
  if (p.res_id >= 0) {  // the level-lt result, read by the next prolongation kernel
    const TailLevel& L = p.lv[p.lt];
    const int N = (L.nx + 1) * (L.ny + 1);
    const double2* src = (const double2*)tail_buf(p, sm, p.lt, p.res_id);
    double2* dst = (double2*)(p.res_id == TB_X ? L.X : (p.res_id == TB_Y ? L.Y : L.B));
    for (int j = threadIdx.x; j < N; j += blockDim.x) dst[j] = src[j];
  }
}

namespace {
unsigned blocks_for(long long n, int nsm) {
  long long b = (n + 255) / 256;
  return (unsigned)std::max<long long>(1, std::min<long long>(b, 8ll * nsm));
}


cudaError_t smooth(bsp_grid* g, const double* a, const double* b, const double* x, double* out,
                   double omega, const int* gate, cudaStream_t s, const bsp_grid* coarse = nullptr,
                   const double* xc = nullptr) {
  StiffArgs p = stiff_args(g);
  p.a = a;
  p.u = (const double2*)x;
  p.rhs = (const double2*)b;
  p.base = (const double2*)x;
  p.beta = omega;
  p.out = (double2*)out;
  p.flags = SF_IN_MASKED | SF_SUB_LOAD | SF_D1DIV | SF_AXPY;
  if (coarse) {  // x + M P~ xc, formed on the fly by the TMA kernel
    p.flags |= SF_PROLONG;
    p.pc = (const double2*)xc;
    p.nxc = coarse->nx;
    p.nyc = coarse->ny;
  }
  p.gate0 = gate;
  return launch_stiff(g, p, s);
}

// the fused prolongation + first post-smoothing sweep runs on the TMA kernel
bool prolong_fusable(const bsp_grid* g) {
  static const bool off = [] {
    const char* e = getenv("BSP_MG_NOFUSE");
    return e && e[0] == '1';
  }();
  return g->use_tma && !off;
}

cudaError_t residual(bsp_grid* g, const double* a, const double* b, const double* x, double* out,
                     const int* gate, cudaStream_t s) {
  StiffArgs p = stiff_args(g);
  p.a = a;
  p.u = (const double2*)x;
  p.rhs = (const double2*)b;
  p.out = (double2*)out;
  p.flags = SF_IN_MASKED | SF_SUB_LOAD;
  p.gate0 = gate;
  return launch_stiff(g, p, s);
}

}  // namespace

static bool fork_enabled() {
  const char* e = std::getenv("BSP_MG_FORK");
  return !(e && e[0] == '0');
}

int mg_setup_enqueue(bsp_mg* mg, const double* a0, const int* gate, cudaStream_t s) {
  mg->a[0] = const_cast<double*>(a0);
  cudaStream_t t = s;
  if (mg->side && fork_enabled()) {
    BSP_CU(cudaEventRecord(mg->ev_fork, s));
    BSP_CU(cudaStreamWaitEvent(mg->side, mg->ev_fork, 0));
    t = mg->side;
  }
  for (int l = 0; l < mg->L; ++l) {
    bsp_grid* f = mg->lv[l];
    bsp_grid* c = mg->lv[l + 1];
    k_mg_coarsen<<<blocks_for(c->E, f->nsm), 256, 0, t>>>(mg->a[l], f->nx, f->ny, mg->a[l + 1],
                                                          c->nx, c->ny, gate);
    BSP_CU(cudaGetLastError());
  }
  if (t != s) BSP_CU(cudaEventRecord(mg->ev_coarse, t));
  bsp_grid* cL = mg->lv[mg->L];
  k_mg_coarse_factor<<<1, kFactorThreads, 0, t>>>(mg->a[mg->L], cL->nx, cL->ny, cL->fixbits,
                                                  mg->ke, mg->Ainv, mg->nc, gate);
  BSP_CU(cudaGetLastError());
  if (t != s) {
    BSP_CU(cudaEventRecord(mg->ev_factor, t));
    mg->wait_coarse = mg->wait_factor = true;
  }
  return BSP_OK;
}

// join the side-stream setup into s before the first use of its results
static cudaError_t mg_join(bsp_mg* mg, bool coarse, bool factor, cudaStream_t s) {
  if (coarse && mg->wait_coarse) {
    mg->wait_coarse = false;
    cudaError_t e = cudaStreamWaitEvent(s, mg->ev_coarse, 0);
    if (e != cudaSuccess) return e;
  }
  if (factor && mg->wait_factor) {
    mg->wait_factor = false;
    mg->wait_coarse = false;  // recorded earlier on the same stream
    return cudaStreamWaitEvent(s, mg->ev_factor, 0);
  }
  return cudaSuccess;
}

// The one-CTA tail covers levels lt..L: every level with <= BSP_MG_TAIL
// nodes (default 600, 0 disables), fewer if their vectors, activations and
// masks exceed kTailSmem of shared memory.  Returns L + 1 for no tail and
// fills the shared-memory layout.
static int plan_tail(const bsp_mg* mg, TailArgs& ta, size_t& smem) {
  const char* e = std::getenv("BSP_MG_TAIL");
  const long long lim = e ? std::atoll(e) : 600ll;
  const int L = mg->L;
  if (lim <= 0 || L + 1 > kTailLevels || mg->lv[0]->generic) return L + 1;
  int lt = L + 1;
  for (int l = L; l >= 0; --l) {
    if (mg->lv[l]->N > lim) break;
    lt = l;
  }
  for (; lt < L; ++lt) {
    size_t off = 0;
    for (int l = lt; l <= L; ++l) {
      const bsp_grid* g = mg->lv[l];
      TailLevel& t = ta.lv[l];
      t = TailLevel{g->nx, g->ny, mg->a[l], g->fixbits, mg->B[l], mg->X[l], mg->Y[l], mg->T[l]};
      const size_t vb = (size_t)g->N * 16;
      t.oB = (int)off; off += vb;
      t.oX = (int)off; off += vb;
      t.oY = (int)off; off += vb;
      t.oT = (int)off; off += vb;
      t.oA = (int)off; off += ((size_t)g->E * 8 + 15) / 16 * 16;
      t.oF = (int)off; off += ((size_t)(g->N + 15) / 16 * 4 + 15) / 16 * 16;
    }
    if (off <= (size_t)kTailSmem) {
      smem = off;
      return lt;
    }
  }
  return L + 1;  // the coarsest level alone: keep the plain solve
}

int mg_vcycle_enqueue(bsp_mg* mg, const double* b0, double* out0, double omega, int nu,
                      const int* gate, cudaStream_t s) {
  const int L = mg->L;
  if (L == 0) {
    BSP_CU(mg_join(mg, true, true, s));
    k_mg_coarse_solve<<<1, 128, 0, s>>>(mg->Ainv, mg->nc, b0, out0, gate);
    BSP_CU(cudaGetLastError());
    return BSP_OK;
  }
  // One schedule for both execution modes: ops on levels >= lt are collected
  // into the one-CTA tail, the others launch as grid-wide kernels.
  TailArgs ta{};
  size_t tail_smem = 0;
  const int lt = plan_tail(mg, ta, tail_smem);
  ta.lt = lt;
  ta.L = L;
  ta.res_id = -1;
  ta.in = b0;
  ta.out = out0;
  ta.Ainv = mg->Ainv;
  ta.nc = mg->nc;
  ta.omega = omega;
  bool tail_done = false;
  auto buf = [&](int l, int id) -> double* {
    switch (id) {
      case TB_B: return mg->B[l];
      case TB_X: return mg->X[l];
      case TB_Y: return mg->Y[l];
      case TB_T: return mg->T[l];
      case TB_IN: return const_cast<double*>(b0);
      default: return out0;
    }
  };
  auto flush_tail = [&]() -> cudaError_t {
    if (tail_done || ta.nops == 0) return cudaSuccess;
    tail_done = true;
    cudaError_t je = mg_join(mg, true, true, s);
    if (je != cudaSuccess) return je;
    cudaError_t e = smem_optin((const void*)k_mg_tail, kTailSmem);
    if (e != cudaSuccess) return e;
    k_mg_tail<<<1, 1024, tail_smem, s>>>(ta, mg->lv[lt]->km, gate);
    return cudaGetLastError();
  };
  auto emit = [&](TailOp op) -> cudaError_t {
    if (op.level >= lt) {
      if (ta.nops >= kTailOps) return cudaErrorInvalidValue;
      ta.op[ta.nops++] = op;
      return cudaSuccess;
    }
    cudaError_t e = flush_tail();
    if (e != cudaSuccess) return e;
    const int l = op.level;
    bsp_grid* g = mg->lv[l];
    switch (op.type) {
      case TO_JACOBI0:
        k_mg_jacobi0<<<node_grid(g->nx, g->ny, wave_blocks((const void*)k_mg_jacobi0, 256)), 256, 0, s>>>(
            (const double2*)buf(l, op.src), (double2*)buf(l, op.dst), mg->a[l], g->nx, g->ny,
            g->fixbits, g->km, omega, gate);
        return cudaGetLastError();
      case TO_SMOOTH:
        return smooth(g, mg->a[l], buf(l, op.rhs), buf(l, op.src), buf(l, op.dst), omega, gate, s);
      case TO_PROSMOOTH:
        return smooth(g, mg->a[l], buf(l, op.rhs), buf(l, op.src), buf(l, op.dst), omega, gate, s,
                      mg->lv[l + 1], buf(l + 1, op.aux));
      case TO_RESID:
        return residual(g, mg->a[l], buf(l, op.rhs), buf(l, op.src), buf(l, op.dst), gate, s);
      case TO_RESTRICT: {
        bsp_grid* c = mg->lv[l + 1];
        e = mg_join(mg, true, false, s);  // reads the coarse activation
        if (e != cudaSuccess) return e;
        k_mg_restrict<<<node_grid(c->nx, c->ny, wave_blocks((const void*)k_mg_restrict, 256)), 256, 0, s>>>(
            (const double2*)mg->T[l], g->nx, g->ny, (double2*)mg->B[l + 1],
            (double2*)mg->X[l + 1], mg->a[l + 1], c->nx, c->ny, c->fixbits, c->km, omega, gate);
        return cudaGetLastError();
      }
      case TO_COARSE:
        e = mg_join(mg, true, true, s);
        if (e != cudaSuccess) return e;
        k_mg_coarse_solve<<<1, 128, 0, s>>>(mg->Ainv, mg->nc, mg->B[l], mg->Y[l], gate);
        return cudaGetLastError();
      default: {
        bsp_grid* c = mg->lv[l + 1];
        k_mg_prolong<<<node_grid(g->nx, g->ny, wave_blocks((const void*)k_mg_prolong, 256)), 256, 0, s>>>(
            (double2*)buf(l, op.dst), g->nx, g->ny, g->fixbits, (const double2*)buf(l + 1, op.src),
            c->nx, gate);
        return cudaGetLastError();
      }
    }
  };
  auto other = [](int8_t id) -> int8_t { return id == TB_X ? TB_Y : TB_X; };
  std::vector<int8_t> cur(L + 1, TB_X);
  for (int l = 0; l < L; ++l) {
    const int8_t b = l == 0 ? TB_IN : TB_B;
    int8_t x = TB_X;
    if (l == 0) BSP_CU(emit(TailOp{TO_JACOBI0, 0, TB_IN, TB_X, TB_IN}));
    for (int it = 1; it < nu; ++it) {
      const int8_t nx_ = other(x);
      BSP_CU(emit(TailOp{TO_SMOOTH, (int8_t)l, x, nx_, b}));
      x = nx_;
    }
    cur[l] = x;
    BSP_CU(emit(TailOp{TO_RESID, (int8_t)l, x, TB_T, b}));
    BSP_CU(emit(TailOp{TO_RESTRICT, (int8_t)l, TB_T, TB_B, TB_B}));
  }
  // coarsest: direct solve B[L] -> Y[L]
  BSP_CU(emit(TailOp{TO_COARSE, (int8_t)L, TB_B, TB_Y, TB_B}));
  int8_t res = TB_Y;
  for (int l = L - 1; l >= 0; --l) {
    const int8_t b = l == 0 ? TB_IN : TB_B;
    int8_t x = cur[l];
    if (l == lt - 1) ta.res_id = res;  // the tail's level-lt result goes back to global
    // per-level kernels on the TMA path: the prolongation is formed while the
    // first post-sweep stages its input (one fine-level pass fewer); the tail
    // and the cp.async path keep the two steps
    const bool fuse = l < lt && prolong_fusable(mg->lv[l]);
    if (!fuse) BSP_CU(emit(TailOp{TO_PROLONG, (int8_t)l, res, x, b, 0}));
    for (int it = 0; it < nu; ++it) {
      const int8_t dst = (l == 0 && it == nu - 1) ? TB_OUT : other(x);
      if (fuse && it == 0)
        BSP_CU(emit(TailOp{TO_PROSMOOTH, (int8_t)l, x, dst, b, res}));
      else
        BSP_CU(emit(TailOp{TO_SMOOTH, (int8_t)l, x, dst, b, 0}));
      x = dst;
    }
    res = x;
  }
  BSP_CU(flush_tail());
  return BSP_OK;
}

}  // namespace bsp

// ------------------------------------------------------------------ C ABI ---
extern "C" int bsp_mg_destroy(bsp_mg* mg) {
  if (!mg) return BSP_OK;
  for (size_t l = 0; l < mg->lv.size(); ++l) {
    if (l >= 1) {
      bsp_grid_destroy(mg->lv[l]);
      cudaFree(mg->a[l]);
    }
    cudaFree(mg->B[l]);
    cudaFree(mg->X[l]);
    cudaFree(mg->Y[l]);
    cudaFree(mg->T[l]);
  }
  cudaFree(mg->Ainv);
  cudaFree(mg->ke);
  if (mg->side) cudaStreamDestroy(mg->side);
  for (cudaEvent_t e : {mg->ev_fork, mg->ev_coarse, mg->ev_factor})
    if (e) cudaEventDestroy(e);
  delete mg;
  return BSP_OK;
}

extern "C" int bsp_mg_create(bsp_grid* g, int max_levels, bsp_mg** out) {
  if (!g || !out) return set_error(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(g->device);
  if (!g->uniform_diag) return set_error(BSP_EUNSUPPORTED, "multigrid needs a uniform ke diagonal");
  if (max_levels < 1) max_levels = kMaxLevels;
  max_levels = std::min(max_levels, kMaxLevels);
  std::vector<double> ke(g->ke, g->ke + 64);
  const long long words0 = (g->N + 15) / 16;
  std::vector<uint32_t> bits0(words0);
  if (cudaMemcpy(bits0.data(), g->fixbits, words0 * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
    return set_error(BSP_ECUDA, "mg create: reading the fixed mask failed");
  bsp_mg* mg = new bsp_mg();
  mg->g0 = g;
  mg->lv.push_back(g);
  std::vector<uint8_t> fine(g->n);
  for (long long j = 0; j < g->N; ++j) {
    const uint32_t b = (bits0[j >> 4] >> (2 * (j & 15))) & 3u;
    fine[2 * j] = b & 1u;
    fine[2 * j + 1] = (b >> 1) & 1u;
  }
  int nx = g->nx, ny = g->ny;
  int rc = BSP_OK;
  while ((int)mg->lv.size() < max_levels &&
         (long long)(nx + 1) * (ny + 1) > kCoarseNodes && (nx > 1 || ny > 1)) {
    const int cx = (nx + 1) / 2, cy = (ny + 1) / 2;
    const long long Nc = (long long)(cx + 1) * (cy + 1);
    std::vector<uint8_t> cf(2 * Nc, 0);
    for (int Y = 0; Y <= cy; ++Y)
      for (int X = 0; X <= cx; ++X)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dx = -1; dx <= 1; ++dx) {
            const int x = 2 * X + dx, y = 2 * Y + dy;
            if (x < 0 || x > nx || y < 0 || y > ny) continue;
            const long long jf = (long long)y * (nx + 1) + x, jc = (long long)Y * (cx + 1) + X;
            cf[2 * jc] |= fine[2 * jf];
            cf[2 * jc + 1] |= fine[2 * jf + 1];
          }
    std::vector<double> zero(2 * Nc, 0.0);
    bsp_grid* c = nullptr;
    rc = bsp_grid_create(cx, cy, ke.data(), cf.data(), zero.data(), &c);
    if (rc) break;
    mg->lv.push_back(c);
    fine.swap(cf);
    nx = cx;
    ny = cy;
  }
  mg->L = (int)mg->lv.size() - 1;
  const size_t nl = mg->lv.size();
  mg->a.assign(nl, nullptr);
  mg->B.assign(nl, nullptr);
  mg->X.assign(nl, nullptr);
  mg->Y.assign(nl, nullptr);
  mg->T.assign(nl, nullptr);
  bool ok = rc == BSP_OK;
  for (size_t l = 0; l < nl && ok; ++l) {
    const size_t nb = mg->lv[l]->n * sizeof(double);
    if (l >= 1) ok = cudaMalloc(&mg->a[l], mg->lv[l]->E * sizeof(double)) == cudaSuccess;
    ok = ok && cudaMalloc(&mg->B[l], nb) == cudaSuccess && cudaMalloc(&mg->X[l], nb) == cudaSuccess &&
         cudaMalloc(&mg->Y[l], nb) == cudaSuccess && cudaMalloc(&mg->T[l], nb) == cudaSuccess;
  }
  bsp_grid* cL = mg->lv[mg->L];
  mg->nc = (int)cL->n;
  ok = ok && mg->nc <= 2 * kCoarseNodes + 2 &&
       cudaMalloc(&mg->Ainv, (size_t)mg->nc * mg->nc * sizeof(double)) == cudaSuccess &&
       cudaMalloc(&mg->ke, 64 * sizeof(double)) == cudaSuccess &&
       cudaMemcpy(mg->ke, ke.data(), 64 * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    if (mg->nc > 2 * kCoarseNodes + 2 && rc == BSP_OK)
      rc = set_error(BSP_EUNSUPPORTED, "coarsest level has %d DOFs (> %d): raise max_levels",
                     mg->nc, 2 * kCoarseNodes + 2);
    bsp_mg_destroy(mg);
    return rc ? rc : set_error(BSP_ENOMEM, "multigrid allocation failed");
  }
  for (size_t l = 0; l < nl; ++l) {
    cudaMemset(mg->X[l], 0, mg->lv[l]->n * sizeof(double));
    cudaMemset(mg->Y[l], 0, mg->lv[l]->n * sizeof(double));
  }
  if (cudaStreamCreateWithFlags(&mg->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&mg->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&mg->ev_coarse, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&mg->ev_factor, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    bsp_mg_destroy(mg);
    return set_error(BSP_ECUDA, "multigrid stream/event creation failed");
  }
  *out = mg;
  return BSP_OK;
}

extern "C" int bsp_mg_info(const bsp_mg* mg, int* levels, int* coarse_dofs) {
  if (!mg) return set_error(BSP_EINVAL, "null multigrid");
  if (levels) *levels = mg->L + 1;
  if (coarse_dofs) *coarse_dofs = mg->nc;
  return BSP_OK;
}

extern "C" int bsp_mg_level(const bsp_mg* mg, int level, int* nx, int* ny, uint8_t* h_fixed) {
  if (!mg) return set_error(BSP_EINVAL, "null multigrid");
  if (level < 0 || level > mg->L) return set_error(BSP_EINVAL, "level %d outside [0, %d]", level, mg->L);
  const bsp_grid* g = mg->lv[level];
  if (nx) *nx = g->nx;
  if (ny) *ny = g->ny;
  if (h_fixed) {
    const long long words = (g->N + 15) / 16;
    std::vector<uint32_t> bits(words);
    BSP_CU(cudaMemcpy(bits.data(), g->fixbits, words * 4, cudaMemcpyDeviceToHost));
    for (long long j = 0; j < g->N; ++j) {
      const uint32_t b = (bits[j >> 4] >> (2 * (j & 15))) & 3u;
      h_fixed[2 * j] = b & 1u;
      h_fixed[2 * j + 1] = (b >> 1) & 1u;
    }
  }
  return BSP_OK;
}

extern "C" int bsp_mg_setup(bsp_mg* mg, const double* d_a, void* stream) {
  if (!mg || !d_a) return set_error(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(mg->g0->device);
  return mg_setup_enqueue(mg, d_a, nullptr, (cudaStream_t)stream);
}

namespace bsp {
__global__ void k_mask_copy(const double* x0, const uint32_t* fixbits, double* x, long long n);
}

extern "C" int bsp_mg_vcycle(bsp_mg* mg, const double* d_b, double* d_x, double omega, int nu,
                             void* stream) {
  if (!mg || !d_b || !d_x) return set_error(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(mg->g0->device);
  if (!mg->a[0]) return set_error(BSP_EINVAL, "bsp_mg_setup must run before bsp_mg_vcycle");
  if (nu < 1) return set_error(BSP_EINVAL, "nu must be >= 1");
  if (!(omega > 0.0)) return set_error(BSP_EINVAL, "omega must be positive");
  cudaStream_t s = (cudaStream_t)stream;
  bsp_grid* g = mg->g0;
  // the V-cycle expects b zero on the fixed DOFs: mask a copy into T[0]... T[0]
  // is the level-0 residual scratch, so use a dedicated copy
  int rc = ensure_wk(g, (size_t)g->n);
  if (rc) return rc;
  k_mask_copy<<<blocks_for(g->n, g->nsm), 256, 0, s>>>(d_b, g->fixbits, g->wk, g->n);
  BSP_CU(cudaGetLastError());
  return mg_vcycle_enqueue(mg, g->wk, d_x, omega, nu, nullptr, s);
}
