// Geometric multigrid hierarchy and V-cycle (see mg.cuh for the algorithm).
//
// B200 mapping: every smoother / residual sweep is the same strip kernel as
// the matvec (k_stiff, stiffness.cu) with the SF_SUB_LOAD (rhs) + SF_D1DIV +
// SF_AXPY epilogue, so a Jacobi sweep costs one matvec of HBM traffic
// (u, b read, x written, a read).  Restriction fuses the next level's first
// (from-zero) Jacobi sweep; prolongation adds in place.  The coarsest level
// (<= 80 DOFs) is one CTA: assembly + in-shared-memory Gauss-Jordan inverse
// once per activation, a dense 80x80 matvec per V-cycle.
#include <algorithm>
#include <cstring>
#include <vector>

#include "mg.cuh"

using namespace bsp;

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
  const double dx = km.kdx * asum, dy = km.kdy * asum;
  double2 x;
  x.x = ((bits & 1u) || dx == 0.0) ? 0.0 : omega * b.x / dx;
  x.y = ((bits & 2u) || dy == 0.0) ? 0.0 : omega * b.y / dy;
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
__global__ void k_mg_restrict(const double2* __restrict__ t, int nx, int ny, double2* __restrict__ bc,
                              double2* __restrict__ xc, const double* __restrict__ ac, int nxc,
                              int nyc, const uint32_t* __restrict__ fixc, KeModes km, double omega,
                              const int* gate) {
  if (gate && *gate) return;
  const long long Nc = (long long)(nxc + 1) * (nyc + 1);
  for (long long J = blockIdx.x * (long long)blockDim.x + threadIdx.x; J < Nc;
       J += (long long)gridDim.x * blockDim.x) {
    const int X = (int)(J % (nxc + 1)), Y = (int)(J / (nxc + 1));
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
    const uint32_t bits = fix_bits(fixc, J);
    const double2 b = apply_mask(make_double2(-sx, -sy), bits);
    bc[J] = b;
    xc[J] = jacobi_start(b, bits, node_asum(ac, nxc, nyc, X, Y), km, omega);
  }
}

// x += M_f P~ x_c  (in place; each fine node reads only coarse values)
__global__ void k_mg_prolong(double2* __restrict__ x, int nx, int ny, const uint32_t* __restrict__ fixf,
                             const double2* __restrict__ xc, int nxc, const int* gate) {
  if (gate && *gate) return;
  const long long N = (long long)(nx + 1) * (ny + 1);
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N;
       j += (long long)gridDim.x * blockDim.x) {
    const int xx = (int)(j % (nx + 1)), yy = (int)(j / (nx + 1));
    const int X0 = xx >> 1, Y0 = yy >> 1, ox = xx & 1, oy = yy & 1;
    const double w = (ox ? 0.5 : 1.0) * (oy ? 0.5 : 1.0);
    double sx = 0.0, sy = 0.0;
    for (int iy = 0; iy <= oy; ++iy)
      for (int ix = 0; ix <= ox; ++ix) {
        const double2 v = xc[(long long)(Y0 + iy) * (nxc + 1) + X0 + ix];
        sx += w * v.x;
        sy += w * v.y;
      }
    const uint32_t bits = fix_bits(fixf, j);
    double2 o = x[j];
    if (!(bits & 1u)) o.x += sx;
    if (!(bits & 2u)) o.y += sy;
    x[j] = o;
  }
}

// level 0 first sweep from zero: x = omega D^{-1} b
__global__ void k_mg_jacobi0(const double2* __restrict__ b, double2* __restrict__ x,
                             const double* __restrict__ a, int nx, int ny,
                             const uint32_t* __restrict__ fix, KeModes km, double omega,
                             const int* gate) {
  if (gate && *gate) return;
  const long long N = (long long)(nx + 1) * (ny + 1);
  for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < N;
       j += (long long)gridDim.x * blockDim.x) {
    const int xx = (int)(j % (nx + 1)), yy = (int)(j / (nx + 1));
    x[j] = jacobi_start(b[j], fix_bits(fix, j), node_asum(a, nx, ny, xx, yy), km, omega);
  }
}

// coarsest level: assemble K(a) densely (fixed DOFs -> identity rows/cols)
// and invert it by in-place Gauss-Jordan (SPD: no pivoting).  The matrix
// lives in registers, kFactorPer entries per thread at fixed (i, j); pivot k
// reads the old column k and row k from a double-buffered shared copy that
// their owners refresh after each update, so a pivot costs one barrier.  The
// arithmetic is A_ij - A_ik (A_kj / A_kk) in that order.
constexpr int kFactorThreads = 1024;
constexpr int kFactorPer = ((2 * kCoarseNodes + 2) * (2 * kCoarseNodes + 2) + kFactorThreads - 1) /
                           kFactorThreads;

__global__ void __launch_bounds__(kFactorThreads) k_mg_coarse_factor(
    const double* __restrict__ a, int nx, int ny, const uint32_t* __restrict__ fix,
    const double* __restrict__ ke, double* __restrict__ Ainv, int nc, const int* gate) {
  if (gate && *gate) return;
  __shared__ double col[2][2 * kCoarseNodes + 2], row[2][2 * kCoarseNodes + 2];
  const int NX1 = nx + 1;
  double A[kFactorPer];
  int I[kFactorPer], J[kFactorPer];
#pragma unroll
  for (int m = 0; m < kFactorPer; ++m) {
    const int t = threadIdx.x + m * kFactorThreads;
    I[m] = t < nc * nc ? t / nc : -1;
    J[m] = t < nc * nc ? t % nc : -1;
    double v = 0.0;
    if (I[m] >= 0) {
      const int nI = I[m] >> 1, cI = I[m] & 1, nJ = J[m] >> 1, cJ = J[m] & 1;
      const bool fI = (fix_bits(fix, nI) >> cI) & 1u, fJ = (fix_bits(fix, nJ) >> cJ) & 1u;
      if (fI || fJ) {
        v = (I[m] == J[m]) ? 1.0 : 0.0;
      } else {
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
      }
      if (J[m] == 0) col[0][I[m]] = v;
      if (I[m] == 0) row[0][J[m]] = v;
    }
    A[m] = v;
  }
  __syncthreads();
  for (int k = 0; k < nc; ++k) {
    const int b = k & 1;
    const double piv = row[b][k];
    const double ip = piv != 0.0 ? 1.0 / piv : 0.0;
#pragma unroll
    for (int m = 0; m < kFactorPer; ++m) {
      if (I[m] < 0) continue;
      const int i = I[m], j = J[m];
      double v;
      if (i == k)
        v = (j == k) ? ip : A[m] * ip;
      else
        v = (j == k) ? -col[b][i] * ip : A[m] - col[b][i] * (row[b][j] * ip);
      A[m] = v;
      if (j == k + 1) col[b ^ 1][i] = v;
      if (i == k + 1) row[b ^ 1][j] = v;
    }
    __syncthreads();
  }
#pragma unroll
  for (int m = 0; m < kFactorPer; ++m)
    if (I[m] >= 0) Ainv[I[m] * nc + J[m]] = A[m];
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

namespace {
unsigned blocks_for(long long n, int nsm) {
  long long b = (n + 255) / 256;
  return (unsigned)std::max<long long>(1, std::min<long long>(b, 8ll * nsm));
}

cudaError_t smooth(bsp_grid* g, const double* a, const double* b, const double* x, double* out,
                   double omega, const int* gate, cudaStream_t s) {
  StiffArgs p = stiff_args(g);
  p.a = a;
  p.u = (const double2*)x;
  p.rhs = (const double2*)b;
  p.base = (const double2*)x;
  p.beta = omega;
  p.out = (double2*)out;
  p.flags = SF_IN_MASKED | SF_SUB_LOAD | SF_D1DIV | SF_AXPY;
  p.gate0 = gate;
  return launch_stiff(g, p, s);
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

int mg_setup_enqueue(bsp_mg* mg, const double* a0, const int* gate, cudaStream_t s) {
  mg->a[0] = const_cast<double*>(a0);
  for (int l = 0; l < mg->L; ++l) {
    bsp_grid* f = mg->lv[l];
    bsp_grid* c = mg->lv[l + 1];
    k_mg_coarsen<<<blocks_for(c->E, f->nsm), 256, 0, s>>>(mg->a[l], f->nx, f->ny, mg->a[l + 1],
                                                          c->nx, c->ny, gate);
    BSP_CU(cudaGetLastError());
  }
  bsp_grid* cL = mg->lv[mg->L];
  k_mg_coarse_factor<<<1, kFactorThreads, 0, s>>>(mg->a[mg->L], cL->nx, cL->ny, cL->fixbits,
                                                  mg->ke, mg->Ainv, mg->nc, gate);
  BSP_CU(cudaGetLastError());
  return BSP_OK;
}

int mg_vcycle_enqueue(bsp_mg* mg, const double* b0, double* out0, double omega, int nu,
                      const int* gate, cudaStream_t s) {
  const int L = mg->L;
  if (L == 0) {
    k_mg_coarse_solve<<<1, 128, 0, s>>>(mg->Ainv, mg->nc, b0, out0, gate);
    BSP_CU(cudaGetLastError());
    return BSP_OK;
  }
  std::vector<double*> cur(L + 1, nullptr);
  auto other = [&](int l, double* p) { return p == mg->X[l] ? mg->Y[l] : mg->X[l]; };
  for (int l = 0; l < L; ++l) {
    bsp_grid* g = mg->lv[l];
    const double* b = l == 0 ? b0 : mg->B[l];
    double* x = mg->X[l];
    if (l == 0) {
      k_mg_jacobi0<<<blocks_for(g->N, g->nsm), 256, 0, s>>>((const double2*)b0, (double2*)x,
                                                            mg->a[0], g->nx, g->ny, g->fixbits,
                                                            g->km, omega, gate);
      BSP_CU(cudaGetLastError());
    }
    for (int it = 1; it < nu; ++it) {
      double* nx_ = other(l, x);
      BSP_CU(smooth(g, mg->a[l], b, x, nx_, omega, gate, s));
      x = nx_;
    }
    cur[l] = x;
    BSP_CU(residual(g, mg->a[l], b, x, mg->T[l], gate, s));
    bsp_grid* c = mg->lv[l + 1];
    k_mg_restrict<<<blocks_for(c->N, g->nsm), 256, 0, s>>>(
        (const double2*)mg->T[l], g->nx, g->ny, (double2*)mg->B[l + 1], (double2*)mg->X[l + 1],
        mg->a[l + 1], c->nx, c->ny, c->fixbits, c->km, omega, gate);
    BSP_CU(cudaGetLastError());
  }
  // coarsest: direct solve B[L] -> Y[L]
  k_mg_coarse_solve<<<1, 128, 0, s>>>(mg->Ainv, mg->nc, mg->B[L], mg->Y[L], gate);
  BSP_CU(cudaGetLastError());
  const double* res = mg->Y[L];
  for (int l = L - 1; l >= 0; --l) {
    bsp_grid* g = mg->lv[l];
    bsp_grid* c = mg->lv[l + 1];
    const double* b = l == 0 ? b0 : mg->B[l];
    double* x = cur[l];
    k_mg_prolong<<<blocks_for(g->N, g->nsm), 256, 0, s>>>((double2*)x, g->nx, g->ny, g->fixbits,
                                                          (const double2*)res, c->nx, gate);
    BSP_CU(cudaGetLastError());
    for (int it = 0; it < nu; ++it) {
      double* dst = (l == 0 && it == nu - 1) ? out0 : other(l, x);
      BSP_CU(smooth(g, mg->a[l], b, x, dst, omega, gate, s));
      x = dst;
    }
    res = x;
  }
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
  delete mg;
  return BSP_OK;
}

extern "C" int bsp_mg_create(bsp_grid* g, int max_levels, bsp_mg** out) {
  if (!g || !out) return set_error(BSP_EINVAL, "null argument");
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
  return mg_setup_enqueue(mg, d_a, nullptr, (cudaStream_t)stream);
}

namespace bsp {
__global__ void k_mask_copy(const double* x0, const uint32_t* fixbits, double* x, long long n);
}

extern "C" int bsp_mg_vcycle(bsp_mg* mg, const double* d_b, double* d_x, double omega, int nu,
                             void* stream) {
  if (!mg || !d_b || !d_x) return set_error(BSP_EINVAL, "null argument");
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
