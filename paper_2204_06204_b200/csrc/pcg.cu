// Preconditioned conjugate gradients as a fixed-step approximate inverse
// (north-star low-level step "u <- u - beta PCG_k(K(a), r)", SURVEY §8(a')),
// Jacobi- or multigrid-preconditioned.  `steps` CG iterations from x = 0;
// steps == 0 applies the preconditioner once (stationary: x = M r).
//
// Per CG step: k_stiff (q = K p with the grid-reduced p.Kp, HK_STORE), then
// k_pcg_update (x += alpha p, r -= alpha q; Jacobi: r.(r/d) reduced in the same
// pass), then the direction update (Jacobi: k_pcg_dir; MG: V-cycle, k_pcg_rz,
// k_pcg_dir).  The last step writes out = base - beta (x + alpha p) directly.
// All scalars stay on the device (graph-capturable, no host sync); every
// reduction is a fixed-order tree, so results are bitwise reproducible.
#include <algorithm>

#include "mg.cuh"

using namespace bsp;

namespace bsp {

__global__ void k_diag(GridView g, KeModes km, const double* __restrict__ a, double2* d);

namespace {
// The vectors are DOF vectors: n is even and every pointer is 16-byte aligned
// (whole nodes; row-slab offsets are whole node rows), so the streaming
// kernels move one double2 per thread-trip.
unsigned vec_blocks(long long n, int nsm) {
  long long b = (n / 2 + 255) / 256;
  return (unsigned)std::max<long long>(1, std::min<long long>(b, 16ll * nsm));
}

BSP_DEV double safe_div(double a, double b) { return (b > 0.0 && a > 0.0) ? a / b : 0.0; }

BSP_DEV double2 ld2(const double* p, long long i) { return reinterpret_cast<const double2*>(p)[i]; }
BSP_DEV void st2(double* p, long long i, double2 v) { reinterpret_cast<double2*>(p)[i] = v; }

#define BSP_PAIRS(i, n)                                                             \
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < (n) / 2; \
       i += (long long)gridDim.x * blockDim.x)
}  // namespace

// Jacobi start: R = b, P = b/D, sc[0] = b.(b/D)
__global__ void __launch_bounds__(256, 4) k_pcg_init_jacobi(const double* b, double* R, double* P, const double* D,
                                  double* sc, RedBuf rb, long long n, const int* gate,
                                  double* defer) {
  if (gate && *gate) return;
  double rz = 0.0;
  BSP_PAIRS(i, n) {
    const double2 bi = ld2(b, i), di = ld2(D, i);
    const double2 zi = make_double2(bi.x / di.x, bi.y / di.y);
    if (R != b) st2(R, i, bi);
    st2(P, i, zi);
    rz += bi.x * zi.x + bi.y * zi.y;
  }
  __shared__ double tot[4];
  double v[4] = {rz, 0.0, 0.0, 0.0};
  if (grid_reduce_n<4>(rb, v, tot) && threadIdx.x == 0) {
    if (defer)
      defer[0] = tot[0];  // row slabs: this rank's partial (all-gathered)
    else
      sc[0] = tot[0];
  }
}

// MG start (Z = V(b) already computed): R = b, P = Z, sc[0] = b.Z
// (defer: row slabs store this rank's partial there)
__global__ void __launch_bounds__(256, 4) k_pcg_init_z(const double* b, double* R, const double* Z, double* P, double* sc,
                             RedBuf rb, long long n, const int* gate, double* defer) {
  if (gate && *gate) return;
  double rz = 0.0;
  BSP_PAIRS(i, n) {
    const double2 bi = ld2(b, i), zi = ld2(Z, i);
    if (R != b) st2(R, i, bi);
    st2(P, i, zi);
    rz += bi.x * zi.x + bi.y * zi.y;
  }
  __shared__ double tot[4];
  double v[4] = {rz, 0.0, 0.0, 0.0};
  if (grid_reduce_n<4>(rb, v, tot) && threadIdx.x == 0) {
    if (defer)
      defer[0] = tot[0];
    else
      sc[0] = tot[0];
  }
}

// alpha = rz / p.Kp;  x += alpha p;  r -= alpha q;  (Jacobi) rz' = r.(r/D)
// LAST: out = base - beta (x + alpha p), nothing else written.  Compile-time
// variants keep the register count low enough for full occupancy; two pairs
// per thread-trip double the loads in flight.
template <bool LAST, bool JAC>
__global__ void __launch_bounds__(256, 4) k_pcg_update_t(double* X, double* R, const double* P,
                                                      const double* Q, const double* D,
                                                      double* sc, RedBuf rb, long long n,
                                                      int first, const double* base, double beta,
                                                      double* out, const int* gate,
                                                      double* defer) {
  if (gate && *gate) return;
  const double alpha = safe_div(sc[0], sc[1]);
  double rz = 0.0;
  const long long pairs = n / 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  auto one = [&](long long i) {
    const double2 pi = ld2(P, i);
    double2 xi = first ? make_double2(0.0, 0.0) : ld2(X, i);
    xi.x += alpha * pi.x;
    xi.y += alpha * pi.y;
    if (LAST) {
      const double2 bi = base ? ld2(base, i) : make_double2(0.0, 0.0);
      st2(out, i, make_double2(bi.x - beta * xi.x, bi.y - beta * xi.y));
      return;
    }
    st2(X, i, xi);
    const double2 qi = ld2(Q, i);
    double2 ri = ld2(R, i);
    ri.x -= alpha * qi.x;
    ri.y -= alpha * qi.y;
    st2(R, i, ri);
    if (JAC) {
      const double2 di = ld2(D, i);
      rz += ri.x * (ri.x / di.x) + ri.y * (ri.y / di.y);
    }
  };
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + stride < pairs; i += 2 * stride) {
    one(i);
    one(i + stride);
  }
  if (i < pairs) one(i);
  if (LAST || !JAC) return;
  __shared__ double tot[4];
  double v[4] = {rz, 0.0, 0.0, 0.0};
  if (grid_reduce_n<4>(rb, v, tot) && threadIdx.x == 0) {
    if (defer) {
      defer[0] = tot[0];  // row slabs: this rank's partial (all-gathered)
    } else {
      sc[6] = safe_div(tot[0], sc[0]);
      sc[0] = tot[0];
    }
  }
}

cudaError_t launch_pcg_update(unsigned blocks, cudaStream_t s, double* X, double* R,
                              const double* P, const double* Q, const double* D, double* sc,
                              RedBuf rb, long long n, int first, int last, const double* base,
                              double beta, double* out, const int* gate, double* defer) {
  if (last)
    k_pcg_update_t<true, false><<<blocks, 256, 0, s>>>(X, R, P, Q, D, sc, rb, n, first, base,
                                                       beta, out, gate, defer);
  else if (D)
    k_pcg_update_t<false, true><<<blocks, 256, 0, s>>>(X, R, P, Q, D, sc, rb, n, first, base,
                                                       beta, out, gate, defer);
  else
    k_pcg_update_t<false, false><<<blocks, 256, 0, s>>>(X, R, P, Q, D, sc, rb, n, first, base,
                                                        beta, out, gate, defer);
  return cudaGetLastError();
}

// rz' = R.Z, beta = rz'/rz (defer: row slabs store this rank's partial there)
__global__ void __launch_bounds__(256, 4) k_pcg_rz(const double* R, const double* Z, double* sc, RedBuf rb, long long n,
                         const int* gate, double* defer) {
  if (gate && *gate) return;
  double rz = 0.0;
  BSP_PAIRS(i, n) {
    const double2 ri = ld2(R, i), zi = ld2(Z, i);
    rz += ri.x * zi.x + ri.y * zi.y;
  }
  __shared__ double tot[4];
  double v[4] = {rz, 0.0, 0.0, 0.0};
  if (grid_reduce_n<4>(rb, v, tot) && threadIdx.x == 0) {
    if (defer) {
      defer[0] = tot[0];
    } else {
      sc[6] = safe_div(tot[0], sc[0]);
      sc[0] = tot[0];
    }
  }
}

// P = z + beta P, z = R/D (Jacobi) or Z (MG); two pairs per thread-trip
__global__ void __launch_bounds__(256, 4) k_pcg_dir(double* P, const double* R, const double* D,
                                                    const double* Z, const double* sc, long long n,
                                                    const int* gate) {
  if (gate && *gate) return;
  const double beta = sc[6];
  const long long pairs = n / 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  auto one = [&](long long i) {
    double2 zi;
    if (D) {
      const double2 ri = ld2(R, i), di = ld2(D, i);
      zi = make_double2(ri.x / di.x, ri.y / di.y);
    } else {
      zi = ld2(Z, i);
    }
    const double2 pi = ld2(P, i);
    st2(P, i, make_double2(zi.x + beta * pi.x, zi.y + beta * pi.y));
  };
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  for (; i + stride < pairs; i += 2 * stride) {
    one(i);
    one(i + stride);
  }
  if (i < pairs) one(i);
}

// steps == 0: out = base - beta z, z = b/D (Jacobi) or Z = V(b) (MG)
__global__ void k_pcg_apply0(const double* b, const double* D, const double* Z, const double* base,
                             double beta, double* out, long long n, const int* gate) {
  if (gate && *gate) return;
  BSP_PAIRS(i, n) {
    double2 zi;
    if (D) {
      const double2 bi = ld2(b, i), di = ld2(D, i);
      zi = make_double2(bi.x / di.x, bi.y / di.y);
    } else {
      zi = ld2(Z, i);
    }
    const double2 ba = base ? ld2(base, i) : make_double2(0.0, 0.0);
    st2(out, i, make_double2(ba.x - beta * zi.x, ba.y - beta * zi.y));
  }
}

int pcg_alloc(PcgWork& w, bsp_grid* g, bool with_mg) {
  pcg_free(w);
  const size_t nb = g->n * sizeof(double);
  const unsigned nbk = vec_blocks(g->n, g->nsm);
  bool ok = cudaMalloc(&w.X, nb) == cudaSuccess && cudaMalloc(&w.R, nb) == cudaSuccess &&
            cudaMalloc(&w.P, nb) == cudaSuccess && cudaMalloc(&w.Q, nb) == cudaSuccess &&
            cudaMalloc(&w.sc, 16 * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&w.cnt, sizeof(unsigned)) == cudaSuccess &&
            cudaMalloc(&w.part, 4ull * nbk * sizeof(double) + 64) == cudaSuccess;
  ok = ok && (with_mg ? cudaMalloc(&w.Z, nb) : cudaMalloc(&w.D, nb)) == cudaSuccess;
  if (!ok) {
    cudaGetLastError();
    pcg_free(w);
    return set_error(BSP_ENOMEM, "PCG workspace allocation failed (n=%lld)", g->n);
  }
  cudaMemset(w.cnt, 0, sizeof(unsigned));
  cudaMemset(w.sc, 0, 16 * sizeof(double));
  w.n = g->n;
  return BSP_OK;
}

void pcg_free(PcgWork& w) {
  cudaFree(w.X);
  cudaFree(w.R);
  cudaFree(w.P);
  cudaFree(w.Q);
  cudaFree(w.Z);
  cudaFree(w.D);
  cudaFree(w.sc);
  cudaFree(w.cnt);
  cudaFree(w.part);
  w = PcgWork{};
}

int pcg_enqueue(bsp_grid* g, PcgWork& w, bsp_mg* mg, const double* a, const double* b, int steps,
                double omega, int nu, const double* base, double beta, double* out,
                const int* gate, cudaStream_t s, bool setup) {
  if (steps < 0) return set_error(BSP_EINVAL, "PCG steps must be >= 0");
  if (!mg && !w.D) return set_error(BSP_EINVAL, "PCG workspace has no diagonal buffer");
  if (mg && !w.Z) return set_error(BSP_EINVAL, "PCG workspace has no preconditioner buffer");
  const long long n = g->n;
  const unsigned nb = vec_blocks(n, g->nsm);
  RedBuf rb{w.part, w.cnt};
  int rc;
  if (!mg) {
    k_diag<<<node_grid(g->nx, g->ny, wave_blocks((const void*)k_diag, 256)), 256, 0, s>>>(g->view(), g->km, a, (double2*)w.D);
    BSP_CU(cudaGetLastError());
  } else {
    if (setup) {
      rc = mg_setup_enqueue(mg, a, gate, s);
      if (rc) return rc;
    }
    rc = mg_vcycle_enqueue(mg, b, w.Z, omega, nu, gate, s);
    if (rc) return rc;
  }
  if (steps == 0) {
    k_pcg_apply0<<<nb, 256, 0, s>>>(b, mg ? nullptr : w.D, w.Z, base, beta, out, n, gate);
    BSP_CU(cudaGetLastError());
    return BSP_OK;
  }
  if (!mg)
    k_pcg_init_jacobi<<<nb, 256, 0, s>>>(b, w.R, w.P, w.D, w.sc, rb, n, gate, nullptr);
  else
    k_pcg_init_z<<<nb, 256, 0, s>>>(b, w.R, w.Z, w.P, w.sc, rb, n, gate, nullptr);
  BSP_CU(cudaGetLastError());
  for (int j = 0; j < steps; ++j) {
    StiffArgs q = stiff_args(g);
    q.a = a;
    q.u = (const double2*)w.P;
    q.out = (double2*)w.Q;
    q.flags = SF_REDUCE | SF_IN_MASKED;  // CG directions stay zero on fixed DOFs
    q.hook = HK_STORE;
    q.red_out = w.sc + 1;                // sc[1] = p.Kp
    q.red_need = 3;                      // (max|t| unused)
    q.gate0 = gate;
    BSP_CU(launch_stiff(g, q, s));
    const int last = j == steps - 1;
    BSP_CU(launch_pcg_update(nb, s, w.X, w.R, w.P, w.Q, mg ? nullptr : w.D, w.sc, rb, n, j == 0,
                             last, base, beta, out, gate, nullptr));
    if (last) break;
    if (mg) {
      rc = mg_vcycle_enqueue(mg, w.R, w.Z, omega, nu, gate, s);
      if (rc) return rc;
      k_pcg_rz<<<nb, 256, 0, s>>>(w.R, w.Z, w.sc, rb, n, gate, nullptr);
      BSP_CU(cudaGetLastError());
    }
    k_pcg_dir<<<nb, 256, 0, s>>>(w.P, w.R, mg ? nullptr : w.D, w.Z, w.sc, n, gate);
    BSP_CU(cudaGetLastError());
  }
  return BSP_OK;
}

}  // namespace bsp

namespace bsp {
__global__ void k_mask_copy(const double* x0, const uint32_t* fixbits, double* x, long long n);
}

extern "C" int bsp_pcg_apply(bsp_grid* g, bsp_mg* mg, const double* d_a, const double* d_b,
                             int steps, double omega, int nu, const double* d_base, double beta,
                             double* d_out, void* stream) {
  if (!g || !d_a || !d_b || !d_out) return set_error(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(g->device);
  if (steps < 0) return set_error(BSP_EINVAL, "steps must be >= 0");
  if (mg && mg->g0 != g) return set_error(BSP_EINVAL, "multigrid built for another grid");
  if (mg && (nu < 1 || !(omega > 0.0))) return set_error(BSP_EINVAL, "need nu >= 1 and omega > 0");
  if (!g->uniform_diag) return set_error(BSP_EUNSUPPORTED, "PCG needs a uniform ke diagonal");
  cudaStream_t s = (cudaStream_t)stream;
  PcgWork*& wp = g->pcg_ws[mg ? 1 : 0];  // per grid, built on first use
  if (!wp) {
    wp = new PcgWork();
    int rc = pcg_alloc(*wp, g, mg != nullptr);
    if (rc) {
      delete wp;
      wp = nullptr;
      return rc;
    }
  }
  PcgWork& w = *wp;
  // b masked into R (consumed by the iteration)
  k_mask_copy<<<vec_blocks(g->n, g->nsm), 256, 0, s>>>(d_b, g->fixbits, w.R, g->n);
  BSP_CU(cudaGetLastError());
  return pcg_enqueue(g, w, mg, d_a, w.R, steps, omega, nu, d_base, beta, d_out, nullptr, s);
}
