// Separable Gaussian density filter C and its exact adjoint C^T.
// Restates reference filtering.py:46-55 (apply_filter) and filtering.py:58-72
// (apply_filter_adjoint), with the truncate-and-renormalise boundary masses of
// filtering.py:38-43 computed in-kernel.  The activation a = v_phys^eta of
// solvers.py:443 is fused into the forward pass.
//
// B200 mapping: one CTA stages a (TY+2r) x (TX+2r) halo tile of the field in
// shared memory with coalesced fp64 loads, runs the two 1-D passes out of
// shared memory and writes TY x TX outputs (+ activation).  HBM traffic is one
// read + one (fwd: two) write per element; the halo re-read hits L2.
#include "common.cuh"
#include "filter.cuh"
#include "solver_state.cuh"

namespace bsp {

namespace {
constexpr int TX = 32;
constexpr int TY = 16;

BSP_DEV double axis_mass(const FilterTaps& w, int i, int len) {
  // kernel mass of the in-range taps at index i (correlate1d of ones, mode
  // constant, filtering.py:38-43): taps k with 0 <= i+k-r < len
  const int k0 = max(0, w.r - i);
  const int k1 = min(w.size, len - i + w.r);
  return w.cum[k1] - w.cum[k0];
}

BSP_DEV double spow(double x, double e) {
  // numpy fast-paths x**2.0 as a square and x**1.0 as identity; other
  // exponents go through pow like the reference's libm call
  if (e == 2.0) return x * x;
  if (e == 1.0) return x;
  return pow(x, e);
}
}  // namespace

// dynamic smem: in[(TY+2r)*(TX+2r)] + mid[(TY+2r)*TX]
__global__ void __launch_bounds__(256) k_filter_fwd(FilterArgs p) {
  if (p.gate0 && *p.gate0) return;
  extern __shared__ double sm[];
  const int r = p.w.r, W = TX + 2 * r, H = TY + 2 * r;
  double* tin = sm;
  double* mid = sm + W * H;
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int nx = p.nx, ny = p.ny;
  const int tid = threadIdx.x;
  for (int i = tid; i < W * H; i += blockDim.x) {
    int yy = i / W, xx = i % W;
    int gx = x0 + xx - r, gy = y0 + yy - r;
    tin[i] = (gx >= 0 && gx < nx && gy >= 0 && gy < ny) ? __ldg(p.in + (long long)gy * nx + gx)
                                                        : 0.0;
  }
  __syncthreads();
  // x pass over all H rows, TX columns
  for (int i = tid; i < TX * H; i += blockDim.x) {
    int yy = i / TX, xx = i % TX;
    int gx = x0 + xx;
    double s = 0.0;
    for (int k = 0; k < p.w.size; ++k) s += p.w.w[k] * tin[yy * W + xx + k];
    mid[yy * TX + xx] = (gx < nx) ? s / axis_mass(p.w, gx, nx) : 0.0;
  }
  __syncthreads();
  for (int i = tid; i < TX * TY; i += blockDim.x) {
    int yy = i / TX, xx = i % TX;
    int gx = x0 + xx, gy = y0 + yy;
    if (gx >= nx || gy >= ny) continue;
    double s = 0.0;
    for (int k = 0; k < p.w.size; ++k) s += p.w.w[k] * mid[(yy + k) * TX + xx];
    double vp = s / axis_mass(p.w, gy + p.gy0, p.gny);
    long long e = (long long)gy * nx + gx;
    p.out[e] = vp;
    if (p.act) p.act[e] = spow(vp, p.eta);
  }
}

__global__ void __launch_bounds__(256) k_filter_adj(FilterArgs p) {
  if (p.gate0 && *p.gate0) return;
  extern __shared__ double sm[];
  const int r = p.w.r, W = TX + 2 * r, H = TY + 2 * r;
  double* tin = sm;          // H x W, divided by sy on load
  double* mid = sm + W * H;  // TY x W, y-correlated then divided by sx
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int nx = p.nx, ny = p.ny;
  const int tid = threadIdx.x;
  for (int i = tid; i < W * H; i += blockDim.x) {
    int yy = i / W, xx = i % W;
    int gx = x0 + xx - r, gy = y0 + yy - r;
    double v = 0.0;
    if (gx >= 0 && gx < nx && gy >= 0 && gy < ny)
      v = __ldg(p.in + (long long)gy * nx + gx) / axis_mass(p.w, gy + p.gy0, p.gny);
    tin[i] = v;
  }
  __syncthreads();
  for (int i = tid; i < TY * W; i += blockDim.x) {
    int yy = i / W, xx = i % W;
    int gx = x0 + xx - r;
    double s = 0.0;
    for (int k = 0; k < p.w.size; ++k) s += p.w.w[k] * tin[(yy + k) * W + xx];
    mid[yy * W + xx] = (gx >= 0 && gx < nx) ? s / axis_mass(p.w, gx, nx) : 0.0;
  }
  __syncthreads();
  double gs = 0.0;
  for (int i = tid; i < TX * TY; i += blockDim.x) {
    int yy = i / TX, xx = i % TX;
    int gx = x0 + xx, gy = y0 + yy;
    if (gx >= nx || gy >= ny) continue;
    double s = 0.0;
    for (int k = 0; k < p.w.size; ++k) s += p.w.w[k] * mid[yy * W + xx + k];
    const long long e = (long long)gy * nx + gx;
    p.out[e] = s;
    if (p.st && gy >= p.red_y0 && gy < p.red_y1 && (!p.active || p.active[e])) gs += s;
  }
  if (p.st) {
    __shared__ double tot[4];
    double v4[4] = {gs, 0.0, 0.0, 0.0};
    if (grid_reduce_n<4>(p.rb, v4, tot) && threadIdx.x == 0) {
      if (p.defer_out)
        p.defer_out[0] = tot[0];
      else
        p.st->gsum = tot[0];
    }
  }
}

size_t filter_smem_bytes(int r) {
  const int W = TX + 2 * r, H = TY + 2 * r;
  return sizeof(double) * (size_t)(W * H + (size_t)(H > TY ? H : TY) * (TX > W ? TX : W));
}

dim3 filter_grid(int nx, int ny) { return dim3((nx + TX - 1) / TX, (ny + TY - 1) / TY); }

}  // namespace bsp
