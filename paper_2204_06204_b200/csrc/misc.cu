// Small stream-ordered helpers (axpy, Jacobi division, deterministic sums).
#include "misc.cuh"

namespace bsp {

__global__ void k_axpy(const double* x, const double* y, double c, double* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = x[i] + c * y[i];
}

__global__ void k_div_sq(const double* r, const double* d, double* out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double di = d[i];
    out[i] = r[i] / (di * di);
  }
}

__global__ void k_sum(const double* x, long long n, RedBuf rb, double* out) {
  double s = 0.0, s1 = 0.0, s2 = 0.0, m = -INFINITY;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    double v = x[i];
    s += v * v;
    s1 += v;
    m = nanmax(m, fabs(v));
  }
  __shared__ double tot[4];
  if (grid_reduce4(rb, s, s1, s2, m, tot)) {
    if (threadIdx.x == 0) {
      out[0] = tot[0];
      out[1] = tot[1];
      out[2] = tot[3];
    }
  }
}

__global__ void k_mean_sub(const double* g, long long n, const double* sum, double* out) {
  const double mu = sum[0] / (double)n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = g[i] - mu;
}

__global__ void k_kry_init(DevState* st) {
  double nb = sqrt(st->scratch[0]);
  st->norms[0] = nb;
  st->kry_count = 0;
  st->kry_stop = (nb == 0.0) ? 1 : 0;
  st->kry_rank = 0;
}

}  // namespace bsp
