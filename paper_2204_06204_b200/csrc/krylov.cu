// Krylov least-squares polynomial step (CPFBTO low level, reference
// solvers.py:205-255): tall-skinny QR of the normalised power basis.
//
// The reference factors the n x count basis with LAPACK dgeqrf, applies Q^T
// to b with dormqr and back-substitutes with dtrtrs after a 1e-13 rank cut.
// Gram / Cholesky-QR are numerically unusable here (kappa ~ 1e12..1e13, SURVEY
// §0.1-3), so this is a Householder TSQR of the augmented matrix
// [P_1..P_count | b]; its R factor carries R (count x count) and Q^T b in the
// last column.
//   leaves (k_tsqr_leaf): one CTA per 512-row chunk (or, for huge n, a
//          stream of chunks under a running R) -> one R per CTA;
//   merges (k_tsqr_merge): fan-in-16 tree; each CTA stacks 16 R factors and
//          re-factors them; the last level (one CTA) also applies the rank cut
//          and solves R c = Q^T b;
//   combine (k_kry_combine): u_next = u - beta * sum_i c_i/(|P_i| growth_i) q_i.
// Householder sweeps are column-per-warp: warp j holds column j of the
// panel in registers (row r at lane r%32, slot r/32).  For column j its owner
// forms the reflector (LAPACK dlarfg convention) and publishes the column to
// a double-buffered shared vector; after ONE barrier every warp k > j forms
// its dot product with a warp reduction and updates its own column in
// registers.  All reduction orders are fixed -> bitwise deterministic.
#include "krylov.cuh"
#include "solver_state.cuh"

namespace bsp {

namespace {

constexpr int CH = 512 - 24;      // rows per leaf chunk (panel = 512 rows = 16 slots)
constexpr int RMAX = 24;          // max columns (count+1) supported by TSQR
constexpr int LDS = RMAX + 1;     // padded smem row (final triangular solve)
constexpr int FAN = 16;           // merge fan-in
constexpr int NT = 32 * RMAX;     // one warp per column
constexpr int LROWS = RMAX + CH;  // leaf panel: running R on top of a chunk
constexpr int LSLOT = (LROWS + 31) / 32;
constexpr int MROWS = FAN * RMAX;  // merge panel: FAN stacked R factors
constexpr int MSLOT = MROWS / 32;

struct QRShared {
  double v[2][LSLOT * 32];  // published column j (unscaled, rows > j), by parity of j
  double scale[2], tau[2];
  int skip[2];
  double rnorm[RMAX];
  double R[RMAX * LDS];     // final R for the triangular solve
};

BSP_DEV double warp_sum(double x) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// Householder QR of the M x nc panel held column-per-warp in x (rows M..
// 32*T-1 are zero).  R ends in rows 0..nc-1; entries below the diagonal are
// zeroed.
template <int T>
BSP_DEV void qr_cols(double (&x)[T], int M, int nc, QRShared& sh) {
  static_assert(RMAX <= 32, "the diagonal rows sit in slot 0");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int j = 0; j < nc; ++j) {
    const int b = j & 1;
    if (w == j) {
      // sum_{i>j} x_i^2 with 4 independent partial chains
      double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int r = lane + 32 * t;
        const double xv = (r > j && r < M) ? x[t] : 0.0;
        s4[t & 3] += xv * xv;
      }
      const double sig = warp_sum((s4[0] + s4[1]) + (s4[2] + s4[3]));
      const double alpha = __shfl_sync(0xffffffffu, x[0], j);
      if (sig == 0.0) {  // H = I (dlarfg with x = 0)
        if (lane == 0) sh.skip[b] = 1;
      } else {
        const double nrm = sqrt(alpha * alpha + sig);
        const double beta = alpha >= 0.0 ? -nrm : nrm;
        if (lane == 0) {
          sh.skip[b] = 0;
          sh.tau[b] = (beta - alpha) / beta;
          sh.scale[b] = 1.0 / (alpha - beta);
        }
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int r = lane + 32 * t;
          sh.v[b][r] = r > j ? x[t] : 0.0;
          x[t] = r == j ? beta : (r > j ? 0.0 : x[t]);
        }
      }
    }
    __syncthreads();
    if (w > j && w < nc && !sh.skip[b]) {
      const double scale = sh.scale[b], tau = sh.tau[b];
      double a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int t = 0; t < T; ++t) a4[t & 3] += sh.v[b][lane + 32 * t] * x[t];  // v = 0 at r <= j, r >= M
      const double acc = warp_sum((a4[0] + a4[1]) + (a4[2] + a4[3]));
      const double xj = __shfl_sync(0xffffffffu, x[0], j);
      const double W = xj + scale * acc;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int r = lane + 32 * t;
        if (r >= j && r < M) {
          const double vi = (r == j) ? 1.0 : sh.v[b][r] * scale;
          x[t] -= (tau * vi) * W;
        }
      }
    }
  }
  __syncthreads();
}

// R factor (rows 0..nc-1 of the panel, slot 0) -> out[i * RMAX + k]
template <int T>
BSP_DEV void store_R(const double (&x)[T], double* out, int nc) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane < RMAX) out[lane * RMAX + w] = (lane < nc && w < nc && lane <= w) ? x[0] : 0.0;
}

}  // namespace

// leaves: CTA b streams chunks b, b+gridDim.x, ... of [P_1..P_count | b]
__global__ void __launch_bounds__(NT) k_tsqr_leaf(KryArgs p) {
  DevState* st = p.st;
  if (st->done || st->kry_count == 0) return;
  __shared__ QRShared sh;
  const int count = st->kry_count;
  const int nc = count + 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long n = p.n;
  double x[LSLOT];
#pragma unroll
  for (int t = 0; t < LSLOT; ++t) x[t] = 0.0;
  // warp w < count: basis column w+1 scaled by 1/|P_{w+1}|; warp count: b = q_0
  const double rn = w < count ? 1.0 / st->norms[w + 1] : 1.0;
  const double* col = w < count ? p.Q + (long long)(w + 1) * p.ldq : p.Q;
  const long long nchunks = (n + CH - 1) / CH;
  for (long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const long long r0 = c * CH - RMAX;  // panel row r holds basis row r0 + r (r >= RMAX)
    if (w < nc) {
#pragma unroll
      for (int t = 0; t < LSLOT; ++t) {
        const int r = lane + 32 * t;
        if (r >= RMAX) {
          const long long row = r0 + r;
          double v = 0.0;
          if (r < LROWS && row < n) v = __ldcg(col + row);
          x[t] = w < count ? v * rn : v;
        }
      }
    }
    qr_cols(x, LROWS, nc, sh);
  }
  if (w < RMAX) store_R(x, p.Rbuf + (long long)blockIdx.x * RMAX * RMAX, nc);
}

// merge FAN R factors per CTA; the single-CTA last level also solves
__global__ void __launch_bounds__(NT) k_tsqr_merge(KryArgs p, const double* Rin, int nin,
                                                   double* Rout) {
  DevState* st = p.st;
  if (st->done || st->kry_count == 0) return;
  __shared__ QRShared sh;
  const int count = st->kry_count;
  const int nc = count + 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b0 = blockIdx.x * FAN;
  const int nb = min(FAN, nin - b0);
  double x[MSLOT];
#pragma unroll
  for (int t = 0; t < MSLOT; ++t) {
    const int r = lane + 32 * t;
    const int blk = r / RMAX, ri = r - blk * RMAX;
    double v = 0.0;
    if (blk < nb && ri < nc && w < nc)
      v = __ldcg(Rin + (long long)(b0 + blk) * RMAX * RMAX + ri * RMAX + w);
    x[t] = v;
  }
  qr_cols(x, MROWS, nc, sh);
  if (gridDim.x > 1 || p.no_solve) {
    store_R(x, Rout + (long long)blockIdx.x * RMAX * RMAX, nc);
    return;
  }
  if (lane < RMAX) sh.R[lane * LDS + w] = x[0];
  __syncthreads();
  if (threadIdx.x == 0) {
    // rank cut |R_ii| <= 1e-13 |R_00| on the basis columns (solvers.py:212-214)
    const double* S = sh.R;
    const double d0 = fabs(S[0]);
    int rank = count;
    for (int i = 0; i < count; ++i) {
      if (fabs(S[i * LDS + i]) <= 1e-13 * d0) {
        rank = i;
        break;
      }
    }
    double c[RMAX];
    for (int i = 0; i < RMAX; ++i) c[i] = 0.0;
    for (int i = rank - 1; i >= 0; --i) {  // dtrtrs on R[:rank,:rank]
      double s = S[i * LDS + count];
      for (int k = i + 1; k < rank; ++k) s -= S[i * LDS + k] * c[k];
      c[i] = s / S[i * LDS + i];
    }
    for (int i = 0; i < count; ++i) st->coef[i] = c[i] / st->norms[i + 1] / st->norms[i];
    st->kry_rank = rank;
    if (p.coef_out)
      for (int i = 0; i < count; ++i) p.coef_out[i] = c[i];
  }
}

// u_next = u - beta * sum_i coef_i q_i   (solvers.py:255 + 280)
__global__ void __launch_bounds__(256) k_kry_combine(KryArgs p) {
  DevState* st = p.st;
  if (st->done) return;
  const int count = st->kry_count;
  __shared__ double coef[RMAX];
  if (threadIdx.x < RMAX) coef[threadIdx.x] = threadIdx.x < count ? st->coef[threadIdx.x] : 0.0;
  __syncthreads();
  const long long n = p.n;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double s = 0.0;
    for (int k = 0; k < count; ++k) s += coef[k] * __ldcg(p.Q + (long long)k * p.ldq + i);
    const double base = p.u ? p.u[i] : 0.0;
    p.out[i] = base - p.beta * s;
  }
}

size_t tsqr_smem_bytes() { return 0; }  // static shared memory only
int tsqr_threads() { return NT; }
cudaError_t tsqr_prepare() { return cudaSuccess; }
int tsqr_max_cols() { return RMAX; }
int tsqr_fan_in() { return FAN; }
int tsqr_leaves(long long n) {
  const long long chunks = (n + CH - 1) / CH;
  return (int)(chunks < 2048 ? chunks : 2048);
}

}  // namespace bsp
