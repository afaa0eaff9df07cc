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
//   merges (k_tsqr_merge): fan-in-8 tree; each CTA stacks 8 R factors and
//          re-factors them; the last level (one CTA) also applies the rank cut
//          and solves R c = Q^T b;
//   combine (k_kry_combine): u_next = u - beta * sum_i c_i/(|P_i| growth_i) q_i.
// Householder sweeps need 3 block barriers per column (norm partials, dot
// products, update); all reduction orders are fixed -> bitwise deterministic.
#include "krylov.cuh"
#include "solver_state.cuh"

namespace bsp {

namespace {

constexpr int CH = 512;        // rows per leaf chunk (fewer leaves and merge levels, 4x rows per sync)
constexpr int RMAX = 24;       // max columns (count+1) supported by TSQR
constexpr int LDS = RMAX + 1;  // padded smem row
constexpr int FAN = 8;         // merge fan-in
constexpr int MROWS = RMAX + CH > FAN * RMAX ? RMAX + CH : FAN * RMAX;
constexpr int NT = 256;        // threads per CTA
constexpr int NW = NT / 32;

struct QRSmem {
  double S[MROWS * LDS];
  double W[RMAX];
  double part[NW];
  double rnorm[RMAX];
};

// Householder QR of S[0:M, 0:nc] in place (LAPACK dlarfg convention:
// beta = -sign(alpha) * norm); R ends in the top nc rows, the strictly lower
// triangle of the top RMAX x RMAX block is cleared for the next stacking.
BSP_DEV void qr_block(QRSmem& q, int M, int nc) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = 0; j < nc; ++j) {
    double s = 0.0;
    for (int i = j + 1 + tid; i < M; i += NT) {
      const double x = q.S[i * LDS + j];
      s += x * x;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) q.part[warp] = s;
    __syncthreads();  // (1) norm partials ready; previous column's update done
    double sig = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) sig += q.part[w];
    const double alpha = q.S[j * LDS + j];
    if (sig == 0.0) {  // H = I (dlarfg with x = 0)
      __syncthreads();
      continue;
    }
    const double nrm = sqrt(alpha * alpha + sig);
    const double beta = alpha >= 0.0 ? -nrm : nrm;
    const double tau = (beta - alpha) / beta;
    const double scale = 1.0 / (alpha - beta);
    // w_k = S[j][k] + sum_{i>j} v_i S[i][k], v_i = S[i][j] * scale
    for (int k = j + 1 + warp; k < nc; k += NW) {
      double acc = 0.0;
      for (int i = j + 1 + lane; i < M; i += 32) acc += q.S[i * LDS + j] * q.S[i * LDS + k];
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) q.W[k] = q.S[j * LDS + k] + scale * acc;
    }
    __syncthreads();  // (2) W ready, everyone done reading column j's x
    for (int i = j + tid; i < M; i += NT) {
      const double vi = (i == j) ? 1.0 : q.S[i * LDS + j] * scale;
      const double tv = tau * vi;
      for (int k = j + 1; k < nc; ++k) q.S[i * LDS + k] -= tv * q.W[k];
    }
    __syncthreads();  // (3) update done (S[i][j], i > j, no longer needed)
    if (tid == 0) q.S[j * LDS + j] = beta;
  }
  __syncthreads();
  for (int t = tid; t < RMAX * RMAX; t += NT) {
    const int i = t / RMAX, k = t % RMAX;
    if (k < i) q.S[i * LDS + k] = 0.0;
  }
  __syncthreads();
}

BSP_DEV void zero_smem(QRSmem& q) {
  for (int t = threadIdx.x; t < MROWS * LDS; t += NT) q.S[t] = 0.0;
  __syncthreads();
}

BSP_DEV void store_R(const QRSmem& q, double* out, int nc) {
  for (int t = threadIdx.x; t < RMAX * RMAX; t += NT) {
    const int i = t / RMAX, k = t % RMAX;
    out[t] = (i < nc && k < nc) ? q.S[i * LDS + k] : 0.0;
  }
}

}  // namespace

// leaves: CTA b streams chunks b, b+gridDim.x, ... of [P_1..P_count | b]
__global__ void __launch_bounds__(NT) k_tsqr_leaf(KryArgs p) {
  DevState* st = p.st;
  if (st->done || st->kry_count == 0) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  QRSmem& q = *reinterpret_cast<QRSmem*>(smraw);
  const int count = st->kry_count;
  const int nc = count + 1;
  const long long n = p.n;
  if (threadIdx.x < RMAX) q.rnorm[threadIdx.x] = threadIdx.x < count ? 1.0 / st->norms[threadIdx.x + 1] : 1.0;
  zero_smem(q);
  const long long nchunks = (n + CH - 1) / CH;
  for (long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const long long r0 = c * CH;
    for (int t = threadIdx.x; t < CH * nc; t += NT) {
      const int j = t / CH, i = t - j * CH;
      const long long row = r0 + i;
      double x = 0.0;
      if (row < n) {
        if (j < count) x = __ldcg(p.Q + (long long)(j + 1) * p.ldq + row) * q.rnorm[j];
        else x = __ldcg(p.Q + row);
      }
      q.S[(RMAX + i) * LDS + j] = x;
    }
    __syncthreads();
    qr_block(q, RMAX + CH, nc);
  }
  store_R(q, p.Rbuf + (long long)blockIdx.x * RMAX * RMAX, nc);
}

// merge FAN R factors per CTA; the single-CTA last level also solves
__global__ void __launch_bounds__(NT) k_tsqr_merge(KryArgs p, const double* Rin, int nin,
                                                   double* Rout) {
  DevState* st = p.st;
  if (st->done || st->kry_count == 0) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  QRSmem& q = *reinterpret_cast<QRSmem*>(smraw);
  const int count = st->kry_count;
  const int nc = count + 1;
  const int b0 = blockIdx.x * FAN;
  const int nb = min(FAN, nin - b0);
  for (int t = threadIdx.x; t < FAN * RMAX * LDS; t += NT) {
    const int row = t / LDS, k = t - row * LDS;
    const int blk = row / RMAX, ri = row - blk * RMAX;
    double x = 0.0;
    if (blk < nb && k < nc && ri < nc) x = __ldcg(Rin + (long long)(b0 + blk) * RMAX * RMAX + ri * RMAX + k);
    q.S[row * LDS + k] = x;
  }
  __syncthreads();
  qr_block(q, FAN * RMAX, nc);
  if (gridDim.x > 1 || p.no_solve) {
    store_R(q, Rout + (long long)blockIdx.x * RMAX * RMAX, nc);
    return;
  }
  if (threadIdx.x == 0) {
    // rank cut |R_ii| <= 1e-13 |R_00| on the basis columns (solvers.py:212-214)
    const double d0 = fabs(q.S[0]);
    int rank = count;
    for (int i = 0; i < count; ++i) {
      if (fabs(q.S[i * LDS + i]) <= 1e-13 * d0) {
        rank = i;
        break;
      }
    }
    double c[RMAX];
    for (int i = 0; i < RMAX; ++i) c[i] = 0.0;
    for (int i = rank - 1; i >= 0; --i) {  // dtrtrs on R[:rank,:rank]
      double s = q.S[i * LDS + count];
      for (int k = i + 1; k < rank; ++k) s -= q.S[i * LDS + k] * c[k];
      c[i] = s / q.S[i * LDS + i];
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

size_t tsqr_smem_bytes() { return sizeof(QRSmem); }

cudaError_t tsqr_prepare() {
  // > 48 KB of dynamic shared memory needs the opt-in, once per process
  static cudaError_t e = [] {
    cudaError_t r = cudaFuncSetAttribute(k_tsqr_leaf, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)tsqr_smem_bytes());
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(k_tsqr_merge, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)tsqr_smem_bytes());
    return r;
  }();
  return e;
}
int tsqr_max_cols() { return RMAX; }
int tsqr_fan_in() { return FAN; }
int tsqr_leaves(long long n) {
  const long long chunks = (n + CH - 1) / CH;
  return (int)(chunks < 2048 ? chunks : 2048);
}

}  // namespace bsp
