// Krylov least-squares polynomial step (CPFBTO low level, reference
// solvers.py:205-255): tall-skinny QR of the normalised power basis.
//
// The reference factors the n x count basis with LAPACK dgeqrf, applies Q^T
// to b with dormqr and back-substitutes with dtrtrs after a 1e-13 rank cut.
// Gram / Cholesky-QR are numerically unusable here, so this is
// a Householder TSQR of the augmented matrix [P_1..P_count | b]: its R factor
// carries R (count x count) and Q^T b in the last column.
//   pass 1 (k_tsqr_local): a persistent grid; every CTA streams row chunks of
//          128 rows into shared memory under its running R and re-factors
//          [R; chunk] with Householder reflections -> one R per CTA;
//   pass 2 (k_tsqr_final): one CTA factors the stacked per-CTA R's the same
//          way, applies the rank cut and solves R c = Q^T b;
//   pass 3 (k_kry_combine): u_next = u - beta * sum_i c_i/(|P_i| growth_i) q_i.
// All orders are fixed -> bitwise deterministic.
#include "krylov.cuh"
#include "solver_state.cuh"

namespace bsp {

namespace {

constexpr int CH = 128;                 // rows per streamed chunk
constexpr int RMAX = 24;                // max columns (count+1) supported by TSQR
constexpr int LDS = RMAX + 1;           // padded smem row
constexpr int MROWS = RMAX + CH;        // stacked rows

struct QRSmem {
  double S[MROWS * LDS];
  double V[MROWS];
  double W[RMAX];
  double sc[4];
};

// Householder QR of S[0:M, 0:nc] in place, R in the top rows (LAPACK dlarfg
// convention: beta = -sign(alpha) * norm).  256 threads.
BSP_DEV void qr_block(QRSmem& q, int M, int nc) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarp = blockDim.x >> 5;
  for (int j = 0; j < nc; ++j) {
    double s = 0.0;
    for (int i = j + 1 + tid; i < M; i += blockDim.x) {
      double x = q.S[i * LDS + j];
      s += x * x;
    }
    double d1 = 0.0, d2 = 0.0, dm = 0.0;
    block_reduce4<false>(s, d1, d2, dm);
    if (tid == 0) {
      double alpha = q.S[j * LDS + j];
      double tau = 0.0, beta = alpha, scale = 0.0;
      if (s != 0.0) {
        double nrm = sqrt(alpha * alpha + s);
        beta = alpha >= 0.0 ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      q.sc[0] = tau;
      q.sc[1] = beta;
      q.sc[2] = scale;
    }
    __syncthreads();
    const double tau = q.sc[0], scale = q.sc[2];
    if (tau == 0.0) {
      __syncthreads();
      continue;
    }
    for (int i = j + 1 + tid; i < M; i += blockDim.x) q.V[i] = q.S[i * LDS + j] * scale;
    __syncthreads();
    // w_k = S[j][k] + sum_{i>j} v_i S[i][k]
    for (int k = j + 1 + warp; k < nc; k += nwarp) {
      double acc = 0.0;
      for (int i = j + 1 + lane; i < M; i += 32) acc += q.V[i] * q.S[i * LDS + k];
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) q.W[k] = q.S[j * LDS + k] + acc;
    }
    __syncthreads();
    const int ncol = nc - j - 1;
    if (ncol > 0) {
      for (int t = tid; t < (M - j) * ncol; t += blockDim.x) {
        int i = j + t / ncol, k = j + 1 + t % ncol;
        double vi = (i == j) ? 1.0 : q.V[i];
        q.S[i * LDS + k] -= tau * q.W[k] * vi;
      }
    }
    __syncthreads();
    if (tid == 0) q.S[j * LDS + j] = q.sc[1];
    __syncthreads();
  }
  // clear everything below the diagonal of the top block (the next chunk is
  // stacked under R)
  for (int t = tid; t < RMAX * RMAX; t += blockDim.x) {
    int i = t / RMAX, k = t % RMAX;
    if (k < i) q.S[i * LDS + k] = 0.0;
  }
  __syncthreads();
}

}  // namespace

__global__ void __launch_bounds__(256) k_tsqr_local(KryArgs p) {
  DevState* st = p.st;
  if (st->done || st->kry_count == 0) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  QRSmem& q = *reinterpret_cast<QRSmem*>(smraw);
  const int count = st->kry_count;
  const int nc = count + 1;
  const long long n = p.n;
  for (int t = threadIdx.x; t < MROWS * LDS; t += blockDim.x) q.S[t] = 0.0;
  __syncthreads();
  const long long nchunks = (n + CH - 1) / CH;
  for (long long c = blockIdx.x; c < nchunks; c += gridDim.x) {
    const long long r0 = c * CH;
    // column j<count: P_{j+1} = q_{j+1}/norms[j+1]; column count: b = q_0
    for (int t = threadIdx.x; t < CH * nc; t += blockDim.x) {
      int j = t / CH, i = t % CH;
      long long row = r0 + i;
      double x = 0.0;
      if (row < n) {
        if (j < count) x = __ldcg(p.Q + (long long)(j + 1) * p.ldq + row) / st->norms[j + 1];
        else x = __ldcg(p.Q + row);
      }
      q.S[(RMAX + i) * LDS + j] = x;
    }
    __syncthreads();
    qr_block(q, MROWS, nc);
  }
  double* out = p.Rbuf + (long long)blockIdx.x * RMAX * RMAX;
  for (int t = threadIdx.x; t < RMAX * RMAX; t += blockDim.x) {
    int i = t / RMAX, k = t % RMAX;
    out[t] = (i < nc && k < nc) ? q.S[i * LDS + k] : 0.0;
  }
}

__global__ void __launch_bounds__(256) k_tsqr_final(KryArgs p, int nblocks) {
  DevState* st = p.st;
  if (st->done || st->kry_count == 0) return;
  extern __shared__ __align__(16) unsigned char smraw[];
  QRSmem& q = *reinterpret_cast<QRSmem*>(smraw);
  const int count = st->kry_count;
  const int nc = count + 1;
  for (int t = threadIdx.x; t < MROWS * LDS; t += blockDim.x) q.S[t] = 0.0;
  __syncthreads();
  const int per = CH / RMAX;  // R blocks per chunk
  for (int b0 = 0; b0 < nblocks; b0 += per) {
    for (int t = threadIdx.x; t < CH * RMAX; t += blockDim.x) {
      int i = t / RMAX, k = t % RMAX;
      int blk = b0 + i / RMAX, ri = i % RMAX;
      double x = 0.0;
      if (i < per * RMAX && blk < nblocks && k < nc)
        x = __ldcg(p.Rbuf + (long long)blk * RMAX * RMAX + ri * RMAX + k);
      q.S[(RMAX + i) * LDS + k] = x;
    }
    __syncthreads();
    qr_block(q, MROWS, nc);
  }
  if (threadIdx.x == 0) {
    // rank cut |R_ii| <= 1e-13 |R_00| on the basis columns (solvers.py:212-214)
    double d0 = fabs(q.S[0]);
    int rank = count;
    for (int i = 0; i < count; ++i) {
      if (fabs(q.S[i * LDS + i]) <= 1e-13 * d0) { rank = i; break; }
    }
    double c[RMAX];
    for (int i = 0; i < RMAX; ++i) c[i] = 0.0;
    for (int i = rank - 1; i >= 0; --i) {
      double s = q.S[i * LDS + count];
      for (int k = i + 1; k < rank; ++k) s -= q.S[i * LDS + k] * c[k];
      c[i] = s / q.S[i * LDS + i];
    }
    for (int i = 0; i < count; ++i) st->coef[i] = c[i] / st->norms[i + 1] / st->norms[i];
    st->kry_rank = rank;
    if (p.coef_out) {
      for (int i = 0; i < count; ++i) p.coef_out[i] = c[i];
    }
  }
}

// u_next = u - beta * sum_i coef_i q_i   (solvers.py:255 + 280)
__global__ void __launch_bounds__(256) k_kry_combine(KryArgs p) {
  DevState* st = p.st;
  if (st->done) return;
  const int count = st->kry_count;
  const long long n = p.n;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double s = 0.0;
    for (int k = 0; k < count; ++k) s += st->coef[k] * __ldcg(p.Q + (long long)k * p.ldq + i);
    double base = p.u ? p.u[i] : 0.0;
    p.out[i] = base - p.beta * s;
  }
}

size_t tsqr_smem_bytes() { return sizeof(QRSmem); }
int tsqr_max_cols() { return RMAX; }

}  // namespace bsp
