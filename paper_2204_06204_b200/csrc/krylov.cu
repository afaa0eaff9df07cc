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
//
// Two widths: the narrow variant (24 columns, one per warp, 512-row leaves,
// fan-in 16) runs the paper's D = 20; the wide one (64 columns, two per warp
// in 32 warps, 256-row leaves, fan-in 4) runs krylov_dim up to 62.  Beyond
// that only the first 63 powers are formed: the reference's answer depends on
// the first `rank` columns only (reflector k touches rows >= k, and the
// coefficients past the 1e-13 rank cut are zero, solvers.py:212-219), so the
// result is the reference's whenever the cut falls inside those columns --
// which the solve checks (DevState::kry_trunc) -- and the power basis is
// numerically rank-deficient long before 63 columns (|R_ii|/|R_00| reaches
// the cut by column ~21).
#include "krylov.cuh"
#include "solver_state.cuh"

namespace bsp {

namespace {

template <int RM_, int CPW_, int CH_, int FAN_>
struct TsqrCfg {
  static constexpr int RM = RM_;                   // max columns (count + 1)
  static constexpr int CPW = CPW_;                 // columns per warp
  static constexpr int NW = (RM_ + CPW_ - 1) / CPW_;  // warps: column c at warp c % NW, slot c / NW
  static constexpr int NT = 32 * NW;
  static constexpr int CH = CH_;                   // rows per leaf chunk
  static constexpr int LROWS = RM_ + CH_;          // leaf panel: running R on top of a chunk
  static constexpr int LSLOT = (LROWS + 31) / 32;
  static constexpr int FAN = FAN_;                 // merge fan-in
  static constexpr int MROWS = FAN_ * RM_;         // merge panel: FAN stacked R factors
  static constexpr int MSLOT = (MROWS + 31) / 32;
  static constexpr int LDS = RM_ + 1;              // padded smem row (final triangular solve)
};
using Narrow = TsqrCfg<24, 1, 512 - 24, 16>;
// Large n: 1024-row leaf panels.  The leaf is bound by its chain of
// Householder columns per chunk (each a warp reduction, a barrier and the
// trailing update), so twice the rows per chain halves the chains: C5
// cpfbto 73.3 -> 56.8 ms/iter.  Small n keeps 512 rows (more leaves in
// flight: C1 0.263 vs 0.300 ms/iter with 1024).
using NarrowL = TsqrCfg<24, 1, 1024 - 24, 16>;
constexpr long long kLargeLeafN = 1ll << 20;
using Wide = TsqrCfg<64, 2, 256 - 64, 4>;

template <class K>
struct QRShared {
  double v[2][K::LSLOT * 32 > K::MSLOT * 32 ? K::LSLOT * 32 : K::MSLOT * 32];
  double scale[2], tau[2];
  int skip[2];
  double R[K::RM * K::LDS];  // final R for the triangular solve
};

BSP_DEV double warp_sum(double x) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// row r of one register column (row r at lane r % 32, slot r / 32)
template <int T>
BSP_DEV double row_of(const double (&x)[T], int r) {
  double v = 0.0;
#pragma unroll
  for (int t = 0; t < T; ++t)
    if (t == (r >> 5)) v = x[t];
  return __shfl_sync(0xffffffffu, v, r & 31);
}

// Householder QR of the M x nc panel held column-per-warp in x (rows M..
// 32*T-1 are zero): column c at warp c % NW, register slot c / NW.  R ends in
// rows 0..nc-1; entries below the diagonal are zeroed.
template <class K, int T>
BSP_DEV void qr_cols(double (&x)[K::CPW][T], int M, int nc, QRShared<K>& sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int j = 0; j < nc; ++j) {
    const int b = j & 1;
    if (w == j % K::NW) {
#pragma unroll
      for (int cs = 0; cs < K::CPW; ++cs) {
        if (cs != j / K::NW) continue;  // warp-uniform
        // sum_{i>j} x_i^2 with 4 independent partial chains
        double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int r = lane + 32 * t;
          const double xv = (r > j && r < M) ? x[cs][t] : 0.0;
          s4[t & 3] += xv * xv;
        }
        const double sig = warp_sum((s4[0] + s4[1]) + (s4[2] + s4[3]));
        const double alpha = row_of(x[cs], j);
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
            sh.v[b][r] = r > j ? x[cs][t] : 0.0;
            x[cs][t] = r == j ? beta : (r > j ? 0.0 : x[cs][t]);
          }
        }
      }
    }
    __syncthreads();
    if (!sh.skip[b]) {
      const double scale = sh.scale[b], tau = sh.tau[b];
#pragma unroll
      for (int cs = 0; cs < K::CPW; ++cs) {
        const int c = w + K::NW * cs;
        if (c <= j || c >= nc) continue;  // warp-uniform
        double a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int t = 0; t < T; ++t) a4[t & 3] += sh.v[b][lane + 32 * t] * x[cs][t];  // v = 0 at r <= j, r >= M
        const double acc = warp_sum((a4[0] + a4[1]) + (a4[2] + a4[3]));
        const double xj = row_of(x[cs], j);
        const double W = xj + scale * acc;
#pragma unroll
        for (int t = 0; t < T; ++t) {
          const int r = lane + 32 * t;
          if (r >= j && r < M) {
            const double vi = (r == j) ? 1.0 : sh.v[b][r] * scale;
            x[cs][t] -= (tau * vi) * W;
          }
        }
      }
    }
  }
  __syncthreads();
}

// R factor (rows 0..nc-1 of the panel) -> out[i * RM + k]
template <class K, int T>
BSP_DEV void store_R(const double (&x)[K::CPW][T], double* out, int nc) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int cs = 0; cs < K::CPW; ++cs) {
    const int c = w + K::NW * cs;
    if (c >= K::RM) continue;
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int r = lane + 32 * t;
      if (r < K::RM) out[r * K::RM + c] = (r < nc && c < nc && r <= c) ? x[cs][t] : 0.0;
    }
  }
}

// leaves: CTA b streams chunks b, b+gridDim.x, ... of [P_1..P_count | b]
template <class K>
BSP_DEV void tsqr_leaf(const KryArgs& p) {
  DevState* st = p.st;
  if (st->done || st->kry_count == 0) return;
  __shared__ QRShared<K> sh;
  const int count = min(st->kry_count, K::RM - 1);
  const int nc = count + 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long long n = p.n;
  double x[K::CPW][K::LSLOT];
  const double* col[K::CPW];
  double rn[K::CPW];
#pragma unroll
  for (int cs = 0; cs < K::CPW; ++cs) {
    // column c < count: basis column c+1 scaled by 1/|P_{c+1}|; column count: b = q_0
    const int c = w + K::NW * cs;
    rn[cs] = c < count ? 1.0 / st->norms[c + 1] : 1.0;
    col[cs] = c < count ? p.Q + (long long)(c + 1) * p.ldq : p.Q;
#pragma unroll
    for (int t = 0; t < K::LSLOT; ++t) x[cs][t] = 0.0;
  }
  const long long nchunks = (n + K::CH - 1) / K::CH;
  for (long long ck = blockIdx.x; ck < nchunks; ck += gridDim.x) {
    const long long r0 = ck * K::CH - K::RM;  // panel row r holds basis row r0 + r (r >= RM)
#pragma unroll
    for (int cs = 0; cs < K::CPW; ++cs) {
      const int c = w + K::NW * cs;
      if (c >= nc) continue;
#pragma unroll
      for (int t = 0; t < K::LSLOT; ++t) {
        const int r = lane + 32 * t;
        if (r >= K::RM) {
          const long long row = r0 + r;
          double v = 0.0;
          if (r < K::LROWS && row < n) v = __ldcg(col[cs] + row);
          x[cs][t] = c < count ? v * rn[cs] : v;
        }
      }
    }
    qr_cols<K>(x, K::LROWS, nc, sh);
  }
  store_R<K>(x, p.Rbuf + (long long)blockIdx.x * K::RM * K::RM, nc);
}

// merge FAN R factors per CTA; the single-CTA last level also solves
template <class K>
BSP_DEV void tsqr_merge(const KryArgs& p, const double* Rin, int nin, double* Rout) {
  DevState* st = p.st;
  if (st->done || st->kry_count == 0) return;
  __shared__ QRShared<K> sh;
  const int count = min(st->kry_count, K::RM - 1);
  const int nc = count + 1;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b0 = blockIdx.x * K::FAN;
  const int nb = min(K::FAN, nin - b0);
  double x[K::CPW][K::MSLOT];
#pragma unroll
  for (int cs = 0; cs < K::CPW; ++cs) {
    const int c = w + K::NW * cs;
#pragma unroll
    for (int t = 0; t < K::MSLOT; ++t) {
      const int r = lane + 32 * t;
      const int blk = r / K::RM, ri = r - blk * K::RM;
      double v = 0.0;
      if (r < K::MROWS && blk < nb && ri < nc && c < nc)
        v = __ldcg(Rin + (long long)(b0 + blk) * K::RM * K::RM + ri * K::RM + c);
      x[cs][t] = v;
    }
  }
  qr_cols<K>(x, K::MROWS, nc, sh);
  if (gridDim.x > 1 || p.no_solve) {
    store_R<K>(x, Rout + (long long)blockIdx.x * K::RM * K::RM, nc);
    return;
  }
#pragma unroll
  for (int cs = 0; cs < K::CPW; ++cs) {
    const int c = w + K::NW * cs;
#pragma unroll
    for (int t = 0; t < K::MSLOT; ++t) {
      const int r = lane + 32 * t;
      if (r < K::RM && c < K::RM) sh.R[r * K::LDS + c] = x[cs][t];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // rank cut |R_ii| <= 1e-13 |R_00| on the basis columns (solvers.py:212-214)
    const double* S = sh.R;
    const double d0 = fabs(S[0]);
    int rank = count;
    for (int i = 0; i < count; ++i) {
      if (fabs(S[i * K::LDS + i]) <= 1e-13 * d0) {
        rank = i;
        break;
      }
    }
    if (p.npow_req > count && st->kry_count == count && rank == count) {
      // the reference's rank cut lies beyond the formed powers: its answer
      // would need more columns than this TSQR holds -> stop, loudly
      st->kry_trunc = 1;
      st->done = 4;
    }
    double c[K::RM];
    for (int i = 0; i < K::RM; ++i) c[i] = 0.0;
    for (int i = rank - 1; i >= 0; --i) {  // dtrtrs on R[:rank,:rank]
      double s = S[i * K::LDS + count];
      for (int k = i + 1; k < rank; ++k) s -= S[i * K::LDS + k] * c[k];
      c[i] = s / S[i * K::LDS + i];
    }
    for (int i = 0; i < count; ++i) st->coef[i] = c[i] / st->norms[i + 1] / st->norms[i];
    st->kry_rank = rank;
    if (p.coef_out)
      for (int i = 0; i < count; ++i) p.coef_out[i] = c[i];
  }
}

}  // namespace

__global__ void __launch_bounds__(Narrow::NT) k_tsqr_leaf(KryArgs p) { tsqr_leaf<Narrow>(p); }
__global__ void __launch_bounds__(NarrowL::NT) k_tsqr_leaf_l(KryArgs p) { tsqr_leaf<NarrowL>(p); }
__global__ void __launch_bounds__(Narrow::NT) k_tsqr_merge(KryArgs p, const double* Rin, int nin,
                                                          double* Rout) {
  tsqr_merge<Narrow>(p, Rin, nin, Rout);
}
__global__ void __launch_bounds__(Wide::NT) k_tsqr_leaf_wide(KryArgs p) { tsqr_leaf<Wide>(p); }
__global__ void __launch_bounds__(Wide::NT) k_tsqr_merge_wide(KryArgs p, const double* Rin,
                                                             int nin, double* Rout) {
  tsqr_merge<Wide>(p, Rin, nin, Rout);
}

// u_next = u - beta * sum_i coef_i q_i   (solvers.py:255 + 280)
__global__ void __launch_bounds__(256) k_kry_combine(KryArgs p) {
  DevState* st = p.st;
  if (st->done) return;
  const int count = min(st->kry_count, kTsqrMaxCols - 1);
  __shared__ double coef[kTsqrMaxCols];
  if (threadIdx.x < kTsqrMaxCols) coef[threadIdx.x] = threadIdx.x < count ? st->coef[threadIdx.x] : 0.0;
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
int tsqr_threads() { return Narrow::NT; }
cudaError_t tsqr_prepare() { return cudaSuccess; }
int tsqr_max_cols() { return Narrow::RM; }
int tsqr_fan_in() { return Narrow::FAN; }
int tsqr_leaves(long long n) { return tsqr_leaves(n, Narrow::RM); }

static bool wide(int nc) { return nc > Narrow::RM; }
int tsqr_rdim(int nc) { return wide(nc) ? Wide::RM : Narrow::RM; }
int tsqr_fan_in(int nc) { return wide(nc) ? Wide::FAN : Narrow::FAN; }
int tsqr_leaves(long long n, int nc) {
  const int ch = wide(nc) ? Wide::CH : (n > kLargeLeafN ? NarrowL::CH : Narrow::CH);
  const long long chunks = (n + ch - 1) / ch;
  return (int)(chunks < 2048 ? chunks : 2048);
}
cudaError_t launch_tsqr_leaf(int nc, int blocks, const KryArgs& ka, cudaStream_t s) {
  if (wide(nc))
    k_tsqr_leaf_wide<<<blocks, Wide::NT, 0, s>>>(ka);
  else if (ka.n > kLargeLeafN)
    k_tsqr_leaf_l<<<blocks, NarrowL::NT, 0, s>>>(ka);
  else
    k_tsqr_leaf<<<blocks, Narrow::NT, 0, s>>>(ka);
  return cudaGetLastError();
}
cudaError_t launch_tsqr_merge(int nc, int nout, const KryArgs& ka, const double* rin, int nin,
                              double* rout, cudaStream_t s) {
  if (wide(nc))
    k_tsqr_merge_wide<<<nout, Wide::NT, 0, s>>>(ka, rin, nin, rout);
  else
    k_tsqr_merge<<<nout, Narrow::NT, 0, s>>>(ka, rin, nin, rout);
  return cudaGetLastError();
}

}  // namespace bsp
