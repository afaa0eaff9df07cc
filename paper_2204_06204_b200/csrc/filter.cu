// Separable Gaussian density filter C and its exact adjoint C^T.
// Restates reference filtering.py:46-55 (apply_filter) and filtering.py:58-72
// (apply_filter_adjoint), with the truncate-and-renormalise boundary masses of
// filtering.py:38-43 computed in-kernel.  The activation a = v_phys^eta of
// solvers.py:443 is fused into the forward pass.
//
// B200 mapping (v2, row streaming): a CTA of 128 threads owns a strip of
// kStrip = 256 columns (2 per thread, 16-byte cp.async) and walks a chunk of
// rows top to bottom.  Input rows stream through an 8-stage shared-memory ring,
// so 7 rows (56 KB per SM at 8 CTAs) are in flight to cover HBM latency.  The
// y-direction pass keeps each column's last 2r+1 values in registers, so it
// needs no shared memory.  The x-direction pass reads neighbouring columns from
// shared memory, and the strip emits 256 - 2r columns.  HBM traffic is the
// algorithmic one: the input once (+2r halo rows per chunk, from L2) and the
// outputs once.  Boundary masses are O(1): prefix sums of the taps.
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "filter.cuh"
#include "highlevel.cuh"
#include "hl_device.cuh"
#include "solver_state.cuh"

namespace bsp {

namespace {
constexpr int kThreads = 128;
constexpr int kStrip = 2 * kThreads;  // columns loaded per CTA
constexpr int kStages = 8;            // power of two
constexpr int kTargetCtas = 148 * 16;

BSP_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

BSP_DEV void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
BSP_DEV void cp_wait_stages() { asm volatile("cp.async.wait_group %0;\n" ::"n"(kStages - 2)); }

BSP_DEV double tap_cum(const FilterTaps& w, int k) {
  return w.size <= kMaxTaps ? w.cum[k] : w.dw[w.size + k];
}

BSP_DEV double axis_mass(const FilterTaps& w, int i, int len) {
  // kernel mass of the in-range taps at index i (correlate1d of ones, mode
  // constant, filtering.py:38-43): taps k with 0 <= i+k-r < len
  const int k0 = max(0, w.r - i);
  const int k1 = min(w.size, len - i + w.r);
  return tap_cum(w, k1) - tap_cum(w, k0);
}

BSP_DEV double spow(double x, double e) { return act_pow(x, e); }

// Stage loader: this thread's two columns (gx, gx+1) of input row yy into the
// ring slot; out-of-grid rows / columns are zero (mode constant padding).
struct Loader {
  const double* in;
  int nx, ny, gx;
  bool lo_in, hi_in;
  uint32_t slot0;  // shared address of this thread's pair in stage 0

  BSP_DEV void issue(int yy, int stage) const {
    const uint32_t d = slot0 + (uint32_t)(stage * kStrip * 8);
    const bool row_in = yy >= 0 && yy < ny;
    const double* base = in + (long long)(row_in ? yy : 0) * nx;
    if (row_in && lo_in && hi_in && ((reinterpret_cast<uintptr_t>(base + gx) & 15) == 0)) {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(base + gx));
    } else {
      const bool a = row_in && lo_in, b = row_in && hi_in;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d),
                   "l"(a ? base + gx : in), "r"(a ? 8 : 0));
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d + 8),
                   "l"(b ? base + gx + 1 : in), "r"(b ? 8 : 0));
    }
  }
};

// Strip geometry: ra = r rounded up to even keeps every pair 16-byte aligned
// (even nx); strip sx loads global columns x0 .. x0+255 (x0 = sx*ow - ra) and
// emits strip columns [ra, ra + ow), ow = 256 - 2 ra.
__host__ __device__ inline int strip_ra(int r) { return (r + 1) & ~1; }
__host__ __device__ inline int strip_ow(int r) { return kStrip - 2 * strip_ra(r); }
BSP_DEV int strip_x0(int sx, int r) { return sx * strip_ow(r) - strip_ra(r); }

template <int NW>
BSP_DEV void push(double (&ring)[NW], double x) {
#pragma unroll
  for (int k = 0; k < NW - 1; ++k) ring[k] = ring[k + 1];
  ring[NW - 1] = x;
}

// x pass at strip columns c0, c0+1 from a shared row: sum_k w_k row[c + k - r]
template <int NW>
BSP_DEV void xpass(const double* row, const double* wl, int r, int c0, double& a, double& b) {
  a = 0.0;
  b = 0.0;
  if (NW == 7 && c0 >= 4 && c0 + 5 < kStrip) {
    // radius 3, interior: five 16-byte loads cover columns c0-4 .. c0+5
    // (conflict-free LDS.128 across the warp) instead of 14 8-byte loads
    double v[10];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const double2 t = *reinterpret_cast<const double2*>(row + c0 - 4 + 2 * q);
      v[2 * q] = t.x;
      v[2 * q + 1] = t.y;
    }
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      a += wl[k] * v[k + 1];  // column c0 + k - 3
      b += wl[k] * v[k + 2];  // column c0 + 1 + k - 3
    }
    return;
  }
  if (c0 >= r && c0 + 1 < kStrip - r) {
#pragma unroll
    for (int k = 0; k < NW; ++k)
      if (k < 2 * r + 1) {
        a += wl[k] * row[c0 + k - r];
        b += wl[k] * row[c0 + 1 + k - r];
      }
  } else {
#pragma unroll
    for (int k = 0; k < NW; ++k)
      if (k < 2 * r + 1) {
        const int ca = c0 + k - r, cb = c0 + 1 + k - r;
        if (ca >= 0 && ca < kStrip) a += wl[k] * row[ca];
        if (cb >= 0 && cb < kStrip) b += wl[k] * row[cb];
      }
  }
}

// y pass: the register window holds rows yout - r .. yout + r in its last slots
template <int NW>
BSP_DEV double ypass(const double (&ring)[NW], const double* wl, int r) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < NW; ++k)
    if (k < 2 * r + 1) s += wl[k] * ring[NW - (2 * r + 1) + k];
  return s;
}
}  // namespace

int filter_rows_per_chunk(int nx, int ny) {
  const long long strips = (nx + strip_ow(3) - 1) / strip_ow(3);
  long long rc = ((long long)ny * strips + kTargetCtas - 1) / kTargetCtas;
  static const int min_rc = [] {
    const char* e = getenv("BSP_MIN_CHUNK");
    return e ? atoi(e) : 2;  // small grids: more CTAs beat the halo re-reads (r01: C2 -8%)
  }();
  if (rc < min_rc) rc = min_rc;
  if (rc > ny) rc = ny;
  return (int)rc;
}

dim3 filter_grid(int nx, int ny, int r) {
  const int ow = strip_ow(r);
  const int rc = filter_rows_per_chunk(nx, ny);
  return dim3((nx + ow - 1) / ow, (ny + rc - 1) / rc);
}

dim3 filter_grid_max(int nx, int ny) { return filter_grid(nx, ny, kMaxTaps / 2); }

size_t filter_smem_bytes(int) { return sizeof(double) * (size_t)(kStages + 2) * kStrip; }

// Forward: rows stream in; the x pass runs from shared memory as a row lands,
// the y pass from the register window; input row yin finalises row yin - r.
template <int R>
__global__ void __launch_bounds__(kThreads) k_filter_fwd_t(FilterArgs p) {
  pdl_begin();
  if (p.gate0 && *p.gate0) return;
  extern __shared__ __align__(16) double sm[];
  constexpr int NW = 2 * (R > 0 ? R : kMaxTaps / 2) + 1;
  const int r = R > 0 ? R : p.w.r;
  const int nx = p.nx, ny = p.ny;
  const int c0 = 2 * threadIdx.x;
  const int gx = strip_x0(blockIdx.x, r) + c0;
  const int y0 = blockIdx.y * p.rc, y1 = min(ny, y0 + p.rc);
  const int yin0 = y0 - r, nrows = y1 - y0 + 2 * r;
  Loader ld{p.in, nx, ny, gx, gx >= 0 && gx < nx, gx + 1 >= 0 && gx + 1 < nx,
            smem_u32(sm) + (uint32_t)c0 * 8};
  const int ra = strip_ra(r);
  const bool emit_lo = c0 >= ra && c0 < kStrip - ra && ld.lo_in;
  const bool emit_hi = c0 + 1 >= ra && c0 + 1 < kStrip - ra && ld.hi_in;
  const double isx_lo = emit_lo ? 1.0 / axis_mass(p.w, gx, nx) : 0.0;
  const double isx_hi = emit_hi ? 1.0 / axis_mass(p.w, gx + 1, nx) : 0.0;
  const double* wl = p.w.w;  // taps stay in the kernel-parameter bank
  // interior rows have the full kernel mass: one division per thread, not per row
  const double isy_in = 1.0 / (p.w.cum[p.w.size] - p.w.cum[0]);
  double ringA[NW], ringB[NW];
#pragma unroll
  for (int k = 0; k < NW; ++k) {
    ringA[k] = 0.0;
    ringB[k] = 0.0;
  }
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nrows) ld.issue(yin0 + s, s);
    cp_commit();
  }
  for (int i = 0; i < nrows; ++i) {
    const int yin = yin0 + i;
    cp_wait_stages();
    __syncthreads();  // row yin visible to all; stage (i-1) free for the refill
    if (i + kStages - 1 < nrows) ld.issue(yin + kStages - 1, (i + kStages - 1) & (kStages - 1));
    cp_commit();
    const double* row = sm + (i & (kStages - 1)) * kStrip;
    double mA, mB;
    xpass<NW>(row, wl, r, c0, mA, mB);
    push(ringA, mA * isx_lo);
    push(ringB, mB * isx_hi);
    const int yout = yin - r;
    if (yout < y0) continue;
    const int gyo = yout + p.gy0;
    const double isy = (gyo >= r && gyo < p.gny - r) ? isy_in : 1.0 / axis_mass(p.w, gyo, p.gny);
    const long long e = (long long)yout * nx + gx;
    const double vpA = ypass(ringA, wl, r) * isy, vpB = ypass(ringB, wl, r) * isy;
    if (emit_lo && emit_hi && ((e & 1) == 0)) {
      __stcs(reinterpret_cast<double2*>(p.out + e), make_double2(vpA, vpB));
      if (p.act)
        __stcs(reinterpret_cast<double2*>(p.act + e),
               make_double2(spow(vpA, p.eta), spow(vpB, p.eta)));
    } else {
      if (emit_lo) {
        p.out[e] = vpA;
        if (p.act) p.act[e] = spow(vpA, p.eta);
      }
      if (emit_hi) {
        p.out[e + 1] = vpB;
        if (p.act) p.act[e + 1] = spow(vpB, p.eta);
      }
    }
  }
  asm volatile("cp.async.wait_all;\n" ::);
  pdl_trigger();
}

// Adjoint: t = s / sy streams into the register window (y pass first); row
// yout's y sum / sx goes to a double-buffered shared row, then the x pass.
template <int R>
__global__ void __launch_bounds__(kThreads) k_filter_adj_t(FilterArgs p) {
  pdl_begin();
  if (p.gate0 && *p.gate0) return;
  extern __shared__ __align__(16) double sm[];
  constexpr int NW = 2 * (R > 0 ? R : kMaxTaps / 2) + 1;
  const int r = R > 0 ? R : p.w.r;
  const int nx = p.nx, ny = p.ny;
  const int c0 = 2 * threadIdx.x;
  const int gx = strip_x0(blockIdx.x, r) + c0;
  const int y0 = blockIdx.y * p.rc, y1 = min(ny, y0 + p.rc);
  const int yin0 = y0 - r, nrows = y1 - y0 + 2 * r;
  double* mrow = sm + kStages * kStrip;  // 2 x kStrip
  Loader ld{p.in, nx, ny, gx, gx >= 0 && gx < nx, gx + 1 >= 0 && gx + 1 < nx,
            smem_u32(sm) + (uint32_t)c0 * 8};
  const int ra = strip_ra(r);
  const bool emit_lo = c0 >= ra && c0 < kStrip - ra && ld.lo_in;
  const bool emit_hi = c0 + 1 >= ra && c0 + 1 < kStrip - ra && ld.hi_in;
  const double isx_lo = ld.lo_in ? 1.0 / axis_mass(p.w, gx, nx) : 0.0;
  const double isx_hi = ld.hi_in ? 1.0 / axis_mass(p.w, gx + 1, nx) : 0.0;
  const double* wl = p.w.w;  // taps stay in the kernel-parameter bank
  // interior rows have the full kernel mass: one division per thread, not per row
  const double isy_in = 1.0 / (p.w.cum[p.w.size] - p.w.cum[0]);
  double ringA[NW], ringB[NW];
#pragma unroll
  for (int k = 0; k < NW; ++k) {
    ringA[k] = 0.0;
    ringB[k] = 0.0;
  }
  double gs = 0.0;
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nrows) ld.issue(yin0 + s, s);
    cp_commit();
  }
  int parity = 0;
  for (int i = 0; i < nrows; ++i) {
    const int yin = yin0 + i;
    cp_wait_stages();
    __syncthreads();  // (a) input row ready; the refilled stage and this mrow buffer are free
    if (i + kStages - 1 < nrows) ld.issue(yin + kStages - 1, (i + kStages - 1) & (kStages - 1));
    cp_commit();
    const double* row = sm + (i & (kStages - 1)) * kStrip;
    const bool yrow = yin >= 0 && yin < ny;
    const int gyi = yin + p.gy0;
    const double isy =
        !yrow ? 0.0 : ((gyi >= r && gyi < p.gny - r) ? isy_in : 1.0 / axis_mass(p.w, gyi, p.gny));
    const double2 in2 = *reinterpret_cast<const double2*>(row + c0);
    push(ringA, in2.x * isy);
    push(ringB, in2.y * isy);
    const int yout = yin - r;
    if (yout < y0) continue;  // uniform across the CTA
    double* mr = mrow + parity * kStrip;
    parity ^= 1;
    *reinterpret_cast<double2*>(mr + c0) =
        make_double2(ypass(ringA, wl, r) * isx_lo, ypass(ringB, wl, r) * isx_hi);
    __syncthreads();  // (b) the y-summed row is complete
    double oA, oB;
    xpass<NW>(mr, wl, r, c0, oA, oB);
    const long long e = (long long)yout * nx + gx;
    const bool red_row = p.st && yout >= p.red_y0 && yout < p.red_y1;
    if (emit_lo && emit_hi && ((e & 1) == 0))
      __stcs(reinterpret_cast<double2*>(p.out + e), make_double2(oA, oB));
    else {
      if (emit_lo) p.out[e] = oA;
      if (emit_hi) p.out[e + 1] = oB;
    }
    if (red_row) {
      if (emit_lo && (!p.active || p.active[e])) gs += oA;
      if (emit_hi && (!p.active || p.active[e + 1])) gs += oB;
    }
  }
  asm volatile("cp.async.wait_all;\n" ::);
  pdl_trigger();
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

// ---------------------------------------------------------------------------
// Radius-3 kernels (filter size 7, the reference default FilterSpec(7, 1.5)),
// 4 columns per thread: a CTA loads a 512-column strip and emits 504.  The
// y window is a rotating register ring indexed by the row phase (the row loop
// is unrolled by 7), so no register moves per row; one x pass of 6 LDS.128
// yields 4 outputs.  Same per-output arithmetic (FMA order, mass scalings) as
// k_filter_fwd_t / k_filter_adj_t.
namespace {
constexpr int kRa4 = 4;  // r = 3 rounded up to keep 16-byte alignment
template <int W> constexpr int strip_w() { return W * kThreads; }
template <int W> constexpr int ow_w() { return W * kThreads - 2 * kRa4; }

template <int W>
struct Loader4 {
  static constexpr int kStrip4 = W * kThreads;
  const double* in;
  int nx, ny, gx;
  uint32_t slot0;
  // this thread's columns lie in the grid and every row's pair is 16-byte
  // aligned (even nx, aligned array): per row only the row test remains
  bool fast;
  // rows are issued in order from y_first: a running source pointer instead
  // of a 64-bit row product per row
  const double* cur;

  BSP_DEV Loader4(const double* in_, int nx_, int ny_, int gx_, uint32_t slot0_, int y_first)
      : in(in_), nx(nx_), ny(ny_), gx(gx_), slot0(slot0_),
        fast(gx_ >= 0 && gx_ + W - 1 < nx_ && (nx_ & 1) == 0 &&
             ((reinterpret_cast<uintptr_t>(in_ + gx_) & 15) == 0)),
        cur(in_ + (long long)y_first * nx_ + gx_) {}

  BSP_DEV void issue(int yy, int stage) {
    const uint32_t d = slot0 + (uint32_t)(stage * kStrip4 * 8);
    const bool row_in = yy >= 0 && yy < ny;
    const double* src = cur;  // row yy, column gx
    cur += nx;
    if (row_in && fast) {
#pragma unroll
      for (int q = 0; q < W; q += 2)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d + 8 * q), "l"(src + q));
    } else {
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const bool v = row_in && gx + j >= 0 && gx + j < nx;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d + 8 * j),
                     "l"(v ? src + j : in), "r"(v ? 8 : 0));
      }
    }
  }
};

// W outputs at strip columns c0..c0+W-1 (4 <= c0, c0 + W + 3 < strip)
template <int W>
BSP_DEV void xpass4(const double* row, const double* wl, int c0, double (&o)[W]) {
  double v[W + 8];
#pragma unroll
  for (int q = 0; q < (W + 8) / 2; ++q) {
    const double2 t = *reinterpret_cast<const double2*>(row + c0 - 4 + 2 * q);
    v[2 * q] = t.x;
    v[2 * q + 1] = t.y;
  }
#pragma unroll
  for (int j = 0; j < W; ++j) {
    double a = 0.0;
#pragma unroll
    for (int k = 0; k < 7; ++k) a += wl[k] * v[j + k + 1];  // column c0 + j + k - 3
    o[j] = a;
  }
}

// y sum over the ring (slot ph holds the newest row): oldest first
template <int PH>
BSP_DEV double ysum7(const double (&ring)[7], const double* wl) {
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 7; ++k) s += wl[k] * ring[(PH + 1 + k) % 7];
  return s;
}

template <int W>
BSP_DEV void store4(double* out, long long e, const double (&o)[W], const bool (&emit)[W],
                    bool all) {
  if (all && ((e & 1) == 0)) {
#pragma unroll
    for (int q = 0; q < W; q += 2)
      __stcs(reinterpret_cast<double2*>(out + e + q), make_double2(o[q], o[q + 1]));
  } else {
#pragma unroll
    for (int j = 0; j < W; ++j)
      if (emit[j]) out[e + j] = o[j];
  }
}
}  // namespace

int filter4_rows_per_chunk(int nx, int ny, int ow) {
  const long long strips = (nx + ow - 1) / ow;
  long long rc = ((long long)ny * strips + kTargetCtas - 1) / kTargetCtas;
  static const int min_rc = [] {
    const char* e = getenv("BSP_MIN_CHUNK");
    return e ? atoi(e) : 2;
  }();
  if (rc < min_rc) rc = min_rc;
  if (rc > ny) rc = ny;
  return (int)rc;
}

// 0: the generic kernels, 2 or 4: columns per thread of the radius-3 kernels
static int filter4_width() {
  static const int w = [] {
    const char* e = getenv("BSP_FILTER4");
    return e ? atoi(e) : 2;
  }();
  return w;
}

template <int W>
__global__ void __launch_bounds__(kThreads) k_filter_fwd4(FilterArgs p) {
  constexpr int kW4 = W, kStrip4 = strip_w<W>(), kOw4 = ow_w<W>();
  pdl_begin();
  if (p.gate0 && *p.gate0) return;
  extern __shared__ __align__(16) double sm[];
  const int nx = p.nx, ny = p.ny;
  const int c0 = kW4 * threadIdx.x;
  const int gx = blockIdx.x * kOw4 - kRa4 + c0;
  const int y0 = blockIdx.y * p.rc, y1 = min(ny, y0 + p.rc);
  const int yin0 = y0 - 3, nrows = y1 - y0 + 6;
  Loader4<W> ld{p.in, nx, ny, gx, smem_u32(sm) + (uint32_t)c0 * 8, yin0};
  const bool inner = c0 >= kRa4 && c0 < kStrip4 - kRa4;  // whole group inside the emitted band
  bool emit[kW4];
  double isx[kW4];
  bool all = inner;
#pragma unroll
  for (int j = 0; j < kW4; ++j) {
    emit[j] = inner && gx + j >= 0 && gx + j < nx;
    all = all && emit[j];
    isx[j] = emit[j] ? 1.0 / axis_mass(p.w, gx + j, nx) : 0.0;
  }
  const double* wl = p.w.w;
  const double isy_in = 1.0 / (p.w.cum[p.w.size] - p.w.cum[0]);
  double ring[kW4][7];
#pragma unroll
  for (int j = 0; j < kW4; ++j)
#pragma unroll
    for (int k = 0; k < 7; ++k) ring[j][k] = 0.0;
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nrows) ld.issue(yin0 + s, s);
    cp_commit();
  }
  auto step = [&](int i, auto ph_c) {
    constexpr int PH = decltype(ph_c)::value;
    const int yin = yin0 + i;
    cp_wait_stages();
    __syncthreads();  // row yin visible to all; stage (i-1) free for the refill
    if (i + kStages - 1 < nrows) ld.issue(yin + kStages - 1, (i + kStages - 1) & (kStages - 1));
    cp_commit();
    if (!inner) return;
    const double* row = sm + (i & (kStages - 1)) * kStrip4;
    double m[kW4];
    xpass4(row, wl, c0, m);
#pragma unroll
    for (int j = 0; j < kW4; ++j) ring[j][PH] = m[j] * isx[j];
    const int yout = yin - 3;
    if (yout < y0) return;
    const int gyo = yout + p.gy0;
    const double isy = (gyo >= 3 && gyo < p.gny - 3) ? isy_in : 1.0 / axis_mass(p.w, gyo, p.gny);
    const long long e = (long long)yout * nx + gx;
    double vp[kW4];
#pragma unroll
    for (int j = 0; j < kW4; ++j) vp[j] = ysum7<PH>(ring[j], wl) * isy;
    store4(p.out, e, vp, emit, all);
    if (p.act) {
      double a[kW4];
#pragma unroll
      for (int j = 0; j < kW4; ++j) a[j] = spow(vp[j], p.eta);
      store4(p.act, e, a, emit, all);
    }
  };
  for (int i0 = 0; i0 < nrows; i0 += 7) {
    step(i0, std::integral_constant<int, 0>{});
    if (i0 + 1 < nrows) step(i0 + 1, std::integral_constant<int, 1>{});
    if (i0 + 2 < nrows) step(i0 + 2, std::integral_constant<int, 2>{});
    if (i0 + 3 < nrows) step(i0 + 3, std::integral_constant<int, 3>{});
    if (i0 + 4 < nrows) step(i0 + 4, std::integral_constant<int, 4>{});
    if (i0 + 5 < nrows) step(i0 + 5, std::integral_constant<int, 5>{});
    if (i0 + 6 < nrows) step(i0 + 6, std::integral_constant<int, 6>{});
  }
  asm volatile("cp.async.wait_all;\n" ::);
  pdl_trigger();
}

template <int W>
__global__ void __launch_bounds__(kThreads) k_filter_adj4(FilterArgs p) {
  constexpr int kW4 = W, kStrip4 = strip_w<W>(), kOw4 = ow_w<W>();
  pdl_begin();
  if (p.gate0 && *p.gate0) return;
  extern __shared__ __align__(16) double sm[];
  const int nx = p.nx, ny = p.ny;
  const int c0 = kW4 * threadIdx.x;
  const int gx = blockIdx.x * kOw4 - kRa4 + c0;
  const int y0 = blockIdx.y * p.rc, y1 = min(ny, y0 + p.rc);
  const int yin0 = y0 - 3, nrows = y1 - y0 + 6;
  double* mrow = sm + kStages * kStrip4;  // 2 x kStrip4
  Loader4<W> ld{p.in, nx, ny, gx, smem_u32(sm) + (uint32_t)c0 * 8, yin0};
  const bool inner = c0 >= kRa4 && c0 < kStrip4 - kRa4;
  bool emit[kW4];
  double isx[kW4];
  bool all = inner;
#pragma unroll
  for (int j = 0; j < kW4; ++j) {
    const bool in_grid = gx + j >= 0 && gx + j < nx;
    emit[j] = inner && in_grid;
    all = all && emit[j];
    isx[j] = in_grid ? 1.0 / axis_mass(p.w, gx + j, nx) : 0.0;
  }
  const double* wl = p.w.w;
  const double isy_in = 1.0 / (p.w.cum[p.w.size] - p.w.cum[0]);
  double ring[kW4][7];
#pragma unroll
  for (int j = 0; j < kW4; ++j)
#pragma unroll
    for (int k = 0; k < 7; ++k) ring[j][k] = 0.0;
  double gs = 0.0;
  const bool do_red = p.st != nullptr;
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nrows) ld.issue(yin0 + s, s);
    cp_commit();
  }
  cp_wait_stages();
  __syncthreads();  // row 0 visible
  int parity = 0;
  // ONE barrier per row: the barrier after the y pass (the summed row is
  // complete) also publishes the NEXT input row -- each thread waits for its
  // own copies of it first -- and retires the row just read, so the refill at
  // the top of the next step and the other half of the double-buffered mrow
  // are free (their last readers ran before this barrier).
  auto step = [&](int i, auto ph_c) {
    constexpr int PH = decltype(ph_c)::value;
    const int yin = yin0 + i;
    // stage (i-1) was retired by the previous step's barrier
    if (i + kStages - 1 < nrows) ld.issue(yin + kStages - 1, (i + kStages - 1) & (kStages - 1));
    cp_commit();
    const double* row = sm + (i & (kStages - 1)) * kStrip4;
    const bool yrow = yin >= 0 && yin < ny;
    const int gyi = yin + p.gy0;
    const double isy =
        !yrow ? 0.0 : ((gyi >= 3 && gyi < p.gny - 3) ? isy_in : 1.0 / axis_mass(p.w, gyi, p.gny));
#pragma unroll
    for (int q = 0; q < kW4; q += 2) {
      const double2 in2 = *reinterpret_cast<const double2*>(row + c0 + q);
      ring[q][PH] = in2.x * isy;
      ring[q + 1][PH] = in2.y * isy;
    }
    const int yout = yin - 3;
    const bool out_row = yout >= y0;  // uniform across the CTA
    double* mr = mrow + parity * kStrip4;
    if (out_row) {
#pragma unroll
      for (int q = 0; q < kW4; q += 2)
        *reinterpret_cast<double2*>(mr + c0 + q) =
            make_double2(ysum7<PH>(ring[q], wl) * isx[q], ysum7<PH>(ring[q + 1], wl) * isx[q + 1]);
    }
    cp_wait_stages();  // this thread's copies of row i+1 have landed
    __syncthreads();   // mrow complete, row i+1 visible, row i retired
    if (!out_row) return;
    parity ^= 1;
    if (!inner) return;
    double o[kW4];
    xpass4(mr, wl, c0, o);
    const long long e = (long long)yout * nx + gx;
    store4(p.out, e, o, emit, all);
    if (do_red && yout >= p.red_y0 && yout < p.red_y1) {
      if (p.active) {
#pragma unroll
        for (int j = 0; j < kW4; ++j)
          if (emit[j] && p.active[e + j]) gs += o[j];
      } else {
#pragma unroll
        for (int j = 0; j < kW4; ++j) gs += emit[j] ? o[j] : 0.0;  // + 0.0: bitwise the skip
      }
    }
  };
  for (int i0 = 0; i0 < nrows; i0 += 7) {
    step(i0, std::integral_constant<int, 0>{});
    if (i0 + 1 < nrows) step(i0 + 1, std::integral_constant<int, 1>{});
    if (i0 + 2 < nrows) step(i0 + 2, std::integral_constant<int, 2>{});
    if (i0 + 3 < nrows) step(i0 + 3, std::integral_constant<int, 3>{});
    if (i0 + 4 < nrows) step(i0 + 4, std::integral_constant<int, 4>{});
    if (i0 + 5 < nrows) step(i0 + 5, std::integral_constant<int, 5>{});
    if (i0 + 6 < nrows) step(i0 + 6, std::integral_constant<int, 6>{});
  }
  asm volatile("cp.async.wait_all;\n" ::);
  pdl_trigger();
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


// The adjoint filter fused with the high-level step (solvers.py:457, 462:
// g = C^T s, then v_next = P(v + alpha (g - mean g))): k_filter_adj4's row
// streaming, and for each finished row the box projection, the stores of
// v_next and the k_hl_write measurements (box sum, volume, interior count and
// sum, max |dv|, max w) with its last-block finalisation: one launch and the
// re-read of g less than the two kernels.  g is still stored (for a lambda
// search, which the last block runs itself on grids up to h.small_fix
// elements: no k_hl_fix launch).  The design rows stream through a second
// cp.async ring in the same commit groups (row yin - 3 with input row yin).
// Requires: no passive region; the mean projection's sum of g in st->gsum
// before the launch (the residual kernel's SF_SUM_SENS).
template <int W>
__global__ void __launch_bounds__(kThreads) k_hl_adj4(FilterArgs p, HLArgs h) {
  constexpr int kW4 = W, kStrip4 = strip_w<W>(), kOw4 = ow_w<W>();
  pdl_begin();
  if (h.st->done) return;
  extern __shared__ __align__(16) double sm[];
  const int nx = p.nx, ny = p.ny;
  const int c0 = kW4 * threadIdx.x;
  const int gx = blockIdx.x * kOw4 - kRa4 + c0;
  const int y0 = blockIdx.y * p.rc, y1 = min(ny, y0 + p.rc);
  const int yin0 = y0 - 3, nrows = y1 - y0 + 6;
  double* mrow = sm + kStages * kStrip4;  // 2 x kStrip4
  double* vring = mrow + 2 * kStrip4;     // kStages x kStrip4
  Loader4<W> ld{p.in, nx, ny, gx, smem_u32(sm) + (uint32_t)c0 * 8, yin0};
  Loader4<W> ldv{h.v, nx, ny, gx, smem_u32(vring) + (uint32_t)c0 * 8, yin0 - 3};
  const bool inner = c0 >= kRa4 && c0 < kStrip4 - kRa4;
  bool emit[kW4];
  double isx[kW4];
  bool all = inner;
#pragma unroll
  for (int j = 0; j < kW4; ++j) {
    const bool in_grid = gx + j >= 0 && gx + j < nx;
    emit[j] = inner && in_grid;
    all = all && emit[j];
    isx[j] = in_grid ? 1.0 / axis_mass(p.w, gx + j, nx) : 0.0;
  }
  const double* wl = p.w.w;
  const double isy_in = 1.0 / (p.w.cum[p.w.size] - p.w.cum[0]);
  double ring[kW4][7];
#pragma unroll
  for (int j = 0; j < kW4; ++j)
#pragma unroll
    for (int k = 0; k < 7; ++k) ring[j][k] = 0.0;
  const double alpha = step_alpha(h), mean = g_mean(h);
  const double lo = h.lo, hi = h.hi;
  const bool mp = h.mean_projection != 0;
  double bs = 0.0, vol = 0.0, nmid = 0.0, smid = 0.0, dv = 0.0, wmax = -INFINITY;
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nrows) {
      ld.issue(yin0 + s, s);
      ldv.issue(yin0 + s - 3, s);
    }
    cp_commit();
  }
  cp_wait_stages();
  __syncthreads();  // row 0 visible
  int parity = 0;
  auto step = [&](int i, auto ph_c) {
    constexpr int PH = decltype(ph_c)::value;
    const int yin = yin0 + i;
    if (i + kStages - 1 < nrows) {
      const int st = (i + kStages - 1) & (kStages - 1);
      ld.issue(yin + kStages - 1, st);
      ldv.issue(yin + kStages - 4, st);
    }
    cp_commit();
    const double* row = sm + (i & (kStages - 1)) * kStrip4;
    const bool yrow = yin >= 0 && yin < ny;
    const int gyi = yin + p.gy0;
    const double isy =
        !yrow ? 0.0 : ((gyi >= 3 && gyi < p.gny - 3) ? isy_in : 1.0 / axis_mass(p.w, gyi, p.gny));
#pragma unroll
    for (int q = 0; q < kW4; q += 2) {
      const double2 in2 = *reinterpret_cast<const double2*>(row + c0 + q);
      ring[q][PH] = in2.x * isy;
      ring[q + 1][PH] = in2.y * isy;
    }
    const int yout = yin - 3;
    const bool out_row = yout >= y0;  // uniform across the CTA
    double* mr = mrow + parity * kStrip4;
    if (out_row) {
#pragma unroll
      for (int q = 0; q < kW4; q += 2)
        *reinterpret_cast<double2*>(mr + c0 + q) =
            make_double2(ysum7<PH>(ring[q], wl) * isx[q], ysum7<PH>(ring[q + 1], wl) * isx[q + 1]);
    }
    cp_wait_stages();  // this thread's copies of row i+1 have landed
    __syncthreads();   // mrow complete, row i+1 visible, row i retired
    if (!out_row) return;
    parity ^= 1;
    if (!inner) return;
    double g[kW4];
    xpass4(mr, wl, c0, g);
    // design row yout: this thread's own columns of vring stage i
    const double* vr = vring + (i & (kStages - 1)) * kStrip4;
    double vv[kW4], out[kW4];
#pragma unroll
    for (int q = 0; q < kW4; q += 2) {
      const double2 t = *reinterpret_cast<const double2*>(vr + c0 + q);
      vv[q] = t.x;
      vv[q + 1] = t.y;
    }
#pragma unroll
    for (int j = 0; j < kW4; ++j) {  // k_hl_write's per-element step
      const double w = vv[j] + alpha * (mp ? g[j] - mean : g[j]);
      out[j] = clampd(w, lo, hi);
      if (emit[j]) {
        bs += out[j];
        wmax = nanmax(wmax, w);
        if (w > lo && w < hi) {
          nmid += 1.0;
          smid += w;
        }
        dv = nanmax(dv, fabs(out[j] - vv[j]));
        vol += vv[j];
      }
    }
    const long long e = (long long)yout * nx + gx;
    if (h.g) store4(const_cast<double*>(h.g), e, g, emit, all);
    store4(h.v_next, e, out, emit, all);
  };
  for (int i0 = 0; i0 < nrows; i0 += 7) {
    step(i0, std::integral_constant<int, 0>{});
    if (i0 + 1 < nrows) step(i0 + 1, std::integral_constant<int, 1>{});
    if (i0 + 2 < nrows) step(i0 + 2, std::integral_constant<int, 2>{});
    if (i0 + 3 < nrows) step(i0 + 3, std::integral_constant<int, 3>{});
    if (i0 + 4 < nrows) step(i0 + 4, std::integral_constant<int, 4>{});
    if (i0 + 5 < nrows) step(i0 + 5, std::integral_constant<int, 5>{});
    if (i0 + 6 < nrows) step(i0 + 6, std::integral_constant<int, 6>{});
  }
  asm volatile("cp.async.wait_all;\n" ::);
  pdl_trigger();
  __shared__ double tot[6];
  double v6[6] = {bs, vol, nmid, smid, dv, wmax};
  if (grid_reduce_nn<6, 4>(h.rb, v6, tot)) {  // last block, all its threads
    if (tot[0] > h.budget && h.E <= h.small_fix)
      block_lambda(h, tot, alpha, mean);  // g of every block is stored and fenced
    else if (threadIdx.x == 0)
      hl_write_hook(h, tot);
  }
}

// ---------------------------------------------------------------------------
// Any radius (FilterSpec.size > kMaxTaps): the reference's two passes as two
// kernels through the caller's scratch, taps from device memory.  One thread
// per output, grid-stride; reads along x are coalesced and the 2r+1 taps of
// neighbouring threads overlap in L1.  Forward: tmp = corr_x(in) / sx, then
// out = corr_y(tmp) / sy (+ activation).  Adjoint: tmp = corr_y(in / sy) / sx,
// then out = corr_x(tmp) (+ the mean projection's masked sum).
namespace {
constexpr int kWideThreads = 256;

__global__ void __launch_bounds__(kWideThreads) k_filter_wide_x(FilterArgs p, int adjoint) {
  if (p.gate0 && *p.gate0) return;
  const int nx = p.nx, ny = p.ny, r = p.w.r, sz = p.w.size;
  const double* w = p.w.dw;
  const double* src = adjoint ? p.w.tmp : p.in;
  double* dst = adjoint ? p.out : p.w.tmp;
  const long long E = (long long)nx * ny;
  double gs = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < E;
       e += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(e % nx), y = (int)(e / nx);
    const double* row = src + (long long)y * nx;
    double acc = 0.0;
    const int k0 = max(0, r - x), k1 = min(sz, nx - x + r);
    for (int k = k0; k < k1; ++k) acc += w[k] * row[x + k - r];
    if (adjoint) {
      dst[e] = acc;
      if (p.st && y >= p.red_y0 && y < p.red_y1 && (!p.active || p.active[e])) gs += acc;
    } else {
      dst[e] = acc * (1.0 / axis_mass(p.w, x, nx));
    }
  }
  if (adjoint && p.st) {
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

__global__ void __launch_bounds__(kWideThreads) k_filter_wide_y(FilterArgs p, int adjoint) {
  if (p.gate0 && *p.gate0) return;
  const int nx = p.nx, ny = p.ny, r = p.w.r, sz = p.w.size;
  const double* w = p.w.dw;
  const double* src = adjoint ? p.in : p.w.tmp;
  double* dst = adjoint ? p.w.tmp : p.out;
  const long long E = (long long)nx * ny;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < E;
       e += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(e % nx), y = (int)(e / nx);
    double acc = 0.0;
    const int k0 = max(0, r - y), k1 = min(sz, ny - y + r);
    for (int k = k0; k < k1; ++k) {
      const int yy = y + k - r;
      const double v = src[(long long)yy * nx + x];
      // adjoint: the input row is divided by its (global-row) mass first
      acc += w[k] * (adjoint ? v * (1.0 / axis_mass(p.w, yy + p.gy0, p.gny)) : v);
    }
    if (adjoint) {
      dst[e] = acc * (1.0 / axis_mass(p.w, x, nx));
    } else {
      const double vp = acc * (1.0 / axis_mass(p.w, y + p.gy0, p.gny));
      dst[e] = vp;
      if (p.act) p.act[e] = spow(vp, p.eta);
    }
  }
}
}  // namespace

static cudaError_t launch_filter_wide(const FilterArgs& fa, int adjoint, cudaStream_t s) {
  if (!fa.w.dw || !fa.w.tmp) return cudaErrorInvalidValue;
  const long long E = (long long)fa.nx * fa.ny;
  const unsigned nb = (unsigned)std::min<long long>((E + kWideThreads - 1) / kWideThreads, 1024);
  if (!adjoint) {
    launch_k(k_filter_wide_x, dim3(nb), dim3(kWideThreads), 0, s, fa, 0);
    return launch_k(k_filter_wide_y, dim3(nb), dim3(kWideThreads), 0, s, fa, 0);
  }
  launch_k(k_filter_wide_y, dim3(nb), dim3(kWideThreads), 0, s, fa, 1);
  return launch_k(k_filter_wide_x, dim3(nb), dim3(kWideThreads), 0, s, fa, 1);
}

// Fused up to 2^22 cells: there the iteration is launch-latency bound and one
// kernel less is the gain (C2 0.039 -> 0.037 ms/iter, C1 0.274 -> 0.270).
// Above, only on a forked graph branch (pfbto / cpfbto), where the fused
// kernel's 32E bytes instead of 40E leave bandwidth to the Jacobi step
// running beside it (C5 3.85 -> 3.77 ms/iter); on the multigrid chain it ran
// serially and lost (C4 7.57 -> 7.63).  BSP_HL_FUSE_MAX=<cells> overrides.
bool hl_adjoint_fusable(const FilterTaps& w, int nx, long long E, bool forked) {
  static const long long env_max = [] {
    const char* e = getenv("BSP_HL_FUSE_MAX");
    return e ? atoll(e) : -1ll;
  }();
  const bool size_ok = env_max >= 0 ? E <= env_max : (E <= (1ll << 22) || forked);
  return size_ok && w.size <= kMaxTaps && w.r == 3 && filter4_width() == 2 && nx % 2 == 0;
}

cudaError_t launch_hl_adjoint(const FilterTaps& w, const double* sens, const HLArgs& h,
                              cudaStream_t s) {
  FilterArgs fa{};
  fa.w = w;
  fa.nx = h.nx;
  fa.ny = h.ny;
  fa.in = sens;
  fa.gy0 = 0;
  fa.gny = h.ny;
  const int ow = ow_w<2>();
  // one output row per CTA on small grids: the 8-step row pipeline of a
  // 2-row chunk becomes 7 steps (C2 end to end 0.0327 -> 0.0305 ms).  Only
  // here: the chunking orders the stand-alone adjoint's sum of g, and moving
  // it moves chaotic (cpfbto) trajectories by rounding
  static const int min_rc = [] {
    const char* e = getenv("BSP_HL_MIN_CHUNK");
    return e ? atoi(e) : 1;
  }();
  const long long strips = (fa.nx + ow - 1) / ow;
  long long rc = ((long long)fa.ny * strips + kTargetCtas - 1) / kTargetCtas;
  fa.rc = (int)std::min<long long>(std::max<long long>(rc, min_rc), fa.ny);
  const dim3 grid((fa.nx + ow - 1) / ow, (fa.ny + fa.rc - 1) / fa.rc);
  const size_t sm = sizeof(double) * (size_t)(2 * kStages + 2) * 2 * kThreads;  // 36 KB
  return launch_k(k_hl_adj4<2>, grid, kThreads, sm, s, fa, h);
}

cudaError_t launch_filter_kernel(const FilterArgs& fa0, int adjoint, cudaStream_t s) {
  FilterArgs fa = fa0;
  if (fa.w.size > kMaxTaps) return launch_filter_wide(fa, adjoint, s);
  const int w4 = filter4_width();
  if (fa.w.r == 3 && (w4 == 2 || w4 == 4)) {
    const int ow = w4 == 4 ? ow_w<4>() : ow_w<2>();
    fa.rc = filter4_rows_per_chunk(fa.nx, fa.ny, ow);
    const dim3 grid((fa.nx + ow - 1) / ow, (fa.ny + fa.rc - 1) / fa.rc);
    const size_t sm = sizeof(double) * (size_t)(kStages + 2) * w4 * kThreads;  // 20 / 40 KB
    if (w4 == 4)
      return adjoint ? launch_k(k_filter_adj4<4>, grid, kThreads, sm, s, fa)
                     : launch_k(k_filter_fwd4<4>, grid, kThreads, sm, s, fa);
    return adjoint ? launch_k(k_filter_adj4<2>, grid, kThreads, sm, s, fa)
                   : launch_k(k_filter_fwd4<2>, grid, kThreads, sm, s, fa);
  }
  fa.rc = filter_rows_per_chunk(fa.nx, fa.ny);
  const dim3 grid = filter_grid(fa.nx, fa.ny, fa.w.r);
  const size_t sm = filter_smem_bytes(fa.w.r);  // 20 KB
  if (fa.w.r == 3)
    return adjoint ? launch_k(k_filter_adj_t<3>, grid, kThreads, sm, s, fa)
                   : launch_k(k_filter_fwd_t<3>, grid, kThreads, sm, s, fa);
  return adjoint ? launch_k(k_filter_adj_t<0>, grid, kThreads, sm, s, fa)
                 : launch_k(k_filter_fwd_t<0>, grid, kThreads, sm, s, fa);
}

}  // namespace bsp
