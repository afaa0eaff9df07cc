// C-ABI: grid residency and stream-ordered operator launches
// (include/bisimp_b200.h).  The outer loop lives in solver.cu.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "grid.cuh"
#include "highlevel.cuh"
#include "krylov.cuh"
#include "mg.cuh"
#include "misc.cuh"

using namespace bsp;

// ------------------------------------------------------------------ errors --
static thread_local std::string g_err;

namespace bsp {
int set_error(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int wave_blocks(const void* kernel, int threads) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find({kernel, dev});
  if (it != cache.end()) return it->second;
  int per = 1, nsm = 148;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, threads, 0) != cudaSuccess)
    per = 1;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaGetLastError();
  const int w = std::max(1, per) * nsm;
  cache[{kernel, dev}] = w;
  return w;
}

cudaError_t smem_optin(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;  // (kernel, device) already opted in
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({kernel, dev})) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({kernel, dev});
  return e;
}
}  // namespace bsp

#define FAIL(code, ...) ::bsp::set_error(code, __VA_ARGS__)

extern "C" const char* bsp_last_error(void) { return g_err.c_str(); }
extern "C" int bsp_version(void) { return 1; }

// -------------------------------------------------------------- helpers ----
namespace bsp {

bool& pdl_enabled() {
  static thread_local bool on = false;
  return on;
}

StiffArgs stiff_args(bsp_grid* g) {
  StiffArgs p{};
  p.g = g->view();
  p.rb = RedBuf{g->part, g->counter};
  p.R = g->R;
  p.red_y0 = 0;
  p.red_y1 = g->ny + 1;
  p.st = g->st;
  p.eta = 1.0;
  return p;
}

int normalize_config(const bsp_solver_config* in, bsp_solver_config& out) {
  if (!in) return FAIL(BSP_EINVAL, "null config");
  if (in->struct_size < BSP_SOLVER_CONFIG_MIN_SIZE || in->struct_size > sizeof(bsp_solver_config))
    return FAIL(BSP_EINVAL, "bsp_solver_config.struct_size %zu outside [%zu, %zu]",
                in->struct_size, (size_t)BSP_SOLVER_CONFIG_MIN_SIZE, sizeof(bsp_solver_config));
  bsp_solver_config c{};
  c.inner_steps = -1;
  c.mg_omega = 0.6;
  c.mg_nu = 2;
  c.mg_levels = 0;
  std::memcpy(&c, in, in->struct_size);
  if (c.inner_steps < 0)
    c.inner_steps = c.algorithm == BSP_ALGO_PCG_JACOBI ? 20 : c.algorithm == BSP_ALGO_MG_PCG ? 4 : 0;
  out = c;
  return BSP_OK;
}

int make_taps(const double* h_taps, int n, FilterTaps& w) {
  if (!h_taps) return FAIL(BSP_EINVAL, "null filter taps");
  if (n < 1 || n % 2 == 0) return FAIL(BSP_EINVAL, "kernel size must be odd and >= 1, got %d", n);
  w = FilterTaps{};
  w.size = n;
  w.r = n / 2;
  if (n <= kMaxTaps) {
    w.cum[0] = 0.0;
    for (int i = 0; i < n; ++i) {
      w.w[i] = h_taps[i];
      w.cum[i + 1] = w.cum[i] + h_taps[i];
    }
    return BSP_OK;
  }
  // wide filters: taps + prefix sums in device memory, interned per (device,
  // taps) for the life of the process (a few KB per distinct FilterSpec)
  static std::mutex mu;
  static std::map<std::pair<int, std::vector<double>>, double*> interned;
  int dev = 0;
  BSP_CU(cudaGetDevice(&dev));
  std::vector<double> key(h_taps, h_taps + n);
  std::lock_guard<std::mutex> lock(mu);
  auto it = interned.find({dev, key});
  if (it == interned.end()) {
    std::vector<double> buf(2 * n + 1);
    buf[n] = 0.0;
    for (int i = 0; i < n; ++i) {
      buf[i] = h_taps[i];
      buf[n + i + 1] = buf[n + i] + h_taps[i];
    }
    double* d = nullptr;
    BSP_CU(cudaMalloc(&d, buf.size() * sizeof(double)));
    BSP_CU(cudaMemcpy(d, buf.data(), buf.size() * sizeof(double), cudaMemcpyHostToDevice));
    it = interned.emplace(std::make_pair(dev, key), d).first;
  }
  w.dw = it->second;
  return BSP_OK;
}

FilterArgs filter_args(const double* in, double* out, double* act, double eta, int nx, int ny,
                       const FilterTaps& w, const int* gate, DevState* st, const uint8_t* active,
                       RedBuf rb) {
  FilterArgs fa{};
  fa.st = st;
  fa.active = active;
  fa.rb = rb;
  fa.w = w;
  fa.nx = nx;
  fa.ny = ny;
  fa.in = in;
  fa.out = out;
  fa.act = act;
  fa.eta = eta;
  fa.gate0 = gate;
  fa.gy0 = 0;
  fa.gny = ny;
  fa.red_y0 = 0;
  fa.red_y1 = ny;
  fa.defer_out = nullptr;
  return fa;
}

int launch_filter_fa(const FilterArgs& fa, int adjoint, cudaStream_t s) {
  BSP_CU(launch_filter_kernel(fa, adjoint, s));
  return BSP_OK;
}

int launch_filter(const double* in, double* out, double* act, double eta, int nx, int ny,
                  const FilterTaps& w, int adjoint, const int* gate, cudaStream_t s,
                  DevState* st, const uint8_t* active, RedBuf rb) {
  return launch_filter_fa(filter_args(in, out, act, eta, nx, ny, w, gate, st, active, rb), adjoint,
                          s);
}

// a standalone launch: wide filters get a stream-ordered scratch of their own
int launch_filter_scratch(const double* in, double* out, double* act, double eta, int nx, int ny,
                          FilterTaps w, int adjoint, cudaStream_t s) {
  if (w.size <= kMaxTaps)
    return launch_filter(in, out, act, eta, nx, ny, w, adjoint, nullptr, s);
  BSP_CU(cudaMallocAsync(&w.tmp, (size_t)nx * ny * sizeof(double), s));
  const int rc = launch_filter(in, out, act, eta, nx, ny, w, adjoint, nullptr, s);
  cudaFreeAsync(w.tmp, s);
  return rc;
}

int ensure_wk(bsp_grid* g, size_t doubles) {
  if (doubles <= g->wk_cap) return BSP_OK;
  if (g->wk) cudaFree(g->wk);
  g->wk = nullptr;
  g->wk_cap = 0;
  cudaError_t e = cudaMalloc(&g->wk, doubles * sizeof(double));
  if (e != cudaSuccess)
    return FAIL(BSP_ENOMEM, "workspace of %zu doubles: %s", doubles, cudaGetErrorString(e));
  g->wk_cap = doubles;
  return BSP_OK;
}

int ensure_tsqr(bsp_grid* g) {
  if (g->Rbuf) return BSP_OK;
  // sized once for either TSQR width (captured graphs keep the pointer); two
  // halves: leaves in the first, tree levels ping-pong between the halves
  const int nw = kTsqrMaxCols, nn = tsqr_max_cols();
  const size_t need = 2ull * std::max<size_t>((size_t)tsqr_leaves(g->n, nw) * nw * nw,
                                              (size_t)tsqr_leaves(g->n, nn) * nn * nn);
  BSP_CU(cudaMalloc(&g->Rbuf, need * sizeof(double)));
  BSP_CU(tsqr_prepare());
  return BSP_OK;
}

}  // namespace bsp

static int strip_rows(long long warps_across, int ny, int nsm) {
  const long long target = (long long)nsm * 24;
  for (int cand : {32, 16, 8, 4})
    if (warps_across * ((ny + cand - 1) / cand) >= target) return cand;
  static const int min_r = [] {  // even (the TMA kernel stages two rows at a time)
    const char* e = getenv("BSP_MIN_STRIP");
    const int r = e ? std::max(2, atoi(e)) : 2;
    return r + (r & 1);
  }();
  return min_r;
}

static void choose_strips(bsp_grid* g) {
  // TMA kernel: 62 node columns per warp, 4 warps per CTA
  const long long W3 = (g->nx + 1 + 61) / 62;
  g->R3 = strip_rows(W3, g->ny, g->nsm);
  g->sgrid3 = dim3((unsigned)((W3 + 3) / 4), (unsigned)((g->ny + g->R3 - 1) / g->R3));
  const int W = (g->nx + 1 + 30) / 31;  // warps across the node columns
  const long long target = (long long)g->nsm * 24;
  int R = 2;
  for (int cand : {32, 16, 8, 4}) {
    if ((long long)W * ((g->ny + cand - 1) / cand) >= target) {
      R = cand;
      break;
    }
  }
  g->R = R;
  g->sgrid = dim3((W + 3) / 4, (g->ny + R - 1) / R);
}

// M = T ke T^T / 16 in the per-component Hadamard mode basis (common.cuh)
static void ke_modes(const double* ke, bsp_grid* g) {
  const double H[4][4] = {{1, 1, 1, 1}, {-1, 1, 1, -1}, {-1, -1, 1, 1}, {1, -1, 1, -1}};
  double T[8][8] = {};
  for (int c = 0; c < 2; ++c)
    for (int m = 0; m < 4; ++m)
      for (int i = 0; i < 4; ++i) T[c * 4 + m][2 * i + c] = H[m][i];
  double M[8][8];
  double kmax = 0.0;
  for (int i = 0; i < 64; ++i) kmax = std::max(kmax, std::fabs(ke[i]));
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) {
      double s = 0.0;
      for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) s += T[a][i] * ke[i * 8 + j] * T[b][j];
      M[a][b] = s / 16.0;
    }
  KeModes& km = g->km;
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) km.M[a * 8 + b] = M[a][b];
  const int keep[][2] = {{1, 1}, {1, 6}, {6, 1}, {6, 6}, {2, 2}, {2, 5}, {5, 2}, {5, 5}, {3, 3}, {7, 7}};
  bool iso = true;
  const double tol = 1e-13 * kmax;
  for (int a = 0; a < 8; ++a)
    for (int b = 0; b < 8; ++b) {
      bool k = false;
      for (auto& kp : keep) k |= (kp[0] == a && kp[1] == b);
      if (!k && std::fabs(M[a][b]) > tol) iso = false;
    }
  km.m11 = M[1][1]; km.m16 = M[1][6]; km.m66 = M[6][6];
  km.m22 = M[2][2]; km.m25 = M[2][5]; km.m55 = M[5][5];
  km.m33 = M[3][3]; km.m77 = M[7][7];
  km.iso = iso ? 1 : 0;
  g->generic = !iso;
  km.kdx = ke[0];
  km.kdy = ke[9];
  km.ikdx = 1.0 / km.kdx;
  km.ikdy = 1.0 / km.kdy;
  km.ikdx2 = km.ikdx * km.ikdx;
  km.ikdy2 = km.ikdy * km.ikdy;
  // diag(ke) must be the same at the 4 local nodes (true for any square Q4
  // element; quadrature rounding may differ in the last ulp)
  g->uniform_diag = true;
  for (int i = 0; i < 4; ++i) {
    if (std::fabs(ke[(2 * i) * 8 + 2 * i] - ke[0]) > 1e-13 * kmax) g->uniform_diag = false;
    if (std::fabs(ke[(2 * i + 1) * 8 + 2 * i + 1] - ke[9]) > 1e-13 * kmax) g->uniform_diag = false;
  }
}

// ------------------------------------------------------------------- grid ---
extern "C" int bsp_grid_destroy(bsp_grid* g) {
  if (!g) return BSP_OK;
  bsp::DeviceGuard dg_(g->device);
  if (g->mg) bsp_mg_destroy(g->mg);
  for (PcgWork*& w : g->pcg_ws)
    if (w) {
      pcg_free(*w);
      delete w;
      w = nullptr;
    }
  cudaFree(g->fixbits);
  cudaFree(g->fixrows);
  cudaFree(g->load);
  cudaFree(g->part);
  cudaFree(g->counter);
  cudaFree(g->st);
  cudaFree(g->red);
  cudaFree(g->hl_part);
  cudaFree(g->wk);
  cudaFree(g->Rbuf);
  if (g->hpin) cudaFreeHost(g->hpin);
  delete g;
  return BSP_OK;
}

namespace {
// Allocation and constants of a grid handle; fixbits, fixrows and load are
// allocated zeroed (no fixed DOF, no load) for the caller to fill.
int grid_alloc(int nx, int ny, const double* h_ke, bsp_grid** out) {
  bsp_grid* g = new bsp_grid();
  g->nx = nx;
  g->ny = ny;
  g->N = (long long)(nx + 1) * (ny + 1);
  g->n = 2 * g->N;
  g->E = (long long)nx * ny;
  cudaGetDevice(&g->device);
  cudaDeviceGetAttribute(&g->nsm, cudaDevAttrMultiProcessorCount, g->device);
  ke_modes(h_ke, g);
  std::memcpy(g->ke, h_ke, sizeof(g->ke));
  choose_strips(g);
  const long long words = (g->N + 15) / 16;
  // one partial set per block of every reducing launch: strip kernel (4),
  // adjoint filter tiles (4; 6 when fused with the high-level step), streaming
  // kernels (<= 8 slots x 16*nsm blocks)
  const dim3 fg = filter_grid_max(nx, ny);
  size_t part = std::max<size_t>(4ull * g->sgrid.x * g->sgrid.y, 6ull * fg.x * fg.y);
  part = std::max<size_t>(part, 4ull * g->sgrid3.x * g->sgrid3.y);
  part = std::max<size_t>(part, 8ull * 16 * g->nsm) + 64;
  g->hl_blocks = highlevel_blocks(g->device);
  // row-aligned copy of the mask for the TMA kernel (rows padded to 16 bytes)
  g->fixrow_words = ((nx + 1 + 15) / 16 + 3) & ~3;
  const size_t rows = (size_t)(ny + 1) * g->fixrow_words;
  if (cudaMalloc(&g->fixbits, words * sizeof(uint32_t)) != cudaSuccess ||
      cudaMalloc(&g->load, g->n * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&g->counter, 16 * sizeof(unsigned)) != cudaSuccess ||
      cudaMalloc(&g->st, sizeof(DevState)) != cudaSuccess ||
      cudaMalloc(&g->red, 64 * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&g->part, part * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&g->hl_part, 4ull * g->hl_blocks * sizeof(double)) != cudaSuccess ||
      cudaMallocHost(&g->hpin, 64 * sizeof(double)) != cudaSuccess) {
    cudaGetLastError();
    bsp_grid_destroy(g);
    return FAIL(BSP_ENOMEM, "grid allocation failed (nx=%d ny=%d)", nx, ny);
  }
  g->part_cap = part;
  if (cudaMalloc(&g->fixrows, rows * sizeof(uint32_t)) != cudaSuccess) {
    cudaGetLastError();
    g->fixrows = nullptr;
  }
  cudaMemset(g->fixbits, 0, words * sizeof(uint32_t));
  if (g->fixrows) cudaMemset(g->fixrows, 0, rows * sizeof(uint32_t));
  cudaMemset(g->load, 0, g->n * sizeof(double));
  cudaMemset(g->counter, 0, 16 * sizeof(unsigned));
  cudaMemset(g->st, 0, sizeof(DevState));
  const char* no_tma = getenv("BSP_NO_TMA");
  g->tma_ok = g->fixrows != nullptr;  // odd nx: element tiles per lane (stiffness_tma.cu)
  g->use_tma = g->tma_ok && !(no_tma && no_tma[0] == '1');
  *out = g;
  return BSP_OK;
}

int grid_finish(bsp_grid* g, bsp_grid** out) {
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) {
    bsp_grid_destroy(g);
    return FAIL(BSP_ECUDA, "grid create: %s", cudaGetErrorString(e));
  }
  *out = g;
  return BSP_OK;
}

// fixed DOFs from a sorted index list: OR the 2-bit node masks into both
// layouts (idempotent and order-free, so duplicates and races are harmless)
__global__ void k_scatter_fixed(const long long* dofs, long long m, int nx, uint32_t* fixbits,
                                uint32_t* fixrows, int wr) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x) {
    const long long d = dofs[i], j = d >> 1;
    const uint32_t b = (d & 1) ? 2u : 1u;
    atomicOr(fixbits + (j >> 4), b << (2 * (j & 15)));
    if (fixrows) {
      const long long y = j / (nx + 1), x = j % (nx + 1);
      atomicOr(fixrows + (size_t)y * wr + (x >> 4), b << (2 * (x & 15)));
    }
  }
}

__global__ void k_scatter_load(const long long* dofs, const double* vals, long long m,
                               double* load) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m;
       i += (long long)gridDim.x * blockDim.x)
    load[dofs[i]] = vals[i];
}
}  // namespace

extern "C" int bsp_grid_create(int nx, int ny, const double* h_ke, const uint8_t* h_fixed,
                               const double* h_load, bsp_grid** out) {
  if (nx < 1 || ny < 1) return FAIL(BSP_EINVAL, "grid must have at least one element per axis");
  if (!h_ke || !h_fixed || !h_load || !out) return FAIL(BSP_EINVAL, "null argument");
  bsp_grid* g = nullptr;
  int rc = grid_alloc(nx, ny, h_ke, &g);
  if (rc) return rc;
  const long long words = (g->N + 15) / 16;
  std::vector<uint32_t> bits(words, 0u);
  for (long long j = 0; j < g->N; ++j) {
    uint32_t b = (h_fixed[2 * j] ? 1u : 0u) | (h_fixed[2 * j + 1] ? 2u : 0u);
    bits[j >> 4] |= b << (2 * (j & 15));
  }
  cudaMemcpy(g->fixbits, bits.data(), words * sizeof(uint32_t), cudaMemcpyHostToDevice);
  if (g->fixrows) {
    const int wr = g->fixrow_words;
    std::vector<uint32_t> rows((size_t)(ny + 1) * wr, 0u);
    for (long long j = 0; j < g->N; ++j) {
      const long long y = j / (nx + 1), x = j % (nx + 1);
      const uint32_t b = (h_fixed[2 * j] ? 1u : 0u) | (h_fixed[2 * j + 1] ? 2u : 0u);
      rows[(size_t)y * wr + (x >> 4)] |= b << (2 * (x & 15));
    }
    cudaMemcpy(g->fixrows, rows.data(), rows.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
  }
  cudaMemcpy(g->load, h_load, g->n * sizeof(double), cudaMemcpyHostToDevice);
  return grid_finish(g, out);
}

extern "C" int bsp_grid_create_sparse(int nx, int ny, const double* h_ke, long long n_fixed,
                                      const long long* h_fixed_dofs, long long n_load,
                                      const long long* h_load_dofs, const double* h_load_vals,
                                      bsp_grid** out) {
  if (nx < 1 || ny < 1) return FAIL(BSP_EINVAL, "grid must have at least one element per axis");
  if (!h_ke || !out || n_fixed < 0 || n_load < 0 || (n_fixed && !h_fixed_dofs) ||
      (n_load && (!h_load_dofs || !h_load_vals)))
    return FAIL(BSP_EINVAL, "null argument");
  const long long n = 2ll * (nx + 1) * (ny + 1);
  for (long long i = 0; i < n_fixed; ++i)
    if (h_fixed_dofs[i] < 0 || h_fixed_dofs[i] >= n)
      return FAIL(BSP_EINVAL, "fixed DOF %lld outside [0, %lld)", h_fixed_dofs[i], n);
  for (long long i = 0; i < n_load; ++i)
    if (h_load_dofs[i] < 0 || h_load_dofs[i] >= n)
      return FAIL(BSP_EINVAL, "load DOF %lld outside [0, %lld)", h_load_dofs[i], n);
  bsp_grid* g = nullptr;
  int rc = grid_alloc(nx, ny, h_ke, &g);
  if (rc) return rc;
  long long* d_idx = nullptr;
  double* d_val = nullptr;
  const long long m = std::max(n_fixed, n_load);
  if (m > 0 && (cudaMalloc(&d_idx, m * sizeof(long long)) != cudaSuccess ||
                cudaMalloc(&d_val, std::max(n_load, 1ll) * sizeof(double)) != cudaSuccess)) {
    cudaGetLastError();
    cudaFree(d_idx);
    bsp_grid_destroy(g);
    return FAIL(BSP_ENOMEM, "sparse grid scratch allocation failed");
  }
  const unsigned nb = (unsigned)std::max<long long>(1, std::min<long long>((m + 255) / 256, 1024));
  if (n_fixed > 0) {
    cudaMemcpy(d_idx, h_fixed_dofs, n_fixed * sizeof(long long), cudaMemcpyHostToDevice);
    k_scatter_fixed<<<nb, 256>>>(d_idx, n_fixed, nx, g->fixbits, g->fixrows, g->fixrow_words);
  }
  if (n_load > 0) {
    cudaDeviceSynchronize();  // d_idx is reused
    cudaMemcpy(d_idx, h_load_dofs, n_load * sizeof(long long), cudaMemcpyHostToDevice);
    cudaMemcpy(d_val, h_load_vals, n_load * sizeof(double), cudaMemcpyHostToDevice);
    k_scatter_load<<<nb, 256>>>(d_idx, d_val, n_load, g->load);
  }
  rc = grid_finish(g, out);
  cudaFree(d_idx);
  cudaFree(d_val);
  return rc;
}

extern "C" int bsp_grid_info(const bsp_grid* g, long long* n_dofs, long long* n_elem, int* flags) {
  if (!g) return FAIL(BSP_EINVAL, "null grid");
  if (n_dofs) *n_dofs = g->n;
  if (n_elem) *n_elem = g->E;
  if (flags) *flags = (g->km.iso ? 1 : 0) | (g->uniform_diag ? 2 : 0);
  return BSP_OK;
}

// -------------------------------------------------------------------- ops ---
extern "C" int bsp_apply_stiffness(bsp_grid* g, const double* d_a, const double* d_u, double* d_y,
                                   void* stream) {
  if (!g || !d_a || !d_u || !d_y) return FAIL(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(g->device);
  StiffArgs p = stiff_args(g);
  p.a = d_a;
  p.u = (const double2*)d_u;
  p.out = (double2*)d_y;
  BSP_CU(launch_stiff(g, p, (cudaStream_t)stream));
  return BSP_OK;
}

extern "C" int bsp_apply_stiffness_premasked(bsp_grid* g, const double* d_a, const double* d_u,
                                             double* d_y, void* stream) {
  if (!g || !d_a || !d_u || !d_y) return FAIL(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(g->device);
  StiffArgs p = stiff_args(g);
  p.a = d_a;
  p.u = (const double2*)d_u;
  p.out = (double2*)d_y;
  p.flags = SF_IN_MASKED;
  BSP_CU(launch_stiff(g, p, (cudaStream_t)stream));
  return BSP_OK;
}

extern "C" int bsp_stiffness_diagonal(bsp_grid* g, const double* d_a, double* d_d, void* stream) {
  if (!g || !d_a || !d_d) return FAIL(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(g->device);
  if (!g->uniform_diag)
    return FAIL(BSP_EUNSUPPORTED, "stiffness_diagonal needs a uniform ke diagonal");
  k_diag<<<node_grid(g->nx, g->ny, wave_blocks((const void*)k_diag, 256)), 256, 0, (cudaStream_t)stream>>>(g->view(), g->km, d_a,
                                                                          (double2*)d_d);
  BSP_CU(cudaGetLastError());
  return BSP_OK;
}

// energies are a-free: the element pass runs with a = 0 and no vector output
static int energies_into(bsp_grid* g, const double* d_u, const double* vp, double eta, double* out,
                         cudaStream_t s) {
  int rc = ensure_wk(g, (size_t)g->E);
  if (rc) return rc;
  BSP_CU(cudaMemsetAsync(g->wk, 0, g->E * sizeof(double), s));
  StiffArgs p = stiff_args(g);
  p.a = g->wk;
  p.u = (const double2*)d_u;
  p.flags = SF_ENERGY;
  p.vp = vp;
  p.eta = eta;
  p.sens = out;
  BSP_CU(launch_stiff(g, p, s));
  return BSP_OK;
}

extern "C" int bsp_element_energies(bsp_grid* g, const double* d_u, double* d_e, void* stream) {
  if (!g || !d_u || !d_e) return FAIL(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(g->device);
  return energies_into(g, d_u, nullptr, 1.0, d_e, (cudaStream_t)stream);
}

extern "C" int bsp_residual(bsp_grid* g, const double* d_a, const double* d_u, double* d_r,
                            double* h_out, void* stream) {
  if (!g || !d_a || !d_u) return FAIL(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(g->device);
  cudaStream_t s = (cudaStream_t)stream;
  StiffArgs p = stiff_args(g);
  p.a = d_a;
  p.u = (const double2*)d_u;
  p.out = (double2*)d_r;
  p.flags = SF_SUB_LOAD | SF_REDUCE;
  p.hook = HK_STORE;
  p.red_out = g->red;
  BSP_CU(launch_stiff(g, p, s));
  if (h_out) {
    BSP_CU(cudaMemcpyAsync(g->hpin, g->red, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    BSP_CU(cudaStreamSynchronize(s));
    for (int i = 0; i < 4; ++i) h_out[i] = g->hpin[i];
  }
  return BSP_OK;
}

extern "C" int bsp_sensitivity(bsp_grid* g, const double* d_vphys, const double* d_u, double eta,
                               const double* h_taps, int n_taps, double* d_out, void* stream) {
  if (!g || !d_vphys || !d_u || !d_out) return FAIL(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(g->device);
  FilterTaps w;
  int rc = make_taps(h_taps, n_taps, w);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  rc = ensure_wk(g, 2 * (size_t)g->E);
  if (rc) return rc;
  double* sens = g->wk + g->E;
  // energies_into uses wk[0:E] for the zero activation
  BSP_CU(cudaMemsetAsync(g->wk, 0, g->E * sizeof(double), s));
  StiffArgs p = stiff_args(g);
  p.a = g->wk;
  p.u = (const double2*)d_u;
  p.flags = SF_ENERGY;
  p.vp = d_vphys;
  p.eta = eta;
  p.sens = sens;
  BSP_CU(launch_stiff(g, p, s));
  return launch_filter_scratch(sens, d_out, nullptr, 1.0, g->nx, g->ny, w, 1, s);
}

extern "C" int bsp_filter(const double* d_in, double* d_out, double* d_act, double eta, int nx,
                          int ny, const double* h_taps, int n_taps, int adjoint, void* stream) {
  if (!d_in || !d_out) return FAIL(BSP_EINVAL, "null argument");
  if (nx < 1 || ny < 1) return FAIL(BSP_EINVAL, "bad shape %dx%d", nx, ny);
  FilterTaps w;
  int rc = make_taps(h_taps, n_taps, w);
  if (rc) return rc;
  return launch_filter_scratch(d_in, d_out, adjoint ? nullptr : d_act, eta, nx, ny, w, adjoint,
                               (cudaStream_t)stream);
}

// ---------------------------------------------------- power iterations -----
// y_i = K(x_i) with x_i = y_{i-1}/|y_{i-1}| applied lazily through in_div
static int power_common(bsp_grid* g, const double* d_a, const double* d_x0, int iters,
                        bool sqjacobi, double* h_rho, cudaStream_t s) {
  int rc = ensure_wk(g, 3 * (size_t)g->n);
  if (rc) return rc;
  double* B[2] = {g->wk, g->wk + g->n};
  double* T = g->wk + 2 * g->n;
  static DevState zero{};
  DevState init = zero;
  init.rho = sqjacobi ? 1.0 : 0.0;
  BSP_CU(cudaMemcpyAsync(g->st, &init, sizeof(DevState), cudaMemcpyHostToDevice, s));
  for (int i = 0; i < iters; ++i) {
    const double2* x = (i == 0) ? (const double2*)d_x0 : (const double2*)B[(i - 1) & 1];
    // the norms ping-pong in pw[0..1]: launch i reads pw[(i-1)&1] (its input
    // scale) and its last block writes pw[i&1]; launch i+1 follows in stream
    // order, so any iteration count works
    const double* xdiv = (i == 0) ? nullptr : &g->st->pw[(i - 1) & 1];
    StiffArgs p = stiff_args(g);
    p.a = d_a;
    p.gate0 = &g->st->pow_stop;
    p.u = x;
    p.in_div = xdiv;
    p.hook_i = i;
    if (!sqjacobi) {
      p.out = (double2*)B[i & 1];
      p.flags = SF_REDUCE | SF_IN_MASKED;  // start vector masked on the host
      p.hook = HK_POWER;
      p.red_need = 3;  // u.Ku, |t|^2
      BSP_CU(launch_stiff(g, p, s));
    } else {
      p.out = (double2*)T;
      p.flags = SF_D2DIV | SF_IN_MASKED;
      BSP_CU(launch_stiff(g, p, s));
      StiffArgs q = stiff_args(g);
      q.a = d_a;
      q.gate0 = &g->st->pow_stop;
      q.u = (const double2*)T;
      q.out = (double2*)B[i & 1];
      q.dotv = x;
      q.dot_div = xdiv;
      q.flags = SF_REDUCE | SF_IN_MASKED;
      q.hook = HK_POWER_DOT;
      q.red_need = 6;  // |t|^2, dot
      q.hook_i = i;
      BSP_CU(launch_stiff(g, q, s));
    }
  }
  BSP_CU(cudaMemcpyAsync(g->hpin, &g->st->rho, sizeof(double), cudaMemcpyDeviceToHost, s));
  BSP_CU(cudaStreamSynchronize(s));
  *h_rho = g->hpin[0];
  return BSP_OK;
}

extern "C" int bsp_estimate_rho_max(bsp_grid* g, const double* d_a, const double* d_x0, int iters,
                                    double* h_rho, void* stream) {
  if (!g || !d_a || !d_x0 || !h_rho) return FAIL(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(g->device);
  if (iters < 5) return FAIL(BSP_EINVAL, "iters must be >= 5");
  return power_common(g, d_a, d_x0, iters, false, h_rho, (cudaStream_t)stream);
}

extern "C" int bsp_estimate_sqjacobi_rho(bsp_grid* g, const double* d_a, const double* d_x0,
                                         int iters, double* h_rho, void* stream) {
  if (!g || !d_a || !d_x0 || !h_rho) return FAIL(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(g->device);
  if (!g->uniform_diag) return FAIL(BSP_EUNSUPPORTED, "Jacobi power iteration needs uniform diag");
  return power_common(g, d_a, d_x0, iters, true, h_rho, (cudaStream_t)stream);
}

// ---------------------------------------------------------------- Krylov ---
// q_0 = b; q_{i+1} = K(q_i/|q_i|) with the norms reduced on the device; TSQR
// of [P_1..P_count | b]; out = base - beta * sum_i c_i/growth_i P_i.
namespace bsp {
int krylov_enqueue(bsp_grid* g, const double* d_a, const double* d_b, int dim, const double* d_base,
                   double beta, double* d_out, double* Q, bool b_in_Q0, const int* gate,
                   cudaStream_t s) {
  const int npow_req = (int)std::min<long long>((long long)dim + 1, g->n);
  const int npow = krylov_formed(npow_req);  // > 63 powers: truncated, checked in the solve
  const int nc = npow + 1;
  const int blocks = tsqr_leaves(g->n, nc);
  int rc = ensure_tsqr(g);
  if (rc) return rc;
  const long long ldq = g->n;
  if (!b_in_Q0) {
    BSP_CU(cudaMemcpyAsync(Q, d_b, g->n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    RedBuf rb{g->part, g->counter};
    k_sum<<<(unsigned)std::min<long long>((g->n + 255) / 256, 4 * g->nsm), 256, 0, s>>>(
        d_b, g->n, rb, &g->st->scratch[0]);
    BSP_CU(cudaGetLastError());
    k_kry_init<<<1, 1, 0, s>>>(g->st);
    BSP_CU(cudaGetLastError());
  }
  for (int i = 0; i < npow; ++i) {
    StiffArgs p = stiff_args(g);
    p.a = d_a;
    p.u = (const double2*)(Q + i * ldq);
    p.in_div = &g->st->norms[i];
    p.out = (double2*)(Q + (i + 1) * ldq);
    // q_i (i >= 1) are masked matvec outputs; a caller's b may not be
    p.flags = SF_REDUCE | ((i > 0 || b_in_Q0) ? SF_IN_MASKED : 0);
    p.hook = HK_KRYLOV;
    p.red_need = 2;  // |t|^2
    p.hook_i = i;
    p.gate0 = gate ? gate : &g->st->done;
    p.gate1 = &g->st->kry_stop;
    BSP_CU(launch_stiff(g, p, s));
  }
  KryArgs ka{};
  ka.Q = Q;
  ka.ldq = ldq;
  ka.n = g->n;
  ka.Rbuf = g->Rbuf;
  ka.st = g->st;
  ka.u = d_base;
  ka.out = d_out;
  ka.beta = beta;
  ka.npow_req = npow_req;
  BSP_CU(launch_tsqr_leaf(nc, blocks, ka, s));
  // fan-in tree down to one CTA, which also applies the rank cut and solves
  const int fan = tsqr_fan_in(nc);
  const size_t half = (size_t)blocks * tsqr_rdim(nc) * tsqr_rdim(nc);
  int nin = blocks, lvl = 0;
  do {
    const int nout = (nin + fan - 1) / fan;
    const double* rin = g->Rbuf + ((lvl & 1) ? half : 0);
    double* rout = g->Rbuf + ((lvl & 1) ? 0 : half);
    BSP_CU(launch_tsqr_merge(nc, nout, ka, rin, nin, rout, s));
    nin = nout;
    ++lvl;
  } while (nin > 1);
  k_kry_combine<<<(unsigned)std::min<long long>((g->n + 255) / 256, 8 * g->nsm), 256, 0, s>>>(ka);
  BSP_CU(cudaGetLastError());
  return BSP_OK;
}
}  // namespace bsp

static int reset_state(bsp_grid* g, cudaStream_t s) {
  static DevState zero{};
  BSP_CU(cudaMemcpyAsync(g->st, &zero, sizeof(DevState), cudaMemcpyHostToDevice, s));
  return BSP_OK;
}

// read back the rank and refuse a truncated basis whose cut the formed
// columns do not contain (krylov.cu)
static int krylov_check(bsp_grid* g, int* h_rank, cudaStream_t s) {
  BSP_CU(cudaMemcpyAsync(g->hpin, &g->st->kry_rank, sizeof(int), cudaMemcpyDeviceToHost, s));
  BSP_CU(cudaMemcpyAsync((int*)g->hpin + 1, &g->st->kry_trunc, sizeof(int),
                         cudaMemcpyDeviceToHost, s));
  BSP_CU(cudaStreamSynchronize(s));
  if (h_rank) *h_rank = ((int*)g->hpin)[0];
  if (((int*)g->hpin)[1])
    return FAIL(BSP_EUNSUPPORTED,
                "Krylov basis numerically full rank past %d powers: krylov_dim > %d needs a "
                "wider TSQR", kTsqrMaxCols - 1, kTsqrMaxCols - 2);
  return BSP_OK;
}

extern "C" int bsp_krylov_apply(bsp_grid* g, const double* d_a, const double* d_b, int dim,
                                double* d_out, int* h_rank, void* stream) {
  if (!g || !d_a || !d_b || !d_out) return FAIL(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(g->device);
  if (dim < 1) return FAIL(BSP_EINVAL, "Krylov dimension must be at least 1");
  cudaStream_t s = (cudaStream_t)stream;
  const int npow = krylov_formed((int)std::min<long long>((long long)dim + 1, g->n));
  int rc = ensure_wk(g, (size_t)(npow + 1) * g->n);
  if (rc) return rc;
  rc = reset_state(g, s);
  if (rc) return rc;
  rc = krylov_enqueue(g, d_a, d_b, dim, nullptr, -1.0, d_out, g->wk, false, nullptr, s);
  if (rc) return rc;
  return krylov_check(g, h_rank, s);
}

extern "C" int bsp_low_level_step(bsp_grid* g, int algorithm, const double* d_a, const double* d_u,
                                  double beta, const double* d_residual, int krylov_dim,
                                  double* d_out, void* stream) {
  if (!g || !d_a || !d_u || !d_out) return FAIL(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(g->device);
  if (algorithm < BSP_ALGO_FBTO || algorithm > BSP_ALGO_CPFBTO_KRYLOV)
    return FAIL(BSP_EINVAL, "low_level_step does not apply to algorithm %d", algorithm);
  if (algorithm == BSP_ALGO_CPFBTO_KRYLOV && krylov_dim < 1)
    return FAIL(BSP_EINVAL, "Krylov dimension must be at least 1");
  cudaStream_t s = (cudaStream_t)stream;
  const int npow = krylov_formed((int)std::min<long long>((long long)std::max(krylov_dim, 1) + 1, g->n));
  int rc = ensure_wk(g, (size_t)(npow + 2) * g->n);
  if (rc) return rc;
  double* r = g->wk + (size_t)(npow + 1) * g->n;
  if (!d_residual) {
    StiffArgs p = stiff_args(g);
    p.a = d_a;
    p.u = (const double2*)d_u;
    p.out = (double2*)r;
    p.flags = SF_SUB_LOAD;
    BSP_CU(launch_stiff(g, p, s));
    d_residual = r;
  }
  const unsigned nb = (unsigned)std::min<long long>((g->n + 255) / 256, 8 * g->nsm);
  switch (algorithm) {
    case BSP_ALGO_FBTO:
      k_axpy<<<nb, 256, 0, s>>>(d_u, d_residual, -beta, d_out, g->n);
      BSP_CU(cudaGetLastError());
      return BSP_OK;
    case BSP_ALGO_PFBTO_JACOBI: {
      if (!g->uniform_diag) return FAIL(BSP_EUNSUPPORTED, "PFBTO needs a uniform ke diagonal");
      double* z = g->wk;
      k_diag<<<node_grid(g->nx, g->ny, wave_blocks((const void*)k_diag, 256)), 256, 0, s>>>(g->view(), g->km, d_a, (double2*)z);
      k_div_sq<<<nb, 256, 0, s>>>(d_residual, z, z, g->n);
      BSP_CU(cudaGetLastError());
      StiffArgs q = stiff_args(g);
      q.a = d_a;
      q.u = (const double2*)z;
      q.out = (double2*)d_out;
      q.base = (const double2*)d_u;
      q.beta = beta;
      q.flags = SF_AXPY;
      BSP_CU(launch_stiff(g, q, s));
      return BSP_OK;
    }
    default: {
      rc = reset_state(g, s);
      if (rc) return rc;
      rc = krylov_enqueue(g, d_a, d_residual, krylov_dim, d_u, beta, d_out, g->wk, false,
                          nullptr, s);
      if (rc) return rc;
      return krylov_check(g, nullptr, s);
    }
  }
}

// -------------------------------------------------------- design updates ---
// standalone projection / high-level step: a private device state per thread
// (gsum in, measurements out) drives the same kernels as the solver loop
struct HLScratch {
  DevState* st = nullptr;
  double* part = nullptr;   // cooperative k_hl_fix
  double* red = nullptr;    // last-block reductions
  unsigned* cnt = nullptr;
  int fix_blocks = 0, nsm = 0;
};

constexpr int kMaxDevices = 64;

static int current_device(int& dev) {
  BSP_CU(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return FAIL(BSP_EUNSUPPORTED, "device %d", dev);
  return BSP_OK;
}

// per thread and device (the buffers live on the device that was current)
static int hl_scratch(HLScratch*& out) {
  static thread_local HLScratch hs[kMaxDevices];
  int dev = 0;
  int rc = current_device(dev);
  if (rc) return rc;
  HLScratch& h = hs[dev];
  if (!h.st) {
    cudaDeviceGetAttribute(&h.nsm, cudaDevAttrMultiProcessorCount, dev);
    h.fix_blocks = highlevel_blocks(dev);
    BSP_CU(cudaMalloc(&h.st, sizeof(DevState)));
    BSP_CU(cudaMalloc(&h.part, 4ull * h.fix_blocks * sizeof(double)));
    BSP_CU(cudaMalloc(&h.red, 8ull * 8 * h.nsm * sizeof(double)));
    BSP_CU(cudaMalloc(&h.cnt, sizeof(unsigned)));
    BSP_CU(cudaMemset(h.cnt, 0, sizeof(unsigned)));
  }
  out = &h;
  return BSP_OK;
}

static int hl_launch(const double* v, const double* gr, long long n, double alpha, double lo,
                     double hi, double budget, const uint8_t* active, double n_active, int mp,
                     double* out, cudaStream_t s) {
  HLScratch* h = nullptr;
  int rc = hl_scratch(h);
  if (rc) return rc;
  static const DevState zero{};
  BSP_CU(cudaMemcpyAsync(h->st, &zero, sizeof(DevState), cudaMemcpyHostToDevice, s));
  RedBuf rb{h->red, h->cnt};
  if (gr && mp) {
    k_masked_sum<<<write_blocks(n, h->nsm), 256, 0, s>>>(gr, active, n, rb, h->st);
    BSP_CU(cudaGetLastError());
  }
  HLArgs a{};
  a.v = v;
  a.g = gr;
  a.v_next = out;
  a.active = active;
  a.E = n;
  a.n_active = n_active;
  a.lo = lo;
  a.hi = hi;
  a.budget = budget;
  a.alpha = alpha;
  a.mean_projection = mp;
  a.rb = rb;
  a.part = h->part;
  a.st = h->st;
  BSP_CU(launch_highlevel(a, h->fix_blocks, h->nsm, s));
  return BSP_OK;
}

extern "C" int bsp_project_simplex(const double* d_v, long long n, double lo, double hi,
                                   double budget, double* d_out, void* stream) {
  if (!d_v || !d_out) return FAIL(BSP_EINVAL, "null argument");
  if (!(0.0 < lo && lo < hi)) return FAIL(BSP_EINVAL, "need 0 < v_lo < v_hi, got [%g, %g]", lo, hi);
  if (!((double)n * lo <= budget && budget <= (double)n * hi))
    return FAIL(BSP_EINVAL, "budget %g infeasible for %lld elements in [%g, %g]", budget, n, lo, hi);
  return hl_launch(d_v, nullptr, n, 0.0, lo, hi, budget, nullptr, (double)n, 0, d_out,
                   (cudaStream_t)stream);
}

extern "C" int bsp_high_level_step(const double* d_v, const double* d_g, long long n, double alpha,
                                   double lo, double hi, double budget, const uint8_t* d_active,
                                   int mean_projection, double* d_out, void* stream) {
  if (!d_v || !d_g || !d_out) return FAIL(BSP_EINVAL, "null argument");
  cudaStream_t s = (cudaStream_t)stream;
  double n_active = (double)n;
  if (d_active) {
    std::vector<uint8_t> h(n);
    BSP_CU(cudaMemcpyAsync(h.data(), d_active, n, cudaMemcpyDeviceToHost, s));
    BSP_CU(cudaStreamSynchronize(s));
    long long c = 0;
    for (long long i = 0; i < n; ++i) c += h[i] ? 1 : 0;
    n_active = (double)c;
  }
  if (n_active < 1) return FAIL(BSP_EINVAL, "mean_project needs at least one entry");
  if (!(0.0 < lo && lo < hi)) return FAIL(BSP_EINVAL, "need 0 < v_lo < v_hi, got [%g, %g]", lo, hi);
  if (!(n_active * lo <= budget && budget <= n_active * hi))
    return FAIL(BSP_EINVAL, "budget %g infeasible for %g elements in [%g, %g]", budget, n_active,
                lo, hi);
  return hl_launch(d_v, d_g, n, alpha, lo, hi, budget, d_active, n_active, mean_projection, d_out,
                   s);
}

extern "C" int bsp_mean_project(const double* d_g, long long n, double* d_out, void* stream) {
  if (!d_g || !d_out) return FAIL(BSP_EINVAL, "null argument");
  if (n < 1) return FAIL(BSP_EINVAL, "mean_project needs at least one entry");
  cudaStream_t s = (cudaStream_t)stream;
  struct MeanScratch {
    double* buf = nullptr;
    unsigned* cnt = nullptr;
    double* part = nullptr;
    int nsm = 0;
  };
  static thread_local MeanScratch ms[kMaxDevices];  // per thread and device
  int dev = 0;
  int rc = current_device(dev);
  if (rc) return rc;
  double*& buf = ms[dev].buf;
  unsigned*& cnt = ms[dev].cnt;
  double*& part = ms[dev].part;
  int& nsm = ms[dev].nsm;
  if (!buf) {
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    BSP_CU(cudaMalloc(&buf, 4 * sizeof(double)));
    BSP_CU(cudaMalloc(&cnt, sizeof(unsigned)));
    BSP_CU(cudaMemset(cnt, 0, sizeof(unsigned)));
    BSP_CU(cudaMalloc(&part, 4ull * 4 * nsm * sizeof(double)));
  }
  const unsigned blocks = (unsigned)std::min<long long>((n + 255) / 256, 4 * nsm);
  RedBuf rb{part, cnt};
  k_sum<<<blocks, 256, 0, s>>>(d_g, n, rb, buf);
  BSP_CU(cudaGetLastError());
  k_mean_sub<<<blocks, 256, 0, s>>>(d_g, n, buf + 1, d_out);
  BSP_CU(cudaGetLastError());
  return BSP_OK;
}
