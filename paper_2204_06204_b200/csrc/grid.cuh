// Host-side handle types shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <string>

#include "../../include/bisimp_b200.h"
#include "common.cuh"
#include "filter.cuh"
#include "solver_state.cuh"
#include "stiffness.cuh"

namespace bsp {
struct PcgWork;
__global__ void k_diag(GridView g, KeModes km, const double* __restrict__ a, double2* d);

int set_error(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));

// Scoped device switch: every entry point that takes a handle runs on the
// device the handle was created on, whatever the caller's current device is.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess)
      prev = cur;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// One-time (per kernel, per device) opt-in to `bytes` of dynamic shared
// memory; thread-safe.  The attribute is per device, so a process-wide flag
// would skip the opt-in on a second GPU.
cudaError_t smem_optin(const void* kernel, int bytes);

// blocks of `threads` threads that one wave of `kernel` holds on the current
// device (occupancy x SMs), cached per kernel and device
int wave_blocks(const void* kernel, int threads);
}  // namespace bsp

#define BSP_CU(call)                                                                           \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      return ::bsp::set_error(BSP_ECUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), \
                              __FILE__, __LINE__);                                             \
  } while (0)

struct bsp_mg;
struct bsp_grid {
  int nx = 0, ny = 0;
  long long N = 0, n = 0, E = 0;
  int device = 0;
  int nsm = 148;
  uint32_t* fixbits = nullptr;
  double* load = nullptr;
  bsp::KeModes km{};
  double ke[64] = {};  // host copy of the element stiffness
  bool generic = false, uniform_diag = true;
  int R = 8;        // element rows per strip
  dim3 sgrid;       // strip-kernel grid
  // TMA strip kernel (stiffness_tma.cu): row-aligned 2-bit fixed mask
  // [ny+1][fixrow_words], its grid, and whether it may run (even nx, driver
  // entry point found; BSP_NO_TMA=1 disables it)
  uint32_t* fixrows = nullptr;
  int fixrow_words = 0;
  bool tma_ok = false, use_tma = false;
  int R3 = 8;
  dim3 sgrid3;
  // scratch: a grid handle is not reentrant
  double* part = nullptr;
  size_t part_cap = 0;
  unsigned* counter = nullptr;
  bsp::DevState* st = nullptr;
  double* red = nullptr;
  double* hpin = nullptr;
  double* wk = nullptr;
  size_t wk_cap = 0;
  double* Rbuf = nullptr;
  int tsqr_blocks = 0;
  int hl_blocks = 0;
  double* hl_part = nullptr;
  bsp_mg* mg = nullptr;   // lazily built hierarchy of exact_solve (owned)
  // workspaces of the standalone PCG calls (bsp_pcg_apply, bsp_exact_solve):
  // [0] Jacobi, [1] multigrid; owned, built on first use
  bsp::PcgWork* pcg_ws[2] = {nullptr, nullptr};

  bsp::GridView view() const {
    return bsp::GridView{nx, ny, N, fixbits, (const double2*)load};
  }
};

namespace bsp {
StiffArgs stiff_args(bsp_grid* g);
cudaError_t launch_stiff(bsp_grid* g, const StiffArgs& p, cudaStream_t s);
int make_taps(const double* h_taps, int n, FilterTaps& w);
int launch_filter_scratch(const double* in, double* out, double* act, double eta, int nx, int ny,
                          FilterTaps w, int adjoint, cudaStream_t s);
// Validate cfg->struct_size and copy the caller's prefix over the defaults of
// the optional fields (include/bisimp_b200.h).
int normalize_config(const bsp_solver_config* in, bsp_solver_config& out);
int launch_filter(const double* in, double* out, double* act, double eta, int nx, int ny,
                  const FilterTaps& w, int adjoint, const int* gate, cudaStream_t s,
                  DevState* st = nullptr, const uint8_t* active = nullptr,
                  RedBuf rb = RedBuf{nullptr, nullptr});
FilterArgs filter_args(const double* in, double* out, double* act, double eta, int nx, int ny,
                       const FilterTaps& w, const int* gate, DevState* st, const uint8_t* active,
                       RedBuf rb);
int launch_filter_fa(const FilterArgs& fa, int adjoint, cudaStream_t s);
int ensure_wk(bsp_grid* g, size_t doubles);
int ensure_tsqr(bsp_grid* g);
}  // namespace bsp
