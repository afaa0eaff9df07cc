// Shared device helpers for the B200 bilevel-SIMP hot path (sm_100a, fp64).
//
// Conventions (reference fea.py:8-11): element e = ey*nx+ex, node j = y*(nx+1)+x,
// DOFs (2j, 2j+1) interleaved (ux, uy) -> every DOF vector is a double2 per node.
// Fixed-DOF mask: 2 bits per node packed 16 nodes per 32-bit word (bit 2*(j&15)
// = x fixed, bit 2*(j&15)+1 = y fixed).
#pragma once
#include <algorithm>

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#define BSP_DEV __device__ __forceinline__

#include <utility>

namespace bsp {

// Programmatic dependent launch (PDL): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor runs.
// Every hot kernel begins with pdl_begin (wait for the predecessor's memory)
// and calls pdl_trigger after its main loop (the successor's launch overlaps
// the tail: reductions, stores in flight).
// Both are no-ops for a kernel launched without the attribute.
BSP_DEV void pdl_begin() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// called after a kernel's main loop: the successor may launch during the tail
BSP_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
// the device's global nanosecond timer (stamps of the ConvergenceRecord rows)
BSP_DEV unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Host: launch through cudaLaunchKernelEx with the PDL attribute when
// `pdl_enabled()` (set while the solver records its iteration graphs).
bool& pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  if (!pdl_enabled()) {
    k<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

constexpr int kWarp = 32;
constexpr int kRed = 4;  // reduction slots per block partial

// Element stiffness in the per-component Hadamard mode basis
//   modes per component: T = a0+a1+a2+a3, dx = -a0+a1+a2-a3, dy = -a0-a1+a2+a3,
//   hg = a0-a1+a2-a3 over the local nodes (0,0),(1,0),(1,1),(0,1) (fea.py:64-66);
// M = T ke T^T / 16 so that ke u = T^T M (T u).  For the isotropic unit quad
// only 8 entries of M are non-zero (rigid translations/rotation in its kernel):
//   (dx_x,dx_x)=m11 (dx_x,dy_y)=m16 (dy_y,dy_y)=m66 (dy_x,dy_x)=m22
//   (dy_x,dx_y)=m25 (dx_y,dx_y)=m55 (hg_x,hg_x)=m33 (hg_y,hg_y)=m77.
struct KeModes {
  double m11, m16, m66, m22, m25, m55, m33, m77;
  double kdx, kdy;   // diag(ke) for x / y DOFs (same at all 4 local nodes)
  double ikdx, ikdy, ikdx2, ikdy2;  // 1/kd and 1/kd^2 (Jacobi epilogues)
  double M[64];      // dense M (generic path), row-major over modes
                     // [T_x, dx_x, dy_x, hg_x, T_y, dx_y, dy_y, hg_y]
  int iso;           // 1: sparse isotropic structure holds
};

struct GridView {
  int nx, ny;
  long long n_nodes;  // (nx+1)*(ny+1)
  const uint32_t* fixbits;
  const double2* load;
};

// The node-parallel kernels map (blockIdx.y, x) -> node row and column, so no
// thread divides a 64-bit node index (a software division: ~60 instructions
// per node, which held these kernels at 42-67% of HBM peak at C4).
#define BSP_NODE_LOOP(xx, yy, j, nx, ny)                                                  \
  for (int yy = blockIdx.y; yy <= (ny); yy += gridDim.y)                                 \
    for (int xx = blockIdx.x * blockDim.x + threadIdx.x; xx <= (nx);                       \
         xx += gridDim.x * blockDim.x)                                                     \
      if (const long long j = (long long)yy * ((nx) + 1) + xx; true)

// BSP_NODE_LOOP's grid over the (nx + 1) x (ny + 1) nodes: column blocks of
// 256 threads and as many row blocks as fill exactly one wave of `wave`
// resident blocks (wave_blocks): a few blocks more than a wave would run as a
// second, nearly empty wave and double the kernel time
inline dim3 node_grid(int nx, int ny, int wave) {
  // every thread covers at most one node of a row: a cap below (nx+1)/256
  // blocks made the C5 rows (16385 nodes) take a second trip for one node
  // (k_diag at C5: 60% of peak)
  const int bx = (nx + 1 + 255) / 256;
  const int by = std::max(1, std::min(std::min(ny + 1, 65535), wave / bx));
  return dim3((unsigned)bx, (unsigned)by);
}

// 1/x for the Jacobi scalings (x = a sum of activations: positive, normal):
// the hardware approximation refined by two Newton steps (error far below an
// ulp before the last rounding), without the division's special-case path.
// Every stiffness kernel's D2DIV / D1DIV epilogue uses it (bit-equal kernels).
BSP_DEV double rcp_pos(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  r = fma(fma(-x, r, 1.0), r, r);
  r = fma(fma(-x, r, 1.0), r, r);
  return r;
}

BSP_DEV uint32_t fix_bits(const uint32_t* fb, long long node) {
  return (__ldg(fb + (node >> 4)) >> (2 * (int)(node & 15))) & 3u;
}

// generic-address variant (the mask may sit in shared memory)
BSP_DEV uint32_t fix_bits_gen(const uint32_t* fb, long long node) {
  return (fb[node >> 4] >> (2 * (int)(node & 15))) & 3u;
}

BSP_DEV double2 apply_mask(double2 v, uint32_t bits) {
  if (bits & 1u) v.x = 0.0;
  if (bits & 2u) v.y = 0.0;
  return v;
}

// NaN-propagating max (np.max semantics: any NaN -> NaN)
// SIMP activation a = v_phys^eta (solvers.py:443): numpy's fast paths for
// **2.0 and **1.0, x*x*x for the default eta = 3 (problems.py:82).  The one
// definition every kernel uses, so a stored and a recomputed activation agree
// bit for bit.
BSP_DEV double act_pow(double x, double e) {
  if (e == 3.0) return x * x * x;
  if (e == 2.0) return x * x;
  if (e == 1.0) return x;
  return pow(x, e);
}

BSP_DEV double nanmax(double a, double b) {
  return (b > a || b != b) ? b : a;
}

BSP_DEV double shfl_down_d(double v, int d) { return __shfl_down_sync(0xffffffffu, v, d); }
BSP_DEV double shfl_up_d(double v, int d) { return __shfl_up_sync(0xffffffffu, v, d); }
BSP_DEV double shfl_xor_d(double v, int d) { return __shfl_xor_sync(0xffffffffu, v, d); }

// Deterministic block reduction of N values: slots [0, NS) are sums, slots
// [NS, N) NaN-propagating maxima.  Result valid in thread 0.  Block size must
// be a multiple of 32 and <= 1024.
template <int NS>
BSP_DEV double red_op(int slot, double a, double b) {
  return slot < NS ? a + b : nanmax(a, b);
}

template <int N, int NS>
BSP_DEV void block_reduce_nn(double (&v)[N]) {
  __shared__ double sh[N][32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = red_op<NS>(i, v[i], shfl_xor_d(v[i], o));
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int nw = (blockDim.x * blockDim.y) >> 5;
  const int lane = tid & 31, w = tid >> 5;
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) sh[i][w] = v[i];
  }
  __syncthreads();
  if (w == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = lane < nw ? sh[i][lane] : (i < NS ? 0.0 : -INFINITY);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] = red_op<NS>(i, v[i], shfl_xor_d(v[i], o));
  }
}

template <int NS>
BSP_DEV void block_reduce_n(double (&v)[4]) { block_reduce_nn<4, NS>(v); }

// legacy 4-slot form: 3 sums + (max if MAX3 else sum)
template <bool MAX3 = true>
BSP_DEV void block_reduce4(double& s0, double& s1, double& s2, double& m3) {
  double v[4] = {s0, s1, s2, m3};
  if (MAX3) block_reduce_nn<4, 3>(v); else block_reduce_nn<4, 4>(v);
  s0 = v[0]; s1 = v[1]; s2 = v[2]; m3 = v[3];
}

// Grid-level deterministic reduction: each block writes its N partials, the
// last block to finish reduces all partials in block order and returns true
// (only in that block, all threads).  Totals land in tot[0..N) (shared).
struct RedBuf {
  double* partials;   // [n_blocks * 8]
  unsigned* counter;  // zero-initialised, self-resetting
};

template <int N, int NS>
BSP_DEV bool grid_reduce_nn(const RedBuf& rb, double (&v)[N], double* tot /* __shared__ [N] */) {
  __shared__ int s_last;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int nthr = blockDim.x * blockDim.y;
  const unsigned bid = blockIdx.y * gridDim.x + blockIdx.x;
  const unsigned nblk = gridDim.x * gridDim.y;
  block_reduce_nn<N, NS>(v);
  if (tid == 0) {
    double* p = rb.partials + (unsigned long long)N * bid;
#pragma unroll
    for (int i = 0; i < N; ++i) p[i] = v[i];
    __threadfence();
    unsigned t = atomicAdd(rb.counter, 1u);
    s_last = (t == nblk - 1);
  }
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  double a[N];
#pragma unroll
  for (int i = 0; i < N; ++i) a[i] = i < NS ? 0.0 : -INFINITY;
  for (unsigned b = tid; b < nblk; b += nthr) {
    const double* p = rb.partials + (unsigned long long)N * b;
#pragma unroll
    for (int i = 0; i < N; ++i) a[i] = red_op<NS>(i, a[i], __ldcg(p + i));
  }
  block_reduce_nn<N, NS>(a);
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < N; ++i) tot[i] = a[i];
    *rb.counter = 0u;
  }
  __syncthreads();
  return true;
}

template <int NS = 3>
BSP_DEV bool grid_reduce_n(const RedBuf& rb, double (&v)[4], double* tot) {
  return grid_reduce_nn<4, NS>(rb, v, tot);
}

BSP_DEV bool grid_reduce4(const RedBuf& rb, double s0, double s1, double s2, double m3,
                          double* tot) {
  double v[4] = {s0, s1, s2, m3};
  return grid_reduce_nn<4, 3>(rb, v, tot);
}

}  // namespace bsp
