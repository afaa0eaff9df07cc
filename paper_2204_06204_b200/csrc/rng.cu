// numpy's seeded normal stream on the device: the power-iteration start
// vector of the reference, np.random.default_rng(seed).standard_normal(n),
// masked and normalised (fea.py:289-292, solvers.py:352-355).  At C5 (268M
// DOFs) numpy needs 3.7 s on one host core; this takes milliseconds.
//
// The algorithm is numpy's (oracle/rng_oracle.py restates it and is pinned to
// numpy bit for bit): PCG64 XSL-RR 128/64 (state <- state*M + inc, output
// rotr64(hi ^ lo, hi >> 58)) and the 256-layer ziggurat of
// random_standard_normal with numpy's own tables (ziggurat_tables.cuh).  The
// ziggurat consumes a variable number of draws per normal (1 for 99%; a
// wedge attempt 2; a tail attempt 1 + 2m), so the k-th normal is not at a
// known draw.  The stream is therefore parsed in parallel:
//   1. k_raw: every 64-bit draw, warp-interleaved (lane l steps by the
//      32-step jump A^32, C_32 from its own jumped start: coalesced stores);
//   2. k_chunk_map: per chunk of kChunk draws and per entry offset o < kK
//      (where the first attempt of the chunk starts), the exit offset into
//      the next chunk and the number of normals emitted.  Attempts are a
//      chain j -> j + len(j); chains from different entries merge within a
//      few draws, so entries o > 0 are walked only until they meet entry 0's
//      chain (a bitmap of its attempt starts);
//   3. k_seg_map / k_seg_walk / k_chunk_walk: the composition of the chunk
//      maps from entry 0 (a scan over functions of kK states) gives every
//      chunk's true entry and its first output index;
//   4. k_emit: every chunk re-walks its chain from the true entry and writes
//      its normals.
// Then the fixed DOFs are zeroed and the vector is scaled by 1/||x||
// (deterministic tree sum; numpy uses BLAS ddot, so the normalised vector
// agrees to rounding, the raw normals bit for bit).
//
// Floating point: the wedge test (fi[i-1]-fi[i])*u + fi[i] < exp(-x*x/2)
// and the tail test yy + yy > xx*xx are evaluated with explicit round-to-
// nearest operations (no FMA contraction, like numpy's baseline x86-64
// build).  exp and log1p are CUDA's (1 ulp) rather than glibc's: an accept
// decision can differ only when the two sides agree to an ulp (never seen),
// and a tail value -kInvR*log1p(-U) may differ in its last bit.
#include <algorithm>
#include <cstring>

#include "grid.cuh"
#include "ziggurat_tables.cuh"

namespace bsp {
namespace {

constexpr int kChunk = 256;  // draws per chunk map
constexpr int kK = 16;       // entry / exit offsets tracked per chunk
constexpr int kSeg = 64;     // chunks per segment of the map scan

struct U128 {
  uint64_t lo, hi;
};
__host__ __device__ inline U128 mul128(U128 a, U128 b) {
#ifdef __CUDA_ARCH__
  const uint64_t hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
#else
  const unsigned __int128 p = (unsigned __int128)a.lo * b.lo;
  const uint64_t hi = (uint64_t)(p >> 64) + a.lo * b.hi + a.hi * b.lo;
#endif
  return U128{a.lo * b.lo, hi};
}
__host__ __device__ inline U128 add128(U128 a, U128 b) {
  const uint64_t lo = a.lo + b.lo;
  return U128{lo, a.hi + b.hi + (lo < a.lo ? 1u : 0u)};
}
constexpr U128 kMult{0x4385DF649FCCF645ull, 0x2360ED051FC65DA4ull};

// (A^delta, C_delta) with state_{t+delta} = A^delta state_t + C_delta
// (pcg_advance_lcg_128)
__host__ __device__ inline void jump(uint64_t delta, U128 inc, U128& am, U128& ap) {
  U128 acc_mult{1, 0}, acc_plus{0, 0}, cur_mult = kMult, cur_plus = inc;
  while (delta) {
    if (delta & 1) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, U128{1, 0}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  am = acc_mult;
  ap = acc_plus;
}

BSP_DEV uint64_t pcg_output(U128 s) {
  const uint64_t x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

struct Stream {
  U128 state, inc;  // numpy's PCG64 state after seeding (before the first draw)
};

// draws j = 0 .. nd-1 (draw j = output after j+1 steps); lane l of warp w
// produces draws base + l + 32 m, base = 32 * kPerLane * w
constexpr int kPerLane = 64;
__global__ void __launch_bounds__(256) k_raw(Stream st, U128 m32, U128 c32, long long nd,
                                             uint64_t* __restrict__ raw) {
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long j0 = warp * 32 * kPerLane + lane;
  if (j0 >= nd) return;
  U128 am, ap;
  jump((uint64_t)j0 + 1, st.inc, am, ap);
  U128 s = add128(mul128(am, st.state), ap);
  for (int m = 0; m < kPerLane; ++m) {
    const long long j = j0 + 32ll * m;
    if (j >= nd) break;
    raw[j] = pcg_output(s);
    s = add128(mul128(m32, s), c32);
  }
}

struct Tables {
  uint64_t ki[256];
  double wi[256], fi[256];
};

BSP_DEV void load_tables(Tables& t) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    t.ki[i] = zig::ki[i];
    t.wi[i] = zig::wi[i];
    t.fi[i] = zig::fi[i];
  }
  __syncthreads();
}

BSP_DEV double next_double(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

// One ziggurat attempt at draw j (random_standard_normal's loop body): its
// length in draws, whether it emits, and the value it emits.  Returns false
// if the attempt needs draws past nd.
BSP_DEV bool attempt(const Tables& t, const uint64_t* __restrict__ raw, long long nd, long long j,
                     int& len, bool& emits, double& value) {
  const uint64_t r0 = raw[j];
  const int idx = (int)(r0 & 0xff);
  const uint64_t r = r0 >> 8;
  const bool neg = r & 1u;
  const uint64_t rabs = (r >> 1) & 0x000fffffffffffffull;
  double x = (double)rabs * t.wi[idx];
  if (neg) x = -x;
  if (rabs < t.ki[idx]) {
    len = 1;
    emits = true;
    value = x;
    return true;
  }
  if (idx == 0) {  // tail: pairs of uniforms until yy + yy > xx * xx
    for (int m = 0;; ++m) {
      const long long a = j + 1 + 2 * m;
      if (a + 1 >= nd) return false;
      const double xx = __dmul_rn(-zig::kInvR, log1p(-next_double(raw[a])));
      const double yy = -log1p(-next_double(raw[a + 1]));
      if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
        len = 2 + 2 * m + 1;
        emits = true;
        value = ((rabs >> 8) & 1u) ? -__dadd_rn(zig::kR, xx) : __dadd_rn(zig::kR, xx);
        return true;
      }
    }
  }
  if (j + 1 >= nd) return false;  // wedge: one uniform
  const double u = next_double(raw[j + 1]);
  const double lhs = __dadd_rn(__dmul_rn(__dadd_rn(t.fi[idx - 1], -t.fi[idx]), u), t.fi[idx]);
  len = 2;
  emits = lhs < exp(__dmul_rn(__dmul_rn(-0.5, x), x));
  value = x;
  return true;
}

struct ChunkMap {
  uint8_t exit[kK];   // exit offset into the next chunk, per entry offset
  uint16_t cnt[kK];   // normals emitted by attempts starting in this chunk
};

// err bits: 1 = an exit offset >= kK, 2 = the draw buffer ran out
__global__ void __launch_bounds__(128) k_chunk_map(const uint64_t* __restrict__ raw, long long nd,
                                                   long long nchunks, ChunkMap* maps, int* err) {
  __shared__ Tables t;
  load_tables(t);
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  const long long b = c * kChunk, e = b + kChunk;
  uint32_t vis[kChunk / 32] = {};
  int len;
  bool em;
  double v;
  // entry 0: the reference chain
  long long p = b;
  int cnt0 = 0;
  while (p < e) {
    vis[(p - b) >> 5] |= 1u << ((p - b) & 31);
    if (!attempt(t, raw, nd, p, len, em, v)) {
      atomicOr(err, 2);
      return;
    }
    cnt0 += em;
    p += len;
  }
  const long long exit0 = p - e;
  ChunkMap m;
  for (int o = 0; o < kK; ++o) {
    long long q = b + o;
    int cnt = 0;
    bool merged = false;
    while (q < e) {
      if ((vis[(q - b) >> 5] >> ((q - b) & 31)) & 1u) {
        merged = true;
        break;
      }
      if (!attempt(t, raw, nd, q, len, em, v)) {
        atomicOr(err, 2);
        return;
      }
      cnt += em;
      q += len;
    }
    long long ex;
    if (merged) {  // add entry 0's normals from q on
      int before = 0;
      for (long long s = b; s < q;) {
        attempt(t, raw, nd, s, len, em, v);
        before += em;
        s += len;
      }
      cnt += cnt0 - before;
      ex = exit0;
    } else {
      ex = q - e;
    }
    if (ex >= kK) atomicOr(err, 1);
    m.exit[o] = (uint8_t)min(ex, (long long)kK - 1);
    m.cnt[o] = (uint16_t)cnt;
  }
  maps[c] = m;
}

struct SegMap {
  uint8_t exit[kK];
  uint32_t cnt[kK];
};

__global__ void __launch_bounds__(128) k_seg_map(const ChunkMap* __restrict__ maps, long long nchunks,
                                                 long long nseg, SegMap* seg) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long sg = t / kK;
  const int o = (int)(t % kK);
  if (sg >= nseg) return;
  int ent = o;
  uint32_t cnt = 0;
  const long long c1 = min(nchunks, (sg + 1) * kSeg);
  for (long long c = sg * kSeg; c < c1; ++c) {
    cnt += maps[c].cnt[ent];
    ent = maps[c].exit[ent];
  }
  seg[sg].exit[o] = (uint8_t)ent;
  seg[sg].cnt[o] = cnt;
}

// one block: the true entry and first output index of every segment
constexpr int kWalkThreads = 256;
__global__ void __launch_bounds__(kWalkThreads) k_seg_walk(const SegMap* __restrict__ seg,
                                                           long long nseg, uint8_t* seg_entry,
                                                           long long* seg_base) {
  __shared__ uint8_t gexit[kWalkThreads][kK];
  __shared__ long long gcnt[kWalkThreads][kK];
  __shared__ uint8_t gent[kWalkThreads];
  __shared__ long long gbase[kWalkThreads];
  const long long per = (nseg + kWalkThreads - 1) / kWalkThreads;
  const long long s0 = threadIdx.x * per, s1 = min(nseg, s0 + per);
  for (int o = 0; o < kK; ++o) {  // this thread's range composed, per entry
    int ent = o;
    long long cnt = 0;
    for (long long s = s0; s < s1; ++s) {
      cnt += seg[s].cnt[ent];
      ent = seg[s].exit[ent];
    }
    gexit[threadIdx.x][o] = (uint8_t)ent;
    gcnt[threadIdx.x][o] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int ent = 0;
    long long base = 0;
    for (int r = 0; r < kWalkThreads; ++r) {
      gent[r] = (uint8_t)ent;
      gbase[r] = base;
      base += gcnt[r][ent];
      ent = gexit[r][ent];
    }
  }
  __syncthreads();
  int ent = gent[threadIdx.x];
  long long base = gbase[threadIdx.x];
  for (long long s = s0; s < s1; ++s) {
    seg_entry[s] = (uint8_t)ent;
    seg_base[s] = base;
    base += seg[s].cnt[ent];
    ent = seg[s].exit[ent];
  }
}

__global__ void __launch_bounds__(128) k_chunk_walk(const ChunkMap* __restrict__ maps,
                                                    long long nchunks, long long nseg,
                                                    const uint8_t* seg_entry,
                                                    const long long* seg_base, uint8_t* entry,
                                                    long long* base) {
  const long long sg = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (sg >= nseg) return;
  int ent = seg_entry[sg];
  long long b = seg_base[sg];
  const long long c1 = min(nchunks, (sg + 1) * kSeg);
  for (long long c = sg * kSeg; c < c1; ++c) {
    entry[c] = (uint8_t)ent;
    base[c] = b;
    b += maps[c].cnt[ent];
    ent = maps[c].exit[ent];
  }
}

__global__ void __launch_bounds__(128) k_emit(const uint64_t* __restrict__ raw, long long nd,
                                              long long nchunks, const uint8_t* entry,
                                              const long long* base, long long n,
                                              double* __restrict__ out) {
  __shared__ Tables t;
  load_tables(t);
  const long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  long long k = base[c];
  if (k >= n) return;
  const long long e = (c + 1) * kChunk;
  int len;
  bool em;
  double v;
  for (long long p = c * kChunk + entry[c]; p < e && k < n; p += len) {
    attempt(t, raw, nd, p, len, em, v);
    if (em) out[k++] = v;
  }
}

__global__ void k_total(const long long* base, const ChunkMap* maps, const uint8_t* entry,
                        long long last, long long* total) {
  *total = base[last] + maps[last].cnt[entry[last]];
}

// x[fixed] = 0 and the partial sums of x^2 (deterministic two-level tree)
__global__ void __launch_bounds__(256) k_mask_sq(double* x, const uint32_t* fixbits, long long n,
                                                 RedBuf rb, double* out) {
  double s = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    if (fixbits) {
      const uint32_t b = fix_bits(fixbits, i >> 1);
      if ((i & 1) ? (b & 2u) : (b & 1u)) x[i] = 0.0;
    }
    const double v = x[i];
    s += v * v;
  }
  __shared__ double tot[4];
  if (grid_reduce4(rb, s, 0.0, 0.0, -INFINITY, tot) && threadIdx.x == 0) out[0] = tot[0];
}

__global__ void __launch_bounds__(256) k_scale_inv_sqrt(double* x, long long n, const double* ss) {
  const double inv = 1.0 / sqrt(ss[0]);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    x[i] *= inv;
}

}  // namespace

// n normals of the stream into d_out; 0 or a BSP_* code
static int standard_normal_into(const uint64_t* h_state, long long n, double* d_out,
                                cudaStream_t s) {
  if (n <= 0) return BSP_OK;
  const Stream st{U128{h_state[0], h_state[1]}, U128{h_state[2], h_state[3]}};
  U128 m32, c32;
  jump(32, st.inc, m32, c32);
  // 1.022 draws per normal on average: 6% + 4096 spare draws
  const long long nd = n + n / 16 + 4096;
  const long long nchunks = (nd - 2 * kK) / kChunk;  // every chunk can read kK-ish past its end
  const long long nseg = (nchunks + kSeg - 1) / kSeg;
  uint64_t* raw = nullptr;
  ChunkMap* maps = nullptr;
  SegMap* seg = nullptr;
  uint8_t *seg_entry = nullptr, *entry = nullptr;
  long long *seg_base = nullptr, *base = nullptr, *total = nullptr;
  int* err = nullptr;
  auto release = [&]() {
    cudaFree(raw);
    cudaFree(maps);
    cudaFree(seg);
    cudaFree(seg_entry);
    cudaFree(entry);
    cudaFree(seg_base);
    cudaFree(base);
    cudaFree(total);
    cudaFree(err);
  };
  if (cudaMalloc(&raw, nd * 8) != cudaSuccess || cudaMalloc(&maps, nchunks * sizeof(ChunkMap)) ||
      cudaMalloc(&seg, nseg * sizeof(SegMap)) || cudaMalloc(&seg_entry, nseg) ||
      cudaMalloc(&seg_base, nseg * 8) || cudaMalloc(&entry, nchunks) ||
      cudaMalloc(&base, nchunks * 8) || cudaMalloc(&total, 8) || cudaMalloc(&err, 4)) {
    cudaGetLastError();
    release();
    return set_error(BSP_ENOMEM, "standard_normal: scratch allocation failed (n=%lld)", n);
  }
  cudaMemsetAsync(err, 0, 4, s);
  const long long warps = (nd + 32ll * kPerLane - 1) / (32ll * kPerLane);
  k_raw<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, s>>>(st, m32, c32, nd, raw);
  k_chunk_map<<<(unsigned)((nchunks + 127) / 128), 128, 0, s>>>(raw, nd, nchunks, maps, err);
  k_seg_map<<<(unsigned)((nseg * kK + 127) / 128), 128, 0, s>>>(maps, nchunks, nseg, seg);
  k_seg_walk<<<1, kWalkThreads, 0, s>>>(seg, nseg, seg_entry, seg_base);
  k_chunk_walk<<<(unsigned)((nseg + 127) / 128), 128, 0, s>>>(maps, nchunks, nseg, seg_entry,
                                                              seg_base, entry, base);
  k_emit<<<(unsigned)((nchunks + 127) / 128), 128, 0, s>>>(raw, nd, nchunks, entry, base, n, d_out);
  k_total<<<1, 1, 0, s>>>(base, maps, entry, nchunks - 1, total);
  int h_err = 0;
  long long h_total = 0;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h_err, err, 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h_total, total, 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  release();
  if (e != cudaSuccess)
    return set_error(BSP_ECUDA, "standard_normal: %s", cudaGetErrorString(e));
  if (h_err || h_total < n)
    return set_error(BSP_ECUDA, "standard_normal: stream parse failed (flags %d, %lld of %lld)",
                     h_err, h_total, n);
  return BSP_OK;
}

}  // namespace bsp

using namespace bsp;

extern "C" int bsp_standard_normal(const uint64_t* h_state, long long n, double* d_out,
                                   void* stream) {
  if (!h_state || (n > 0 && !d_out)) return set_error(BSP_EINVAL, "null argument");
  if (n < 0) return set_error(BSP_EINVAL, "negative length");
  return standard_normal_into(h_state, n, d_out, (cudaStream_t)stream);
}

extern "C" int bsp_start_vector(bsp_grid* g, const uint64_t* h_state, double* d_x, void* stream) {
  if (!g || !h_state || !d_x) return set_error(BSP_EINVAL, "null argument");
  bsp::DeviceGuard dg_(g->device);
  cudaStream_t s = (cudaStream_t)stream;
  int rc = standard_normal_into(h_state, g->n, d_x, s);
  if (rc) return rc;
  const unsigned nb = (unsigned)std::min<long long>((g->n + 255) / 256, 4ll * g->nsm);
  k_mask_sq<<<nb, 256, 0, s>>>(d_x, g->fixbits, g->n, RedBuf{g->part, g->counter}, g->red);
  k_scale_inv_sqrt<<<nb, 256, 0, s>>>(d_x, g->n, g->red);
  BSP_CU(cudaGetLastError());
  return BSP_OK;
}
