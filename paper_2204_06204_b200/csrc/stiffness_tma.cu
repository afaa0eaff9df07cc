// Q4 stiffness strip kernel, TMA version (v3).  Same algebra, epilogues and
// summation order per node as the cp.async kernel (stiffness.cu); what
// changes is the data movement.  Inputs that are zero on the fixed DOFs
// (SF_IN_MASKED: every vector the solver produces) are used as staged; the
// public apply_stiffness (unmasked input) zeroes the fixed DOFs of each
// staged node from the staged mask words.
//
// Each warp owns 64 element columns: two per lane, elements eS+2l and
// eS+2l+1 with eS = 62w - 2, which is even.  So every TMA box starts on a
// 16-byte boundary, as TMA requires.  The warp emits the 62 node columns
// [62w, 62w+62) and the energies of the 62 elements [62w, 62w+62), and walks a
// strip of R element rows.  Per row, ONE elected lane issues 2-D TMA tile loads
// (cp.async.bulk.tensor) into a 6-stage per-warp ring:
//   u    (130 doubles), a (64), fixed-mask words (8),
//   plus, per epilogue, f / v_phys / axpy base / dot vector.
// Each stage completes on an mbarrier.  TMA zero-fills every out-of-grid
// coordinate: row -1, row ny+1, column -1, past nx.  So the element loop has no
// bounds logic, and virtual elements with a = 0 contribute nothing.  The
// per-element integer overhead of the per-lane cp.async version (address
// selects, validity predicates, 7 pointer cursors per row) disappears: the
// loop is shared-memory reads, fp64 algebra, one shuffle per node pair and the
// stores.
//
// Layout requirements (checked on the host; otherwise the cp.async kernel
// runs): even nx (element rows must be 16-byte multiples) and 16-byte aligned
// arrays.  The fixed mask is read from its row-aligned copy (grid.cuh
// fixrows).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "grid.cuh"
#include "q4.cuh"

namespace bsp {

namespace {
constexpr int kW3 = 4;     // warps per CTA
constexpr int kS3max = 6;  // ring stages per warp (fewer for the wide epilogue shapes)
constexpr int kEmit = 62;  // node columns emitted per warp
// 4 resident CTAs (16 warps) per SM: the residual variant is bound by fp64
// dependency latency at 3 CTAs (measured: C5 pfbto 4.52 -> 4.30 ms/iter on one
// box); the generic-Ke instances keep their registers (they would spill)
#ifndef BSP_K3_MINB
#define BSP_K3_MINB 4
#endif

struct Maps3 {
  CUtensorMap u, a, m, f, vp, base, dotv, pc;
};

struct L3 {
  int u, a, m, f, vp, base, dotv, pc, size;
  uint32_t tx;  // bytes per stage (TMA counts OOB-filled bytes too)
};

// SF_PROLONG: the two coarse node rows under a fine node row, 34 coarse nodes
// each (68 doubles) starting at coarse column eS/2; each in its own 128-byte
// aligned slot (TMA destinations must be)
constexpr int kCoarseBox = 68;
constexpr int kCoarseSlot = 640;

__host__ __device__ constexpr L3 layout3(int flags) {
  // u: 65 nodes (1040 B), a: 64 elements (512 B), mask: 8 words (32 B),
  // f / base / dotv: 62 nodes (992 B), v_phys: 64 elements; 128-byte slots
  L3 L{0, 1152, 1664, -1, -1, -1, -1, -1, 1792, 1040 + 512 + 32};
  int o = L.size;
  if (flags & SF_SUB_LOAD) { L.f = o; o += 1024; L.tx += 992; }
  if ((flags & SF_STAGE_VP) && !(flags & SF_A_POW)) { L.vp = o; o += 512; L.tx += 512; }
  if ((flags & SF_STAGE_VP) && (flags & SF_A_POW)) L.vp = L.a;  // the a tile is v_phys
  if ((flags & SF_AXPY) && !(flags & SF_BASE_U)) { L.base = o; o += 1024; L.tx += 992; }
  if (flags & SF_REDUCE_DOT) { L.dotv = o; o += 1024; L.tx += 992; }
  if (flags & SF_PROLONG) { L.pc = o; o += 2 * kCoarseSlot; L.tx += 2 * kCoarseBox * 8; }
  L.size = o;
  return L;
}

// stages per warp: as many as fit the per-CTA ring budget, 3..6
// (52 KB: with the static shared memory and the per-CTA reservation, four
// CTAs of the widest residual shape fit the SM's 228 KB)
#ifndef BSP_K3_RING
#define BSP_K3_RING 53248
#endif
__host__ __device__ constexpr int stages3(int flags) {
  const int s = BSP_K3_RING / (kW3 * layout3(flags).size);
  return s < 3 ? 3 : (s > kS3max ? kS3max : s);
}

constexpr int kBarBytes = 256;  // kW3 * kS3max mbarriers (8 B), 128-aligned

BSP_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
BSP_DEV void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
BSP_DEV void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
}
BSP_DEV bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
BSP_DEV void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
BSP_DEV void tma2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}

BSP_DEV double2 ld2(const unsigned char* sp, int off, int idx) {
  return reinterpret_cast<const double2*>(sp + off)[idx];
}

BSP_DEV double2 add2(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
BSP_DEV double2 shfl_up2(double2 v) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1));
}

}  // namespace

template <bool GENERIC, int F>
__global__ void __launch_bounds__(32 * kW3, GENERIC ? 1 : BSP_K3_MINB) k_stiff3(StiffArgs p, KeModes km,
                                                     const __grid_constant__ Maps3 tm) {
  pdl_begin();
  if ((p.gate0 && *p.gate0) || (p.gate1 && *p.gate1)) return;
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr L3 L = layout3(F);
  constexpr int kS3 = stages3(F);
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int eS = (blockIdx.x * kW3 + wib) * kEmit - 2;  // first element column (even)
  const int x0 = eS + 2;                                   // first emitted node column
  // first mask word, 16-byte aligned, at or before node eS: the 8-word mask
  // tile covers every node of the u tile (eS .. eS+64), which input masking
  // needs, and the emitted nodes (arithmetic shift: eS = -2 gives word -4,
  // zero-filled by TMA)
  const int wS = (eS >> 4) & ~3;
  const int nx = p.g.nx, ny = p.g.ny;
  const long long NX1 = nx + 1;
  const int y0 = blockIdx.y * p.R;
  const int y1 = min(y0 + p.R, ny);
  const int nrows = y1 - y0 + 2;  // node rows y0-1 .. y1
  const uint32_t bar0 = smem_u32(smem) + wib * kS3 * 8;
  unsigned char* ring = smem + kBarBytes + (size_t)wib * kS3 * L.size;
  const uint32_t ring_s = smem_u32(ring);

  if (lane == 0) {
    for (int s = 0; s < kS3; ++s) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int t) {  // lane 0: stage t <- node row / element row y0-1+t
    const int slot = t % kS3;
    const uint32_t bar = bar0 + 8 * slot;
    const uint32_t d = ring_s + slot * L.size;
    const int row = y0 - 1 + t;
    mbar_expect_tx(bar, L.tx);
    tma2d(d + L.u, &tm.u, 2 * eS, row, bar);
    tma2d(d + L.a, &tm.a, eS, row, bar);
    tma2d(d + L.m, &tm.m, wS, row, bar);
    if (L.f >= 0) tma2d(d + L.f, &tm.f, 2 * x0, row, bar);
    if (L.vp >= 0 && L.vp != L.a) tma2d(d + L.vp, &tm.vp, eS, row, bar);
    if (L.base >= 0) tma2d(d + L.base, &tm.base, 2 * x0, row, bar);
    if (L.dotv >= 0) tma2d(d + L.dotv, &tm.dotv, 2 * x0, row, bar);
    if (L.pc >= 0) {  // coarse rows row>>1 and row>>1 + 1 (arithmetic shift: row -1 -> -1)
      tma2d(d + L.pc, &tm.pc, eS, row >> 1, bar);
      tma2d(d + L.pc + kCoarseSlot, &tm.pc, eS, (row >> 1) + 1, bar);
    }
  };
  auto wait = [&](int t) { mbar_wait(bar0 + 8 * (t % kS3), (t / kS3) & 1); };

  if (lane == 0)
    for (int t = 0; t < kS3 - 1 && t < nrows; ++t) issue(t);

  const double rinv = p.in_div ? 1.0 / *p.in_div : 1.0;
  const double dinv = p.dot_div ? 1.0 / *p.dot_div : 1.0;
  const int xA = eS + 2 * lane;  // this lane's node columns xA, xA+1, xA+2
  const bool emitA = lane >= 1 && xA <= nx;
  const bool emitB = lane >= 1 && xA + 1 <= nx;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, m3 = -INFINITY;

  // epilogue of one emitted node: ku (already scaled), top-row u, masks
  auto emit = [&](const unsigned char* sp, int x, long long node, double2 ku, double2 uT,
                  double as, bool red) {
    const int wofs = (x >> 4) - wS;
    const uint32_t bits = (reinterpret_cast<const uint32_t*>(sp + L.m)[wofs] >> (2 * (x & 15))) & 3u;
    ku = apply_mask(ku, bits);
    double2 t = ku;
    if (F & SF_SUB_LOAD) {
      const double2 f = ld2(sp, L.f, x - x0);
      t.x -= f.x;
      t.y -= f.y;
    }
    if ((F & SF_REDUCE) && red) {
      s0 += rinv * (uT.x * ku.x + uT.y * ku.y);
      s1 += t.x * t.x + t.y * t.y;
      // plain max (3 instructions, not 7): a NaN reaches s1 = sum t^2 and the
      // finaliser turns the max into NaN (stiff_hook), as np.max would be
      m3 = fmax(m3, fabs(t.x));
      m3 = fmax(m3, fabs(t.y));
      if (F & SF_REDUCE_DOT) {
        const double2 dv = apply_mask(ld2(sp, L.dotv, x - x0), bits);
        s2 += dinv * (dv.x * ku.x + dv.y * ku.y);
      }
    }
    if (F & (SF_D2DIV | SF_D1DIV)) {
      const double ias = 1.0 / as;
      if (F & SF_D2DIV) {
        const double i2 = ias * ias;
        t.x = (bits & 1u) ? t.x : t.x * (km.ikdx2 * i2);
        t.y = (bits & 2u) ? t.y : t.y * (km.ikdy2 * i2);
      } else {
        t.x = (bits & 1u) ? t.x : t.x * (km.ikdx * ias);
        t.y = (bits & 2u) ? t.y : t.y * (km.ikdy * ias);
      }
    }
    if (F & SF_AXPY) {
      // base == input u: node x of the u tile (which starts at node eS)
      const double2 b = (F & SF_BASE_U) ? uT : ld2(sp, L.base, x - x0);
      t.x = b.x - p.beta * t.x;
      t.y = b.y - p.beta * t.y;
    }
    if (p.out) reinterpret_cast<double2*>(p.out)[node] = t;
  };

  // unmasked input (the public apply_stiffness, fea.py:162): fixed DOFs of u
  // read as zero, from the staged mask words of the same node row
  constexpr bool MASK_IN = !(F & SF_IN_MASKED);
  auto mask_in = [&](const unsigned char* sp, int x, double2 v) -> double2 {
    if (!MASK_IN) return v;
    const uint32_t w = reinterpret_cast<const uint32_t*>(sp + L.m)[(x >> 4) - wS];
    return apply_mask(v, (w >> (2 * (x & 15))) & 3u);
  };
  // SF_PROLONG: u(x, r) + M P~ pc, exactly as k_mg_prolong forms it (mg.cu
  // prolong_sum: the same weights and summation order), masked by the fine
  // fixed DOFs of node row r (stage sp)
  constexpr bool PRO = (F & SF_PROLONG) != 0;
  auto prolong_in = [&](const unsigned char* sp, int x, int r, double2 v) -> double2 {
    if (!PRO) return v;
    const int ox = x & 1, oy = r & 1;
    const int c = (x >> 1) - (eS >> 1);  // coarse column within the tile
    const double w = (ox ? 0.5 : 1.0) * (oy ? 0.5 : 1.0);
    const double2* c0 = reinterpret_cast<const double2*>(sp + L.pc);
    const double2* c1 = c0 + kCoarseSlot / 16;
    const double2 v00 = c0[c];
    double sx = w * v00.x, sy = w * v00.y;
    if (ox) {
      const double2 v01 = c0[c + 1];
      sx += w * v01.x;
      sy += w * v01.y;
    }
    if (oy) {
      const double2 v10 = c1[c];
      sx += w * v10.x;
      sy += w * v10.y;
      if (ox) {
        const double2 v11 = c1[c + 1];
        sx += w * v11.x;
        sy += w * v11.y;
      }
    }
    const uint32_t mw = reinterpret_cast<const uint32_t*>(sp + L.m)[(x >> 4) - wS];
    const uint32_t bits = (mw >> (2 * (x & 15))) & 3u;
    if (!(bits & 1u)) v.x += sx;
    if (!(bits & 2u)) v.y += sy;
    return v;
  };

  wait(0);
  double2 uT0 = prolong_in(ring, xA, y0 - 1, mask_in(ring, xA, ld2(ring, L.u, 2 * lane))),
          uT1 = prolong_in(ring, xA + 1, y0 - 1, mask_in(ring, xA + 1, ld2(ring, L.u, 2 * lane + 1))),
          uT2 = prolong_in(ring, xA + 2, y0 - 1, mask_in(ring, xA + 2, ld2(ring, L.u, 2 * lane + 2)));
  // carried bottom-corner terms of the previous element row (o2: BR, o3: BL)
  double2 pA2 = make_double2(0.0, 0.0), pA3 = pA2, pB2 = pA2, pB3 = pA2;
  double aPA = 0.0, aPB = 0.0;
  double* ps = (F & SF_ENERGY) ? p.sens : nullptr;
  // SIMP prefactor eta * v_phys^(eta-1): numpy squares for **2.0 (decided once)
  const double e1 = p.eta - 1.0;
  const int ecase = e1 == 2.0 ? 2 : (e1 == 1.0 ? 1 : 0);
  const int nsteps = nrows - 1;
  // Node sums in the cp.async kernel's order: (left element: o2' + o1) +
  // (right element: o3' + o0), so both kernels agree bit for bit.
#pragma unroll 2
  for (int t = 0; t < nsteps; ++t) {
    const int ey = y0 - 1 + t;
    __syncwarp();  // every lane is done with stage t-1's slot
    if (lane == 0 && t + kS3 - 1 < nrows) issue(t + kS3 - 1);
    wait(t + 1);
    const unsigned char* spT = ring + (t % kS3) * L.size;
    const unsigned char* spB = ring + ((t + 1) % kS3) * L.size;
    const double2 uB0 = prolong_in(spB, xA, ey + 1, mask_in(spB, xA, ld2(spB, L.u, 2 * lane))),
                  uB1 = prolong_in(spB, xA + 1, ey + 1,
                                   mask_in(spB, xA + 1, ld2(spB, L.u, 2 * lane + 1))),
                  uB2 = prolong_in(spB, xA + 2, ey + 1,
                                   mask_in(spB, xA + 2, ld2(spB, L.u, 2 * lane + 2)));
    double2 aAB = ld2(spT, L.a, lane);
    if (F & SF_A_POW) aAB = make_double2(act_pow(aAB.x, p.eta), act_pow(aAB.y, p.eta));
    double2 oA0, oA1, oA2, oA3, oB0, oB1, oB2, oB3;
    double eA = 0.0, eB = 0.0;
    constexpr bool EN = (F & SF_ENERGY) != 0;
    element<GENERIC, EN>(km, aAB.x, uT0, uT1, uB1, uB0, oA0, oA1, oA2, oA3, eA);
    element<GENERIC, EN>(km, aAB.y, uT1, uT2, uB2, uB1, oB0, oB1, oB2, oB3, eB);
    if (EN && ey >= y0) {
      const long long erow = (long long)ey * nx;
      double preA = 1.0, preB = 1.0;
      if (L.vp >= 0) {
        const double2 vp = ld2(spT, L.vp, lane);
        preA = p.eta * (ecase == 2 ? vp.x * vp.x : (ecase == 1 ? vp.x : pow(vp.x, e1)));
        preB = p.eta * (ecase == 2 ? vp.y * vp.y : (ecase == 1 ? vp.y : pow(vp.y, e1)));
      }
      // xA is even and so is erow (even nx), so the pair is one 16-byte store
      if (lane >= 1 && xA + 1 < nx)
        *reinterpret_cast<double2*>(ps + erow + xA) = make_double2(preA * eA, preB * eB);
      else if (lane >= 1 && xA < nx)
        ps[erow + xA] = preA * eA;
    }
    const double2 lB = shfl_up2(add2(pB2, oB1));  // left element of node xA (lane-1's eB)
    const double sAB = aPB + aAB.y;
    const double sL = __shfl_up_sync(0xffffffffu, sAB, 1);
    if (ey >= y0) {
      const bool red = ey >= p.red_y0 && ey < p.red_y1;
      const long long nrow = (long long)ey * NX1;
      const double sA = aPA + aAB.x;
      if (emitA) {
        const double2 k0 = add2(lB, add2(pA3, oA0));
        emit(spT, xA, nrow + xA, make_double2(k0.x * rinv, k0.y * rinv), uT0, sL + sA, red);
      }
      if (emitB) {
        const double2 k1 = add2(add2(pA2, oA1), add2(pB3, oB0));
        emit(spT, xA + 1, nrow + xA + 1, make_double2(k1.x * rinv, k1.y * rinv), uT1, sA + sAB,
             red);
      }
    }
    pA2 = oA2;
    pA3 = oA3;
    pB2 = oB2;
    pB3 = oB3;
    aPA = aAB.x;
    aPB = aAB.y;
    uT0 = uB0;
    uT1 = uB1;
    uT2 = uB2;
  }
  if (y1 == ny) {  // bottom node row: contributions from element row ny-1 only
    const unsigned char* spB = ring + (nsteps % kS3) * L.size;
    const double2 lB = shfl_up2(pB2);
    const double sL = __shfl_up_sync(0xffffffffu, aPB, 1);
    const bool red = ny >= p.red_y0 && ny < p.red_y1;
    const long long nrow = (long long)ny * NX1;
    if (emitA) {
      const double2 k0 = add2(lB, pA3);
      emit(spB, xA, nrow + xA, make_double2(k0.x * rinv, k0.y * rinv), uT0, sL + aPA, red);
    }
    if (emitB) {
      const double2 k1 = add2(pA2, pB3);
      emit(spB, xA + 1, nrow + xA + 1, make_double2(k1.x * rinv, k1.y * rinv), uT1, aPA + aPB,
           red);
    }
  }

  pdl_trigger();
  if (F & SF_REDUCE) {
    __shared__ double tot[4];
    if (grid_reduce4(p.rb, s0, s1, s2, m3, tot)) {
      if (threadIdx.x == 0) stiff_hook(p, tot);
    }
  }
}

// ------------------------------------------------------------------ host ---
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
  });
  return fn;
}

bool enc(CUtensorMap* m, CUtensorMapDataType dt, size_t esz, const void* ptr, uint64_t inner,
         uint64_t rows, uint32_t box) {
  auto fn = encode_fn();
  if (!fn || !ptr || (reinterpret_cast<uintptr_t>(ptr) & 15) || (inner * esz) % 16) return false;
  const cuuint64_t dims[2] = {inner, rows};
  const cuuint64_t strides[1] = {inner * esz};
  const cuuint32_t boxd[2] = {box, 1};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, dt, 2, const_cast<void*>(ptr), dims, strides, boxd, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool GENERIC, int F>
cudaError_t launch3(bsp_grid* g, const StiffArgs& p, const Maps3& tm, cudaStream_t s) {
  constexpr L3 L = layout3(F);
  const size_t sm = kBarBytes + (size_t)kW3 * stages3(F) * L.size;
  cudaError_t e = smem_optin((const void*)k_stiff3<GENERIC, F>, (int)sm);
  if (e != cudaSuccess) return e;
  return launch_k(k_stiff3<GENERIC, F>, g->sgrid3, dim3(32 * kW3), sm, s, p, g->km, tm);
}

template <bool GENERIC>
cudaError_t dispatch3(bsp_grid* g, const StiffArgs& p, const Maps3& tm, cudaStream_t s,
                      bool& handled) {
  handled = true;
  switch (p.flags) {
#define BSP_CASE3(f) \
  case (f):          \
    return launch3<GENERIC, (f)>(g, p, tm, s);
    BSP_STIFF_SHAPES_TMA(BSP_CASE3)
#undef BSP_CASE3
    default:
      handled = false;
      return cudaSuccess;
  }
}

}  // namespace

// TMA path: returns true (with *err) if it launched, false to fall back.
bool launch_stiff_tma(bsp_grid* g, const StiffArgs& p, cudaStream_t s, cudaError_t* err) {
  if (!g->tma_ok || !g->fixrows) return false;
  const int nx = g->nx, ny = g->ny;
  Maps3 tm;
  memset(&tm, 0, sizeof(tm));
  const auto F64 = CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  bool ok = enc(&tm.u, F64, 8, p.u, 2ull * (nx + 1), ny + 1, 130) &&
            enc(&tm.a, F64, 8, p.a, nx, ny, 64) &&
            enc(&tm.m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, g->fixrows, g->fixrow_words, ny + 1, 8);
  if (ok && (p.flags & SF_SUB_LOAD))
    ok = enc(&tm.f, F64, 8, p.rhs ? (const void*)p.rhs : (const void*)g->load, 2ull * (nx + 1),
             ny + 1, 124);
  if (ok && (p.flags & SF_STAGE_VP) && !(p.flags & SF_A_POW))
    ok = enc(&tm.vp, F64, 8, p.vp, nx, ny, 64);
  if (ok && (p.flags & SF_AXPY)) ok = enc(&tm.base, F64, 8, p.base, 2ull * (nx + 1), ny + 1, 124);
  if (ok && (p.flags & SF_REDUCE_DOT))
    ok = enc(&tm.dotv, F64, 8, p.dotv, 2ull * (nx + 1), ny + 1, 124);
  if (ok && (p.flags & SF_PROLONG))
    ok = p.pc && enc(&tm.pc, F64, 8, p.pc, 2ull * (p.nxc + 1), p.nyc + 1, kCoarseBox);
  if (!ok) return false;
  StiffArgs q = p;
  q.R = g->R3;
  if ((q.flags & SF_AXPY) && q.base == q.u && !q.in_div) q.flags |= SF_BASE_U;
  bool handled = false;
  cudaError_t e = g->generic ? dispatch3<true>(g, q, tm, s, handled)
                             : dispatch3<false>(g, q, tm, s, handled);
  if (!handled) return false;
  *err = e;
  return true;
}

}  // namespace bsp
