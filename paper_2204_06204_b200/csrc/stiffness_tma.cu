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
// strip of R element rows, two rows per step.  Per two rows, ONE lane issues
// 2-D TMA tile loads (cp.async.bulk.tensor) into a 2-3 stage per-warp ring:
//   u (3 node rows of 130 doubles), a (2 x 64), fixed-mask words (3 x 8),
//   plus, per epilogue, f / v_phys / axpy base / dot vector (2 rows each).
// Each stage completes on an mbarrier.  TMA zero-fills every out-of-grid
// coordinate: row -1, row ny+1, column -1, past nx.  So the element loop has no
// bounds logic, and virtual elements with a = 0 contribute nothing.  The
// per-element integer overhead of the per-lane cp.async version (address
// selects, validity predicates, 7 pointer cursors per row) disappears: the
// loop is shared-memory reads, fp64 algebra, one shuffle per node pair and the
// stores.
//
// Layout requirements (checked on the host; otherwise the cp.async kernel
// runs): 16-byte aligned arrays.  The fixed mask is read from its row-aligned
// copy (grid.cuh fixrows).  Odd nx: element rows are not 16-byte multiples,
// which a 2-D tensor map needs, so the element tiles (a, v_phys) are read per
// lane from global memory (two 8-byte loads) and the energies stored as
// scalars; the node tiles (u, mask, f, base, dot, coarse rows) stay on TMA.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "grid.cuh"
#include "q4.cuh"

namespace bsp {

namespace {
constexpr int kW3 = 4;     // warps per CTA
constexpr int kS3max = 3;  // ring stages per warp (two element rows each)
constexpr int kEmit = 62;  // node columns emitted per warp
// Resident CTAs per SM the register budget is sized for.  With one row per
// stage, 4 (128 registers) beat 3 (C5 pfbto 4.52 -> 4.30 ms/iter); with two
// rows per stage the residual spills at 128 and 3 is better (C5 4.15 -> 4.09,
// same box; a deeper ring at 3 CTAs measured neutral).  The generic-Ke
// instances keep their registers (they would spill).
#ifndef BSP_K3_MINB
#define BSP_K3_MINB 3
#endif

struct Maps3 {
  CUtensorMap u, a, m, f, vp, base, dotv, pc;
};

// A ring stage covers the element rows b, b+1 (b = y0 - 1 + 2j for stage j):
// the node-row tiles (u, fixed-mask words, coarse rows) hold 3 rows from row
// b (node row b is the previous stage's last; it is re-staged from L2 so
// that one stage serves both element rows), the element-row tiles (a, v_phys)
// and the emission-row tiles (f, axpy base, dot vector: node rows b, b+1)
// hold 2.  One TMA per tile per two rows, one mbarrier wait per two rows, and
// no barrier between the two rows' instruction streams.
constexpr int kRowU = 1040;  // 65 nodes (130 doubles)
constexpr int kRowA = 512;   // 64 elements
constexpr int kRowM = 32;    // 8 mask words
constexpr int kRowN = 992;   // 62 emitted nodes
// SF_PROLONG: the coarse node rows under the 3 fine node rows, 34 coarse
// nodes each (68 doubles) from coarse column eS/2
constexpr int kCoarseBox = 68;
constexpr int kRowPC = kCoarseBox * 8;

struct L3 {
  int u, a, m, f, vp, base, dotv, pc, size;
  uint32_t tx;  // bytes per stage (TMA counts OOB-filled bytes too)
};

__host__ __device__ constexpr int up128(int b) { return (b + 127) & ~127; }

__host__ __device__ constexpr L3 layout3(int flags) {
  L3 L{0, up128(3 * kRowU), up128(3 * kRowU) + up128(2 * kRowA), -1, -1, -1, -1, -1, 0,
       3 * kRowU + 2 * kRowA + 3 * kRowM};
  int o = L.m + up128(3 * kRowM);
  if (flags & SF_SUB_LOAD) { L.f = o; o += up128(2 * kRowN); L.tx += 2 * kRowN; }
  if ((flags & SF_STAGE_VP) && !(flags & SF_A_POW)) { L.vp = o; o += up128(2 * kRowA); L.tx += 2 * kRowA; }
  if ((flags & SF_STAGE_VP) && (flags & SF_A_POW)) L.vp = L.a;  // the a tile is v_phys
  if ((flags & SF_AXPY) && !(flags & SF_BASE_U)) { L.base = o; o += up128(2 * kRowN); L.tx += 2 * kRowN; }
  if (flags & SF_REDUCE_DOT) { L.dotv = o; o += up128(2 * kRowN); L.tx += 2 * kRowN; }
  if (flags & SF_PROLONG) { L.pc = o; o += up128(3 * kRowPC); L.tx += 3 * kRowPC; }
  L.size = o;
  return L;
}

// stages per warp: as many as fit the per-CTA ring budget, 2..3 (two: the
// stage being computed and the next one in flight).  52 KB per CTA: four CTAs
// of the residual shape fit the SM's 228 KB where registers allow it.
#ifndef BSP_K3_RING
#define BSP_K3_RING 53248
#endif
__host__ __device__ constexpr int stages3(int flags) {
  const int s = BSP_K3_RING / (kW3 * layout3(flags).size);
  return s < 2 ? 2 : (s > kS3max ? kS3max : s);
}

constexpr int kBarBytes = 128;  // kW3 * kS3max mbarriers (8 B), 128-aligned

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

template <bool B>
using bool_c = std::integral_constant<bool, B>;

}  // namespace

template <bool GENERIC, int F, bool ODD>
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
  const int y0 = blockIdx.y * p.R;  // p.R is even: every stage starts on an odd row b
  const int y1 = min(y0 + p.R, ny);
  const int nsteps = y1 - y0 + 1;   // element rows y0-1 .. y1-1
  const int nst = (nsteps + 1) >> 1;
  constexpr bool odd = ODD;  // odd nx: element tiles read per lane (see the header)
  constexpr uint32_t kElemTx = 2 * kRowA + ((L.vp >= 0 && L.vp != L.a) ? 2 * kRowA : 0);
  const uint32_t tx = odd ? L.tx - kElemTx : L.tx;
  const uint32_t bar0 = smem_u32(smem) + wib * kS3 * 8;
  unsigned char* ring = smem + kBarBytes + (size_t)wib * kS3 * L.size;
  const uint32_t ring_s = smem_u32(ring);

  if (lane == 0) {
    for (int s = 0; s < kS3; ++s) mbar_init(bar0 + 8 * s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  auto issue = [&](int j) {  // lane 0: stage j <- rows from b = y0 - 1 + 2j
    const int slot = j % kS3;
    const uint32_t bar = bar0 + 8 * slot;
    const uint32_t d = ring_s + slot * L.size;
    const int b = y0 - 1 + 2 * j;
    mbar_expect_tx(bar, tx);
    tma2d(d + L.u, &tm.u, 2 * eS, b, bar);
    if (!odd) tma2d(d + L.a, &tm.a, eS, b, bar);
    tma2d(d + L.m, &tm.m, wS, b, bar);
    if (L.f >= 0) tma2d(d + L.f, &tm.f, 2 * x0, b, bar);
    if (L.vp >= 0 && L.vp != L.a && !odd) tma2d(d + L.vp, &tm.vp, eS, b, bar);
    if (L.base >= 0) tma2d(d + L.base, &tm.base, 2 * x0, b, bar);
    if (L.dotv >= 0) tma2d(d + L.dotv, &tm.dotv, 2 * x0, b, bar);
    if (L.pc >= 0) tma2d(d + L.pc, &tm.pc, eS, b >> 1, bar);  // b odd: coarse rows (b-1)/2 ..
  };
  auto wait = [&](int j) { mbar_wait(bar0 + 8 * (j % kS3), (j / kS3) & 1); };

  if (lane == 0)
    for (int j = 0; j < kS3 && j < nst; ++j) issue(j);

  // residual shapes (SF_SUB_LOAD) never scale their input (launch_stiff
  // refuses in_div with them): the 1.0 factors fold away at compile time
  constexpr bool SCALES = !(F & SF_SUB_LOAD);
  const double rinv = (SCALES && p.in_div) ? 1.0 / *p.in_div : 1.0;
  const double dinv = (SCALES && p.dot_div) ? 1.0 / *p.dot_div : 1.0;
  const int xA = eS + 2 * lane;  // this lane's node columns xA, xA+1, xA+2
  const bool emitA = lane >= 1 && xA <= nx;
  const bool emitB = lane >= 1 && xA + 1 <= nx;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, m3 = -INFINITY;

  // fixed-mask bits of node x in mask-tile row i (node row b + i)
  auto mbits = [&](const unsigned char* sp, int i, int x) -> uint32_t {
    const uint32_t w = reinterpret_cast<const uint32_t*>(sp + L.m + i * kRowM)[(x >> 4) - wS];
    return (w >> (2 * (x & 15))) & 3u;
  };

  // epilogue of one emitted node of emission row i: ku (already scaled),
  // top-row u, a-sum.  `ok`: this lane emits the node; `red`: the row is in
  // the reduction rows.  Branch-free but for the stores.  G: the emission
  // tiles are read from global memory (the grid's last node row, which the
  // 2-row emission tiles of its stage may not hold).
  auto emit = [&](const unsigned char* sp, int i, int x, long long node, double2 ku, double2 uT,
                  double as, bool ok, bool red, auto g_c) {
    constexpr bool G = decltype(g_c)::value;
    const uint32_t bits = mbits(sp, i, x);
    ku = apply_mask(ku, bits);
    double2 t = ku;
    const double2 z2 = make_double2(0.0, 0.0);
    if (F & SF_SUB_LOAD) {
      const double2* fsrc = p.rhs ? p.rhs : p.g.load;
      const double2 f = G ? (ok ? fsrc[node] : z2) : ld2(sp, L.f + i * kRowN, x - x0);
      t.x -= f.x;
      t.y -= f.y;
    }
    if (F & SF_REDUCE) {
      const bool r = red && ok;
      if constexpr (!(F & SF_RED_NOS0)) {
        const double n0 = s0 + rinv * (uT.x * ku.x + uT.y * ku.y);
        s0 = r ? n0 : s0;
      }
      const double n1 = s1 + (t.x * t.x + t.y * t.y);
      s1 = r ? n1 : s1;
      if constexpr (!(F & SF_RED_NOMAX)) {
        // plain max (3 instructions, not 7): a NaN reaches s1 = sum t^2 and
        // the finaliser turns the max into NaN (stiff_hook), as np.max would
        const double n3 = fmax(fmax(m3, fabs(t.x)), fabs(t.y));
        m3 = r ? n3 : m3;
      }
      if (F & SF_REDUCE_DOT) {
        const double2 dv = apply_mask(G ? (ok ? p.dotv[node] : z2) : ld2(sp, L.dotv + i * kRowN, x - x0),
                                      bits);
        const double n2 = s2 + dinv * (dv.x * ku.x + dv.y * ku.y);
        s2 = r ? n2 : s2;
      }
    }
    if (F & (SF_D2DIV | SF_D1DIV)) {
      const double ias = rcp_pos(as);
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
      const double2 b = (F & SF_BASE_U) ? uT
                        : (G ? (ok ? p.base[node] : z2) : ld2(sp, L.base + i * kRowN, x - x0));
      t.x = b.x - p.beta * t.x;
      t.y = b.y - p.beta * t.y;
    }
    if (ok && p.out) reinterpret_cast<double2*>(p.out)[node] = t;
  };

  // unmasked input (the public apply_stiffness, fea.py:162): fixed DOFs of u
  // read as zero, from the staged mask words of the same node row
  constexpr bool MASK_IN = !(F & SF_IN_MASKED);
  // SF_PROLONG: u(x, r) + M P~ pc, exactly as k_mg_prolong forms it (mg.cu
  // prolong_sum: the same weights and summation order), masked by the fine
  // fixed DOFs of node row r; coarse tile row ci holds coarse row r >> 1
  constexpr bool PRO = (F & SF_PROLONG) != 0;
  // node x of node row b + i (u tile row i, element column index idx)
  auto load_u = [&](const unsigned char* sp, int i, int b, int x, int idx) -> double2 {
    double2 v = ld2(sp, L.u + i * kRowU, idx);
    if (!MASK_IN && !PRO) return v;
    const uint32_t bits = mbits(sp, i, x);
    if (MASK_IN) v = apply_mask(v, bits);
    if (PRO) {
      const int r = b + i;
      const int ox = x & 1, oy = r & 1;
      const int c = (x >> 1) - (eS >> 1);  // coarse column within the tile
      const double w = (ox ? 0.5 : 1.0) * (oy ? 0.5 : 1.0);
      const double2* c0 =
          reinterpret_cast<const double2*>(sp + L.pc + ((r >> 1) - (b >> 1)) * kRowPC);
      const double2* c1 = c0 + kRowPC / 16;
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
      if (!(bits & 1u)) v.x += sx;
      if (!(bits & 2u)) v.y += sy;
    }
    return v;
  };

  // element pair (eS + 2 lane, +1) of element row ey from global memory
  // (odd nx): zero outside the grid, as TMA's out-of-bounds fill
  auto ld_elem2 = [&](const double* arr, int ey) -> double2 {
    const int e0 = eS + 2 * lane;
    double2 r = make_double2(0.0, 0.0);
    if (ey >= 0 && ey < ny) {
      const double* row = arr + (long long)ey * nx;
      if (e0 >= 0 && e0 < nx) r.x = __ldg(row + e0);
      if (e0 + 1 >= 0 && e0 + 1 < nx) r.y = __ldg(row + e0 + 1);
    }
    return r;
  };

  double2 uT0, uT1, uT2;  // top node row of the current element row
  // carried bottom-corner terms of the previous element row (o2: BR, o3: BL)
  double2 pA2 = make_double2(0.0, 0.0), pA3 = pA2, pB2 = pA2, pB3 = pA2;
  double aPA = 0.0, aPB = 0.0;
  double* ps = (F & SF_ENERGY) ? p.sens : nullptr;
  // SIMP prefactor eta * v_phys^(eta-1): numpy squares for **2.0 (decided once)
  const double e1 = p.eta - 1.0;
  const int ecase = e1 == 2.0 ? 2 : (e1 == 1.0 ? 1 : 0);
  constexpr bool EN = (F & SF_ENERGY) != 0;

  // Element row ey = b + i of stage sp: its elements, energies and (EMIT) the
  // nodes of its top node row.  Node sums in the cp.async kernel's order:
  // (left element: o2' + o1) + (right element: o3' + o0), so both kernels
  // agree bit for bit.
  // odd nx: the element pairs of the stage's two rows, loaded one stage
  // ahead (the element tiles' TMA prefetch, in registers): eA[i] / eV[i]
  double2 eA[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)}, eV[2] = {eA[0], eA[1]};
  double2 nA[2] = {eA[0], eA[1]}, nV[2] = {eA[0], eA[1]};
  constexpr bool SEP_VP = (F & SF_ENERGY) && L.vp >= 0 && L.vp != L.a;
  auto prefetch = [&](int b, double2 (&oa)[2], double2 (&ov)[2]) {
    oa[0] = ld_elem2(p.a, b);
    oa[1] = ld_elem2(p.a, b + 1);
    if (SEP_VP) {
      ov[0] = ld_elem2(p.vp, b);
      ov[1] = ld_elem2(p.vp, b + 1);
    }
  };
  auto step = [&](const unsigned char* sp, int i, int b, auto emit_c) {
    constexpr bool EMIT = decltype(emit_c)::value;
    const int ey = b + i;
    const double2 uB0 = load_u(sp, i + 1, b, xA, 2 * lane),
                  uB1 = load_u(sp, i + 1, b, xA + 1, 2 * lane + 1),
                  uB2 = load_u(sp, i + 1, b, xA + 2, 2 * lane + 2);
    const double2 aRaw = odd ? eA[i] : ld2(sp, L.a + i * kRowA, lane);
    double2 aAB = aRaw;
    if (F & SF_A_POW) aAB = make_double2(act_pow(aAB.x, p.eta), act_pow(aAB.y, p.eta));
    double2 oA0, oA1, oA2, oA3, oB0, oB1, oB2, oB3;
    double eA = 0.0, eB = 0.0;
    element<GENERIC, EN>(km, aAB.x, uT0, uT1, uB1, uB0, oA0, oA1, oA2, oA3, eA);
    element<GENERIC, EN>(km, aAB.y, uT1, uT2, uB2, uB1, oB0, oB1, oB2, oB3, eB);
    if constexpr (EN && EMIT) {
      const long long erow = (long long)ey * nx;
      double preA = 1.0, preB = 1.0;
      if (L.vp >= 0) {
        const double2 vp = (L.vp == L.a) ? aRaw : (odd ? eV[i] : ld2(sp, L.vp + i * kRowA, lane));
        preA = p.eta * (ecase == 2 ? vp.x * vp.x : (ecase == 1 ? vp.x : pow(vp.x, e1)));
        preB = p.eta * (ecase == 2 ? vp.y * vp.y : (ecase == 1 ? vp.y : pow(vp.y, e1)));
      }
      const double sA = preA * eA, sB = preB * eB;
      // xA is even and so is erow for even nx: the pair is one 16-byte store
      if (odd) {
        if (lane >= 1 && xA < nx) ps[erow + xA] = sA;
        if (lane >= 1 && xA + 1 < nx) ps[erow + xA + 1] = sB;
      } else if (lane >= 1 && xA + 1 < nx) {
        *reinterpret_cast<double2*>(ps + erow + xA) = make_double2(sA, sB);
      } else if (lane >= 1 && xA < nx) {
        ps[erow + xA] = sA;
      }
      if constexpr ((F & SF_SUM_SENS) != 0) {
        const bool red = ey >= p.red_y0 && ey < p.red_y1;
        const double t = (lane >= 1 && xA < nx ? sA : 0.0) + (lane >= 1 && xA + 1 < nx ? sB : 0.0);
        s2 = red ? s2 + t : s2;
      }
    }
    const double2 lB = shfl_up2(add2(pB2, oB1));  // left element of node xA (lane-1's eB)
    const double sAB = aPB + aAB.y;
    const double sL = __shfl_up_sync(0xffffffffu, sAB, 1);
    if constexpr (EMIT) {
      const bool red = ey >= p.red_y0 && ey < p.red_y1;
      const long long nrow = (long long)ey * NX1;
      const double sA = aPA + aAB.x;
      const double2 k0 = add2(lB, add2(pA3, oA0));
      emit(sp, i, xA, nrow + xA, make_double2(k0.x * rinv, k0.y * rinv), uT0, sL + sA, emitA, red,
           bool_c<false>{});
      const double2 k1 = add2(add2(pA2, oA1), add2(pB3, oB0));
      emit(sp, i, xA + 1, nrow + xA + 1, make_double2(k1.x * rinv, k1.y * rinv), uT1, sA + sAB,
           emitB, red, bool_c<false>{});
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
  };

  // stage 0: element row y0-1 (carried terms only) and y0
  if (odd) {
    prefetch(y0 - 1, eA, eV);
    if (nst > 1) prefetch(y0 + 1, nA, nV);
  }
  wait(0);
  {
    const int b = y0 - 1;
    uT0 = load_u(ring, 0, b, xA, 2 * lane);
    uT1 = load_u(ring, 0, b, xA + 1, 2 * lane + 1);
    uT2 = load_u(ring, 0, b, xA + 2, 2 * lane + 2);
    step(ring, 0, b, bool_c<false>{});
    if (nsteps > 1) step(ring, 1, b, bool_c<true>{});
  }
  for (int j = 1; j < nst; ++j) {
    __syncwarp();  // every lane is done with stage j-1's slot
    if (lane == 0 && j - 1 + kS3 < nst) issue(j - 1 + kS3);
    wait(j);
    const unsigned char* sp = ring + (j % kS3) * L.size;
    const int b = y0 - 1 + 2 * j;
    if (odd) {  // this stage's pairs were loaded a stage ago; start the next
      eA[0] = nA[0];
      eA[1] = nA[1];
      eV[0] = nV[0];
      eV[1] = nV[1];
      if (j + 1 < nst) prefetch(b + 2, nA, nV);
    }
    step(sp, 0, b, bool_c<true>{});
    if (2 * j + 1 < nsteps) step(sp, 1, b, bool_c<true>{});
  }
  if (y1 == ny) {  // bottom node row: contributions from element row ny-1 only
    const int jl = (nsteps - 1) >> 1, il = ((nsteps - 1) & 1) + 1;  // its stage and tile row
    const unsigned char* sp = ring + (jl % kS3) * L.size;
    const double2 lB = shfl_up2(pB2);
    const double sL = __shfl_up_sync(0xffffffffu, aPB, 1);
    const bool red = ny >= p.red_y0 && ny < p.red_y1;
    const long long nrow = (long long)ny * NX1;
    const double2 k0 = add2(lB, pA3);
    emit(sp, il, xA, nrow + xA, make_double2(k0.x * rinv, k0.y * rinv), uT0, sL + aPA, emitA, red,
         bool_c<true>{});
    const double2 k1 = add2(pA2, pB3);
    emit(sp, il, xA + 1, nrow + xA + 1, make_double2(k1.x * rinv, k1.y * rinv), uT1, aPA + aPB,
         emitB, red, bool_c<true>{});
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
         uint64_t rows, uint32_t box, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn || !ptr || (reinterpret_cast<uintptr_t>(ptr) & 15) || (inner * esz) % 16) return false;
  const cuuint64_t dims[2] = {inner, rows};
  const cuuint64_t strides[1] = {inner * esz};
  const cuuint32_t boxd[2] = {box, box_rows};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, dt, 2, const_cast<void*>(ptr), dims, strides, boxd, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool GENERIC, int F, bool ODD>
cudaError_t launch3(bsp_grid* g, const StiffArgs& p, const Maps3& tm, cudaStream_t s) {
  constexpr L3 L = layout3(F);
  const size_t sm = kBarBytes + (size_t)kW3 * stages3(F) * L.size;
  cudaError_t e = smem_optin((const void*)k_stiff3<GENERIC, F, ODD>, (int)sm);
  if (e != cudaSuccess) return e;
  return launch_k(k_stiff3<GENERIC, F, ODD>, g->sgrid3, dim3(32 * kW3), sm, s, p, g->km, tm);
}

// ODD: odd nx (element tiles per lane), a separate instance so that the even
// path carries none of it (a run-time switch cost the even C5 iteration 1.2%);
// odd nx with a generic Ke runs the cp.async kernel
template <bool GENERIC, bool ODD>
cudaError_t dispatch3(bsp_grid* g, const StiffArgs& p, const Maps3& tm, cudaStream_t s,
                      bool& handled) {
  handled = true;
  switch (p.flags) {
#define BSP_CASE3(f) \
  case (f):          \
    return launch3<GENERIC, (f), ODD>(g, p, tm, s);
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
  // box rows: node-row tiles 3, element- and emission-row tiles 2 (layout3)
  const bool odd = (nx & 1) != 0;  // element tiles per lane in the kernel
  bool ok = enc(&tm.u, F64, 8, p.u, 2ull * (nx + 1), ny + 1, 130, 3) &&
            (odd || enc(&tm.a, F64, 8, p.a, nx, ny, 64, 2)) &&
            enc(&tm.m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 4, g->fixrows, g->fixrow_words, ny + 1, 8, 3);
  if (ok && (p.flags & SF_SUB_LOAD))
    ok = enc(&tm.f, F64, 8, p.rhs ? (const void*)p.rhs : (const void*)g->load, 2ull * (nx + 1),
             ny + 1, 124, 2);
  if (ok && (p.flags & SF_STAGE_VP) && !(p.flags & SF_A_POW) && !odd)
    ok = enc(&tm.vp, F64, 8, p.vp, nx, ny, 64, 2);
  if (ok && (p.flags & SF_AXPY)) ok = enc(&tm.base, F64, 8, p.base, 2ull * (nx + 1), ny + 1, 124, 2);
  if (ok && (p.flags & SF_REDUCE_DOT))
    ok = enc(&tm.dotv, F64, 8, p.dotv, 2ull * (nx + 1), ny + 1, 124, 2);
  if (ok && (p.flags & SF_PROLONG))
    ok = p.pc && enc(&tm.pc, F64, 8, p.pc, 2ull * (p.nxc + 1), p.nyc + 1, kCoarseBox, 3);
  if (!ok) return false;
  StiffArgs q = p;
  q.R = g->R3;
  if ((q.flags & SF_AXPY) && q.base == q.u && !q.in_div) q.flags |= SF_BASE_U;
  bool handled = false;
  if (odd && g->generic) return false;
  cudaError_t e = odd ? dispatch3<false, true>(g, q, tm, s, handled)
                      : (g->generic ? dispatch3<true, false>(g, q, tm, s, handled)
                                    : dispatch3<false, false>(g, q, tm, s, handled));
  if (!handled) return false;
  *err = e;
  return true;
}

}  // namespace bsp
