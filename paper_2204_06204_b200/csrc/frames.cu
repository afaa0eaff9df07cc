// Density frames emitted from the device at the snapshot cadence:
//  * the service's streaming payload, v_phys as row-major little-endian float32
//    (reference service/sessions.py:97, `state.v_phys.astype("<f4").tobytes()`);
//  * the PGM pixel map, round-half-up of 255·(1 − v_phys) as uint8
//    (reference outputs.py:21-30, `np.floor(255.0 * (1.0 - v) + 0.5)`).
// Both are byte-identical to the reference's host conversions: cvt.rn.f32.f64
// is numpy's round-to-nearest-even cast, and the pixel arithmetic is spelled
// with explicitly rounded fp64 ops so nvcc cannot contract it into an FMA.
// HBM-bound streams: 8 B read + 4 B (frame) or 1 B (pixels) written per cell.
#include "frames.cuh"
#include "grid.cuh"
#include <algorithm>

namespace bsp {

__global__ void k_frame_f32(const double* __restrict__ v, long long E, float* __restrict__ out) {
  const long long quads = E / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  // 16-byte aligned pointers (cudaMalloc / torch allocations): double2 in, float4 out
  for (long long i = t0; i < quads; i += stride) {
    const double2 a = reinterpret_cast<const double2*>(v)[2 * i];
    const double2 b = reinterpret_cast<const double2*>(v)[2 * i + 1];
    reinterpret_cast<float4*>(out)[i] = make_float4(__double2float_rn(a.x), __double2float_rn(a.y),
                                                    __double2float_rn(b.x), __double2float_rn(b.y));
  }
  for (long long i = 4 * quads + t0; i < E; i += stride) out[i] = __double2float_rn(v[i]);
}

BSP_DEV uint8_t pixel(double v, int& bad) {
  if (v < 0.0 || v > 1.0) bad = 1;
  const double p = floor(__dadd_rn(__dmul_rn(255.0, __dsub_rn(1.0, v)), 0.5));
  return (uint8_t)(int)p;
}

__global__ void k_frame_pixels(const double* __restrict__ v, long long E,
                               uint8_t* __restrict__ out, int* bad_flag) {
  const long long quads = E / 4;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int bad = 0;
  for (long long i = t0; i < quads; i += stride) {
    const double2 a = reinterpret_cast<const double2*>(v)[2 * i];
    const double2 b = reinterpret_cast<const double2*>(v)[2 * i + 1];
    uchar4 q;
    q.x = pixel(a.x, bad);
    q.y = pixel(a.y, bad);
    q.z = pixel(b.x, bad);
    q.w = pixel(b.y, bad);
    reinterpret_cast<uchar4*>(out)[i] = q;
  }
  for (long long i = 4 * quads + t0; i < E; i += stride) out[i] = pixel(v[i], bad);
  if (bad_flag && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(bad_flag, 1);
}

static unsigned frame_blocks(long long E) {
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  long long b = (E / 4 + 255) / 256;
  return (unsigned)std::max<long long>(1, std::min<long long>(b, 8ll * nsm));
}

cudaError_t launch_frame(int kind, const double* v, long long E, void* out, int* bad_flag,
                         cudaStream_t s) {
  if (E <= 0) return cudaSuccess;
  const unsigned nb = frame_blocks(E);
  if (kind == BSP_FRAME_F32)
    k_frame_f32<<<nb, 256, 0, s>>>(v, E, (float*)out);
  else
    k_frame_pixels<<<nb, 256, 0, s>>>(v, E, (uint8_t*)out, bad_flag);
  return cudaGetLastError();
}

}  // namespace bsp

using namespace bsp;

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

extern "C" int bsp_density_frame(const double* d_vphys, long long E, float* d_out, void* stream) {
  if (E < 0) return set_error(BSP_EINVAL, "negative length");
  if (E > 0 && (!d_vphys || !d_out)) return set_error(BSP_EINVAL, "null argument");
  if (E > 0 && (!aligned16(d_vphys) || !aligned16(d_out)))
    return set_error(BSP_EINVAL, "frame buffers must be 16-byte aligned");
  BSP_CU(launch_frame(BSP_FRAME_F32, d_vphys, E, d_out, nullptr, (cudaStream_t)stream));
  return BSP_OK;
}

extern "C" int bsp_density_pixels(const double* d_vphys, long long E, uint8_t* d_out, int* d_bad,
                                  void* stream) {
  if (E < 0) return set_error(BSP_EINVAL, "negative length");
  if (E > 0 && (!d_vphys || !d_out)) return set_error(BSP_EINVAL, "null argument");
  if (E > 0 && (!aligned16(d_vphys) || !aligned16(d_out)))
    return set_error(BSP_EINVAL, "frame buffers must be 16-byte aligned");
  BSP_CU(launch_frame(BSP_FRAME_PGM, d_vphys, E, d_out, d_bad, (cudaStream_t)stream));
  return BSP_OK;
}
