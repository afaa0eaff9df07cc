#pragma once
#include "common.cuh"
#include "bisimp_b200.h"

namespace bsp {
// kind: BSP_FRAME_F32 (float out[E]) or BSP_FRAME_PGM (uint8 out[E]; *bad_flag |= 1
// when a value lies outside [0, 1]).  Pointers 16-byte aligned.
cudaError_t launch_frame(int kind, const double* v, long long E, void* out, int* bad_flag,
                         cudaStream_t s);
}  // namespace bsp
