#pragma once
#include "common.cuh"
#include "solver_state.cuh"

namespace bsp {
__global__ void k_axpy(const double* x, const double* y, double c, double* out, long long n);
__global__ void k_div_sq(const double* r, const double* d, double* out, long long n);
// out[0] = sum x^2, out[1] = sum x, out[2] = max|x|
__global__ void k_sum(const double* x, long long n, RedBuf rb, double* out);
__global__ void k_mean_sub(const double* g, long long n, const double* sum, double* out);
// Krylov start: norms[0] = sqrt(st->scratch[0]), count/stop/rank reset
__global__ void k_kry_init(DevState* st);
}  // namespace bsp
