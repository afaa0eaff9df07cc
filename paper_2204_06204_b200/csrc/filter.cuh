#pragma once
#include "common.cuh"

namespace bsp {

constexpr int kMaxTaps = 31;

struct DevState;

struct FilterTaps {
  double w[kMaxTaps];
  double cum[kMaxTaps + 1];  // cum[k] = w[0] + ... + w[k-1]: O(1) boundary masses
  int size, r;
  // size > kMaxTaps (any odd FilterSpec.size, filtering.py:24-27): the taps
  // live on the device, dw[0..size) then cum dw[size..2 size], and the two
  // passes run as separate kernels through an (rows x nx) scratch `tmp` owned
  // by the caller (the solver allocates it; standalone calls stream-allocate)
  const double* dw;
  double* tmp;
};

struct FilterArgs {
  FilterTaps w;
  int nx, ny;
  const double* in;
  double* out;
  double* act;              // fwd only, nullable: act = out^eta
  double eta;
  const int* gate0;
  // adjoint only, nullable st: reduce sum(out) over active elements -> st->gsum
  DevState* st;
  const uint8_t* active;
  RedBuf rb;
  // row slabs (distributed.cu): the field holds rows [gy0, gy0 + ny) of a
  // grid with gny rows -> the y boundary masses use global rows.  The adjoint
  // reduction covers local rows [red_y0, red_y1) only; with defer_out set the
  // last block stores the partial sum there instead of st->gsum.
  int gy0, gny;
  int red_y0, red_y1;
  double* defer_out;
  int rc;  // rows per CTA chunk (set by launch_filter_kernel)
};

size_t filter_smem_bytes(int r);
int filter_rows_per_chunk(int nx, int ny);
dim3 filter_grid(int nx, int ny, int r);
dim3 filter_grid_max(int nx, int ny);  // upper bound on the CTA count for any radius
cudaError_t launch_filter_kernel(const FilterArgs& fa, int adjoint, cudaStream_t s);

}  // namespace bsp
