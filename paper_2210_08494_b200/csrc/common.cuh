// Shared device helpers for the bkfac library (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define BKFAC_DEV __device__ __forceinline__

namespace bkfac {

// per-factor device status word bits
enum : int {
  ST_CHOL_DROP = 1,        // info: a Cholesky pivot was dropped (rank-deficient residual)
  ST_NONFINITE = 1 << 8,   // error: NaN/Inf seen in the eigensolver input
  ST_EIG_FAIL = 1 << 9,    // error: eigensolver did not converge / produced non-finite
  ST_BAD_INDEX = 1 << 10,  // error: a light-correction column index outside [0, r)
  ST_ERROR_MASK = 0xff00,
};

BKFAC_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
BKFAC_DEV double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum; `red` must hold >= 32 floats of shared memory. All threads get the result.
BKFAC_DEV float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.f;
  if (warp == 0) t = warp_sum(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  float r = red[0];
  __syncthreads();
  return r;
}

BKFAC_DEV double block_sum_d(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum_d(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = (threadIdx.x < nw) ? red[threadIdx.x] : 0.0;
  if (warp == 0) t = warp_sum_d(t);
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  double r = red[0];
  __syncthreads();
  return r;
}

inline int ceil_div(long a, long b) { return (int)((a + b - 1) / b); }

}  // namespace bkfac
