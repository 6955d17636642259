// common.cuh -- small device helpers shared by the libsquint kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define SQ_DEV __device__ __forceinline__

namespace sq {

constexpr int kWarp = 32;

SQ_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
SQ_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Deterministic block-wide sum (fixed tree order).  `red` has >= blockDim.x/32 floats.
SQ_DEV float block_sum(float v, float* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  float t = 0.f;
  if (wid == 0) {
    t = lane < nw ? red[lane] : 0.f;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

SQ_DEV bool is_finite(float x) { return isfinite(x); }

}  // namespace sq
