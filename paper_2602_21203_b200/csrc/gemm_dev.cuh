// gemm_dev.cuh -- device helpers shared by the tensor-core GEMM kernels (gemm.cu, chain.cu):
// per-thread row I/O, warp column sums, and the 64 x 32 bf16 epilogue boxes moved by TMA.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"
#include "gemm.cuh"
#include "tc.cuh"

namespace sq {
namespace gd {

__device__ __forceinline__ int round16(int x) { return (x + 15) & ~15; }

// ---- per-thread row I/O: thread = one tile row, 32 consecutive columns ---------------------
// Vector (16-byte) accesses when the row segment is aligned and complete, predicated scalar
// accesses for tails; global loads are issued together (memory-level parallelism).
__device__ __forceinline__ bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

__device__ __forceinline__ void row_ld_f32(const float* __restrict__ p, int ncv, float (&v)[32]) {
  if (ncv == 32 && al16(p)) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(p) + j);
      v[4 * j] = f.x, v[4 * j + 1] = f.y, v[4 * j + 2] = f.z, v[4 * j + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = j < ncv ? __ldg(p + j) : 0.f;
  }
}
__device__ __forceinline__ void row_ld_bf16(const bf16* __restrict__ p, int ncv, float (&v)[32]) {
  if (ncv == 32 && al16(p)) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(p) + j);
      const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(h[k]);
        v[8 * j + 2 * k] = f.x, v[8 * j + 2 * k + 1] = f.y;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = j < ncv ? __bfloat162float(p[j]) : 0.f;
  }
}
__device__ __forceinline__ void row_st_f32(float* p, int ncv, const float (&v)[32]) {
  if (ncv == 32 && al16(p)) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      reinterpret_cast<float4*>(p)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < ncv) p[j] = v[j];
  }
}
__device__ __forceinline__ void row_st_bf16(bf16* p, int ncv, const float (&v)[32]) {
  if (ncv == 32 && al16(p)) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float f[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) f[k] = v[8 * j + k];
      reinterpret_cast<uint4*>(p)[j] = tc::pack_bf16x8(f);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < ncv) p[j] = __float2bfloat16_rn(v[j]);
  }
}
// Column sums over the warp's 32 rows by a butterfly transpose-reduce (31 shuffles): on return
// lane l holds sum over lanes of v[l].  v is destroyed.
__device__ __forceinline__ float colsum32(float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int j = 0; j < s; ++j) {
      const float send = up ? v[j] : v[j + s];
      const float keep = up ? v[j + s] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

// column sums of 16 values per lane over the warp's 32 rows: every lane returns the sum of
// column (lane & 15) (fixed-order butterfly, then the two 16-lane halves)
__device__ __forceinline__ float colsum16(float (&v)[16]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 8; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int j = 0; j < s; ++j) {
      const float send = up ? v[j] : v[j + s];
      const float keep = up ? v[j + s] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
}

// ---- epilogue staging: per-warp ring of four 64-column x 32-row bf16 boxes (128B swizzle) ---
// A lane owns one row of the box; the tile moves between smem and global memory by TMA.
constexpr int kSlotBytes = 4096;
__device__ __forceinline__ uint32_t box_off(int row, int chunk16) {
  return (uint32_t)(row * 128 + ((chunk16 ^ (row & 7)) << 4));
}
// write 32 values (columns 32c .. 32c+31 of the box) of this lane's row
__device__ __forceinline__ void box_put(uint8_t* slot, int c, const float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float f[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = v[8 * j + k];
    *reinterpret_cast<uint4*>(slot + box_off(lane, 4 * c + j)) = tc::pack_bf16x8(f);
  }
}
// box_put of 32 values already packed as bf16 pairs (w[j] = columns 2j, 2j + 1 of 32c ..)
__device__ __forceinline__ void box_put_pk(uint8_t* slot, int c, const uint32_t (&w)[16]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    *reinterpret_cast<uint4*>(slot + box_off(lane, 4 * c + j)) = make_uint4(w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
}
// two floats -> a bf16 pair (round to nearest even; one paired conversion instead of two scalar
// ones) and the pair's values back as floats (exact)
__device__ __forceinline__ uint32_t bf2_rn(float lo, float hi) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ float bf2_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf2_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
// LayerNorm forward of 32 accumulator columns of this lane's row (DESIGN R-bf16: x_hat rounded
// to bf16 before the affine): xp = bf16 x_hat = (v + bias - mean) rs, yp = bf16 act(x_hat g + beta)
template <bool RELU>
__device__ __forceinline__ void ln_fwd32(const float (&v)[32], const float* sb, const float* sg, const float* sbe,
                                         float mean, float rs, uint32_t (&yp)[16], uint32_t (&xp)[16]) {
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const uint32_t w = bf2_rn((v[2 * j] + sb[2 * j] - mean) * rs, (v[2 * j + 1] + sb[2 * j + 1] - mean) * rs);
    xp[j] = w;
    const float n0 = fmaf(bf2_lo(w), sg[2 * j], sbe[2 * j]), n1 = fmaf(bf2_hi(w), sg[2 * j + 1], sbe[2 * j + 1]);
    yp[j] = RELU ? bf2_rn(fmaxf(n0, 0.f), fmaxf(n1, 0.f)) : bf2_rn(tanh_fast(n0), tanh_fast(n1));
  }
}
__device__ __forceinline__ void box_get(const uint8_t* slot, int c, float (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint4 u = *reinterpret_cast<const uint4*>(slot + box_off(lane, 4 * c + j));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(h[k]);
      v[8 * j + 2 * k] = f.x, v[8 * j + 2 * k + 1] = f.y;
    }
  }
}
// both warps of pair q have written their halves of the box: make it visible to the TMA unit
// and store it from the pair's first warp
__device__ __forceinline__ void pair_store(uint8_t* slot, const void* map, int col, int row, int q, int hh) {
  tc::fence_async_smem();
  tc::named_bar(1 + q, 64);
  if (hh == 0 && (threadIdx.x & 31) == 0) {
    tc::tma_store_2d(map, slot, col, row);
    tc::bulk_commit();
  }
}


}  // namespace gd
}  // namespace sq
