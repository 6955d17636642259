// common.cuh -- small device helpers shared by the libsquint kernels (sm_100a).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <utility>

#define SQ_DEV __device__ __forceinline__

namespace sq {

// Programmatic dependent launch: a kernel launched by launch_pdl may start while its stream
// predecessor is still running; it must call grid_wait() before touching anything a predecessor
// wrote (griddepcontrol.wait: predecessor grids complete, their writes visible) and then
// grid_trigger() so its own dependents may launch.  Both are no-ops without the launch attribute.
SQ_DEV void grid_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
SQ_DEV void grid_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

constexpr int kWarp = 32;

// Adam bias correction 1 / (1 - beta^t) = -1 / expm1(t ln(beta)), ln(beta) = log1p(beta - 1)
// (beta - 1 exact): float, no cancellation
SQ_DEV float bias_corr(float beta, int64_t t) { return -1.f / expm1f((float)t * log1pf(beta - 1.f)); }

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

// Round to bf16 and back.  The LayerNorm forward epilogues of the bf16 path normalise with the x_hat
// they cache in bf16 (n = g bf16(x_hat) + beta), so the backward, which recomputes n from the cache,
// takes exactly the forward's ReLU'(n) decisions (an element whose n is within bf16 rounding of 0
// would otherwise flip its mask and carry a full dY of error into the layer's gradients).
SQ_DEV float bf16_round(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// 1 - tanh(u)^2 without cancellation: sech^2 u = 4 t / (1 + t)^2, t = exp(-2|u|).
// (1 - a*a with a = tanhf(u) loses ~all digits once |u| > 4; log pi's squash term and the
// entropy shift of the C51 target depend on it.)
SQ_DEV float sech2f(float u) {
  const float t = expf(-2.f * fabsf(u));
  const float d = 1.f + t;
  return 4.f * t / (d * d);
}

// Fast variants for the bf16 path's per-element epilogues (results are rounded to bf16 or feed
// bf16 GEMMs): MUFU exp2 + fast divide, ~1e-6 relative error, a handful of instructions.
SQ_DEV float sech2_fast(float u) {
  const float t = __expf(-2.f * fabsf(u));
  const float d = 1.f + t;
  return __fdividef(4.f * t, d * d);
}
SQ_DEV float tanh_fast(float u) {
  const float t = __expf(-2.f * fabsf(u));
  return copysignf(__fdividef(1.f - t, 1.f + t), u);
}

}  // namespace sq

namespace sq {
// Host-side count of kernel launches issued by libsquint (bench "gpu_launches" claim).
// Call right before each launch on stream s: kernel name and its algorithmic work (FLOPs and
// DRAM/L2 bytes by the problem definition, 0 when not tracked) for the bench's roofline.
void note_launch(cudaStream_t s, const char* name, double flops, double bytes);
long launch_count();
// Optional phase instrumentation (squint_set_phase_events): records cudaEvent pairs
// around named phases of squint_update / squint_act / squint_insert on the launch stream.
struct PhaseScope {
  PhaseScope(int phase, int rep, cudaStream_t s);
  ~PhaseScope();
  int idx;
  cudaStream_t s;
};
}  // namespace sq
