// optim.cu -- temperature step (Algorithm 1 L17 with the sign of Q17), fused Adam (Q26),
// Polyak (Algorithm 1 L24, Q28) and the per-update metrics row.  All reductions are fixed
// order so results are bitwise reproducible and identical across data-parallel replicas.
#include <cuda_runtime.h>

#include <cstring>

#include "common.cuh"
#include "optim.cuh"

namespace sq {

namespace {

// Per-thread partial sums of two row vectors over i = tid, tid + blockDim, ... in that order; the
// loads of four strides are issued before their adds (the loop was one dependent L2 round trip per
// stride: ~10 us for B = 4096 on one block).
__device__ __forceinline__ void row_sums2(const float* __restrict__ ra, const float* __restrict__ rb, int B, float& a,
                                          float& b) {
  const int st = blockDim.x;
  int i = threadIdx.x;
  for (; i + 3 * st < B; i += 4 * st) {
    float va[4], vb[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      va[k] = ra[i + k * st];
      vb[k] = rb[i + k * st];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a += va[k];
      b += vb[k];
    }
  }
  for (; i < B; i += st) {
    a += ra[i];
    b += rb[i];
  }
}

__global__ void __launch_bounds__(256) k_row_sums(const float* __restrict__ logp, const float* __restrict__ row_loss,
                                                  int B, float* __restrict__ extras) {
  grid_wait();
  grid_trigger();
  __shared__ float red[32];
  float a = 0.f, b = 0.f;
  row_sums2(logp, row_loss, B, a, b);
  a = block_sum(a, red);
  b = block_sum(b, red);
  if (threadIdx.x == 0) {
    extras[X_SUM_LOGP] = a;
    extras[X_SUM_LQ] = b;
  }
}


__global__ void __launch_bounds__(256) k_scalars(const __grid_constant__ ScalarsArgs a) {
  grid_wait();
  grid_trigger();
  __shared__ float red[32];
  float sl = 0.f, sq = 0.f;
  if (a.compute_sums) {
    for (int i = threadIdx.x; i < a.B; i += blockDim.x) {
      sl += a.logp[i];
      sq += a.row_loss[i];
    }
    sl = block_sum(sl, red);
    sq = block_sum(sq, red);
  }
  if (threadIdx.x != 0) return;
  if (a.compute_sums) {
    a.extras[X_SUM_LOGP] = sl;
    a.extras[X_SUM_LQ] = sq;
  } else {
    sl = a.extras[X_SUM_LOGP];
    sq = a.extras[X_SUM_LQ];
  }
  const float mean_logp = sl * a.inv_btotal;
  const float la = a.log_alpha[0];
  const float alpha0 = expf(la);
  const float loss = -alpha0 * (mean_logp + a.target_entropy);
  const float g = loss;  // d/dlog_alpha of -exp(log_alpha) (...)
  const int64_t t = ++a.step[2];
  const float m = a.beta1 * a.m_alpha[0] + (1.f - a.beta1) * g;
  const float v = a.beta2 * a.v_alpha[0] + (1.f - a.beta2) * g * g;
  const float c1 = bias_corr(a.beta1, t);
  const float c2 = bias_corr(a.beta2, t);
  const float la1 = la - a.lr_alpha * (m * c1) / (sqrtf(v * c2) + a.adam_eps);
  a.m_alpha[0] = m;
  a.v_alpha[0] = v;
  a.log_alpha[0] = la1;
  const float alpha1 = expf(la1);
  a.scal[S_ALPHA1] = alpha1;
  a.scal[S_ALPHA1_SCALE] = alpha1 * a.loss_scale;
  a.scal[S_MEAN_LOGP] = mean_logp;
  a.scal[S_LALPHA] = loss;
  a.scal[S_LQ] = sq;
  if (a.steps_done) return;  // critic / actor steps and corrections already taken (k_target_ce)
  const int64_t tc = ++a.step[0], ta = ++a.step[1];
  a.scal[S_C1_CRITIC] = bias_corr(a.beta1, tc);
  a.scal[S_C2_CRITIC] = bias_corr(a.beta2, tc);
  a.scal[S_C1_ACTOR] = bias_corr(a.beta1, ta);
  a.scal[S_C2_ACTOR] = bias_corr(a.beta2, ta);
}

__global__ void __launch_bounds__(256) k_adam(float4* __restrict__ p, const float4* __restrict__ g,
                                              float4* __restrict__ m, float4* __restrict__ v, int64_t n4, float lr,
                                              float b1, float b2, float eps, const float* __restrict__ c1p,
                                              const float* __restrict__ c2p, float* __restrict__ part) {
  grid_wait();
  grid_trigger();
  __shared__ float red[32];
  const float c1 = c1p[0], c2 = c2p[0];
  float ss = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 gg = g[i], mm = m[i], vv = v[i], pp = p[i];
    float* gf = reinterpret_cast<float*>(&gg);
    float* mf = reinterpret_cast<float*>(&mm);
    float* vf = reinterpret_cast<float*>(&vv);
    float* pf = reinterpret_cast<float*>(&pp);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      ss = fmaf(gf[k], gf[k], ss);
      mf[k] = b1 * mf[k] + (1.f - b1) * gf[k];
      vf[k] = b2 * vf[k] + (1.f - b2) * gf[k] * gf[k];
      pf[k] = pf[k] - lr * (mf[k] * c1) / (sqrtf(vf[k] * c2) + eps);
    }
    m[i] = mm;
    v[i] = vv;
    p[i] = pp;
  }
  if (part) {
    ss = block_sum(ss, red);
    if (threadIdx.x == 0) part[blockIdx.x] = ss;
  }
}

__global__ void __launch_bounds__(256) k_polyak(float* __restrict__ t, const float* __restrict__ o, int64_t n,
                                                float tau) {
  grid_wait();
  grid_trigger();
  const float keep = 1.f - tau;
  const bool vec = ((reinterpret_cast<uintptr_t>(t) | reinterpret_cast<uintptr_t>(o)) & 15) == 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (vec) {
    const int64_t n4 = n / 4;
    float4* t4 = reinterpret_cast<float4*>(t);
    const float4* o4 = reinterpret_cast<const float4*>(o);
    for (int64_t i = i0; i < n4; i += stride) {
      float4 a = t4[i];
      const float4 b = o4[i];
      a.x = keep * a.x + tau * b.x;
      a.y = keep * a.y + tau * b.y;
      a.z = keep * a.z + tau * b.z;
      a.w = keep * a.w + tau * b.w;
      t4[i] = a;
    }
    for (int64_t i = n4 * 4 + i0; i < n; i += stride) t[i] = keep * t[i] + tau * o[i];
  } else {
    for (int64_t i = i0; i < n; i += stride) t[i] = keep * t[i] + tau * o[i];
  }
}

__global__ void __launch_bounds__(256) k_lpi_sums(const float* __restrict__ row_lpi, const float* __restrict__ row_q,
                                                  int B, float* __restrict__ out2) {
  grid_wait();
  grid_trigger();
  __shared__ float red[32];
  float a = 0.f, b = 0.f;
  row_sums2(row_lpi, row_q, B, a, b);
  a = block_sum(a, red);
  b = block_sum(b, red);
  if (threadIdx.x == 0) {
    out2[0] = a;
    out2[1] = b;
  }
}

__global__ void __launch_bounds__(256) k_metrics(const __grid_constant__ MetricsArgs a) {
  grid_wait();
  grid_trigger();
  __shared__ float red[32];
  float lpi = 0.f, q = 0.f, gs = 0.f;
  if (a.reduce_local) {
    for (int i = threadIdx.x; i < a.B; i += blockDim.x) {
      lpi += a.row_lpi[i];
      q += a.row_q[i];
    }
    lpi = block_sum(lpi, red);
    q = block_sum(q, red);
  } else {
    lpi = a.extras2[0];
    q = a.extras2[1];
  }
  const int npart = a.npart > 0 ? a.npart : kAdamBlocks;
  for (int i = threadIdx.x; i < npart; i += blockDim.x) gs += a.sumsq_part[i];
  gs = block_sum(gs, red);
  if (threadIdx.x == 0) {
    const float LQ = a.scal[S_LQ], La = a.scal[S_LALPHA];
    float* o = a.out;
    o[0] = LQ;
    o[1] = lpi;
    o[2] = La;
    o[3] = a.scal[S_ALPHA1];
    o[4] = q * a.inv_btotal;
    o[5] = -a.scal[S_MEAN_LOGP];
    o[6] = sqrtf(gs);
    o[7] = (isfinite(LQ) && isfinite(lpi) && isfinite(La)) ? 0.f : 1.f;
  }
}

// flat index i of a group buffer -> its shadow slot, or -1 (32-bit index math: every group
// buffer is < 2^31 floats)
__device__ __forceinline__ int shadow_slot(const ShadowTable& t, int i) {
  for (int k = 0; k < t.n; ++k) {
    const ShadowEnt& e = t.e[k];
    const int l = i - (int)e.src;
    if (l >= 0 && l < e.rows * e.cols) {
      const int row = l / e.cols, col = l - row * e.cols;
      int cc = col;
      if (e.perm_c > 0) {
        const int ch = col / e.perm_p, pix = col - ch * e.perm_p;
        cc = pix * e.perm_c + ch;
      }
      return (int)e.dst + row * e.ld + cc;
    }
  }
  return -1;
}

// The shadow slots of flat indices i .. i + 3 (i % 4 == 0) after an optimizer step: one entry
// search per float4; the four values go out as one 8-byte store when they sit in one row of a
// plain entry (every entry with cols % 4 == 0), else element by element.
// (base: this table's shadow buffer, or another rank's copy of it -- same layout)
__device__ __forceinline__ void shadow_store4(const ShadowTable& t, __nv_bfloat16* base, int i, const float* f) {
  for (int k = 0; k < t.n; ++k) {
    const ShadowEnt& e = t.e[k];
    const int l = i - (int)e.src;
    if (l >= 0 && l < e.rows * e.cols) {
      if (e.perm_c == 0 && ((e.cols | l | e.ld | (int)e.dst) & 3) == 0) {
        const int row = l / e.cols, col = l - row * e.cols;
        const __nv_bfloat162 lo = __floats2bfloat162_rn(f[0], f[1]), hi = __floats2bfloat162_rn(f[2], f[3]);
        uint2 w;
        w.x = *reinterpret_cast<const uint32_t*>(&lo);
        w.y = *reinterpret_cast<const uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(base + e.dst + (int64_t)row * e.ld + col) = w;
        return;
      }
      break;
    }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int sl = shadow_slot(t, i + k);
    if (sl >= 0) base[sl] = __float2bfloat16_rn(f[k]);
  }
}
__device__ __forceinline__ void shadow_store4(const ShadowTable& t, int i, const float* f) {
  shadow_store4(t, t.base, i, f);
}

// One group's shadow refresh.  Work unit = (row, 128-column segment) of an entry, one warp per
// unit: a float4 per lane (-> 4 bf16) for plain entries; for the projection weight's (channel,
// pixel) -> (pixel, channel) column permutation, 4 gathered elements per lane in destination order,
// all loads issued before the stores.  (The element-wise version spent two runtime divisions per
// element and walked the entries one after another.)
__device__ __forceinline__ void shadow_rows(const float* __restrict__ master, const ShadowTable& t, int gw, int nw) {
  const int lane = threadIdx.x & 31;
  const bool m16 = (reinterpret_cast<uintptr_t>(master) & 15) == 0;
  int ubase = 0;
  for (int k = 0; k < t.n; ++k) {
    const ShadowEnt& e = t.e[k];
    const int nseg = (e.cols + 127) >> 7, units = e.rows * nseg;
    int u0 = (gw - ubase) % nw;
    if (u0 < 0) u0 += nw;
    const bool vec = e.perm_c == 0 && m16 && ((e.cols | (int)e.src | e.ld | (int)e.dst) & 3) == 0;
    for (int u = u0; u < units; u += nw) {
      const int row = u / nseg, c0 = (u - row * nseg) << 7;
      const float* src = master + e.src + (int64_t)row * e.cols;
      __nv_bfloat16* dst = t.base + e.dst + (int64_t)row * e.ld;
      if (vec) {
        const int c = c0 + 4 * lane;
        if (c < e.cols) {
          const float4 v = *reinterpret_cast<const float4*>(src + c);
          const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
          uint2 w;
          w.x = *reinterpret_cast<const uint32_t*>(&lo);
          w.y = *reinterpret_cast<const uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(dst + c) = w;
        }
      } else {
        float v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int cc = c0 + lane + 32 * i;
          v[i] = 0.f;
          if (cc < e.cols) {
            int sc = cc;
            if (e.perm_c > 0) {
              const int pix = cc / e.perm_c, ch = cc - pix * e.perm_c;
              sc = ch * e.perm_p + pix;
            }
            v[i] = src[sc];
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int cc = c0 + lane + 32 * i;
          if (cc < e.cols) dst[cc] = __float2bfloat16_rn(v[i]);
        }
      }
    }
    ubase += units;
  }
}

__global__ void __launch_bounds__(256) k_shadow(const float* __restrict__ master, const __grid_constant__ ShadowTable t) {
  grid_wait();
  grid_trigger();
  shadow_rows(master, t, blockIdx.x * 8 + (threadIdx.x >> 5), gridDim.x * 8);
}

__global__ void __launch_bounds__(256) k_adam_sh(float4* __restrict__ p, const float4* __restrict__ g,
                                                 float4* __restrict__ m, float4* __restrict__ v, int64_t n4, float lr,
                                                 float b1, float b2, float eps, const float* __restrict__ c1p,
                                                 const float* __restrict__ c2p, float* __restrict__ part,
                                                 const __grid_constant__ ShadowTable t, int base, int grad_perm) {
  grid_wait();
  grid_trigger();
  __shared__ float red[32];
  const float c1 = c1p[0], c2 = c2p[0];
  // grad_perm: the gradient of a shadow entry with a column permutation (the projection weight)
  // is stored in the shadow's (pixel-major) column order, row pitch = cols: gathered here
  int pe = -1;
  int64_t plo = 0, phi = 0;
  if (grad_perm)
    for (int k = 0; k < t.n; ++k)
      if (t.e[k].perm_c > 0) {
        pe = k;
        plo = t.e[k].src - base;
        phi = plo + (int64_t)t.e[k].rows * t.e[k].cols;
      }
  const float* gs = reinterpret_cast<const float*>(g);
  float ss = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 gg, mm = m[i], vv = v[i], pp = p[i];
    if (pe >= 0 && 4 * i >= plo && 4 * i < phi) {
      const ShadowEnt& e = t.e[pe];
      float* gf = reinterpret_cast<float*>(&gg);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int l = (int)(4 * i + k - plo), row = l / e.cols, col = l - row * e.cols;
        const int ch = col / e.perm_p, pix = col - ch * e.perm_p;
        gf[k] = gs[plo + (int64_t)row * e.cols + pix * e.perm_c + ch];
      }
    } else {
      gg = g[i];
    }
    float* gf = reinterpret_cast<float*>(&gg);
    float* mf = reinterpret_cast<float*>(&mm);
    float* vf = reinterpret_cast<float*>(&vv);
    float* pf = reinterpret_cast<float*>(&pp);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      ss = fmaf(gf[k], gf[k], ss);
      mf[k] = b1 * mf[k] + (1.f - b1) * gf[k];
      vf[k] = b2 * vf[k] + (1.f - b2) * gf[k] * gf[k];
      pf[k] = pf[k] - lr * (mf[k] * c1) / (sqrtf(vf[k] * c2) + eps);
    }
    m[i] = mm;
    v[i] = vv;
    p[i] = pp;
    if (t.n) shadow_store4(t, base + (int)(4 * i), pf);
  }
  if (part) {
    ss = block_sum(ss, red);
    if (threadIdx.x == 0) part[blockIdx.x] = ss;
  }
}

__global__ void __launch_bounds__(256) k_polyak_sh(float4* __restrict__ t4, const float4* __restrict__ o4, int64_t n4,
                                                   float tau, const __grid_constant__ ShadowTable t) {
  grid_wait();
  grid_trigger();
  const float keep = 1.f - tau;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = t4[i];
    const float4 b = o4[i];
    a.x = keep * a.x + tau * b.x;
    a.y = keep * a.y + tau * b.y;
    a.z = keep * a.z + tau * b.z;
    a.w = keep * a.w + tau * b.w;
    t4[i] = a;
    if (t.n) shadow_store4(t, (int)(4 * i), reinterpret_cast<const float*>(&a));
  }
}

}  // namespace

// up to three (master, table) pairs in one launch (blockIdx.y = pair)
struct ShadowJobs {
  const float* master[3];
  ShadowTable t[3];
};
__global__ void __launch_bounds__(256) k_shadow3(const __grid_constant__ ShadowJobs j) {
  grid_wait();
  grid_trigger();
  shadow_rows(j.master[blockIdx.y], j.t[blockIdx.y], blockIdx.x * 8 + (threadIdx.x >> 5), gridDim.x * 8);
}

__global__ void __launch_bounds__(256) k_split_sum(const __grid_constant__ SplitSumJobs j) {
  grid_wait();
  grid_trigger();
  const int job = blockIdx.y;
  const int n = j.n[job];
  const float* src = j.src[job];
  float* dst = j.dst[job];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    float acc = src[i];
    for (int r = 1; r < j.nsplit; ++r) acc += src[(int64_t)r * n + i];
    dst[i] = acc;
  }
}

int launch_split_sum(const SplitSumJobs& j, cudaStream_t s) {
  if (j.njobs <= 0) return 0;
  note_launch(s, "k_split_sum", 0, 0);
  launch_pdl(k_split_sum, dim3(148, j.njobs), dim3(256), 0, s, j);
  return (int)cudaGetLastError();
}

int launch_shadow3(const float* const master[3], const ShadowTable* const t[3], cudaStream_t s) {
  ShadowJobs j;
  memset(&j, 0, sizeof(j));
  for (int i = 0; i < 3; ++i) {
    j.master[i] = master[i];
    if (t[i]) j.t[i] = *t[i];
  }
  note_launch(s, "k_shadow", 0, 0);
  launch_pdl(k_shadow3, dim3(148, 3), dim3(256), 0, s, j);
  return (int)cudaGetLastError();
}

int launch_shadow(const float* master, const ShadowTable& t, cudaStream_t s) {
  if (t.n == 0) return 0;
  note_launch(s, "k_shadow", 0, 0); launch_pdl(k_shadow, dim3(148 * 2), dim3(256), 0, s, master, t);
  return (int)cudaGetLastError();
}

int launch_adam_shadow(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                       float eps, const float* c1, const float* c2, float* sumsq_part, const ShadowTable* t,
                       cudaStream_t s, int64_t base, int nblocks, int grad_perm) {
  ShadowTable none;
  memset(&none, 0, sizeof(none));
  note_launch(s, "k_adam", 0, 28.0 * (double)n);
  launch_pdl(k_adam_sh, dim3(nblocks), dim3(256), 0, s, reinterpret_cast<float4*>(p), reinterpret_cast<const float4*>(g),
                                    reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), n / 4, lr, b1, b2, eps,
                                    c1, c2, sumsq_part, t ? *t : none, (int)base, grad_perm);
  return (int)cudaGetLastError();
}

__global__ void __launch_bounds__(256) k_stage_pinned(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                                      size_t bytes) {
  grid_wait();
  grid_trigger();
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x, nt = (size_t)gridDim.x * blockDim.x;
  if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
    const size_t n16 = bytes / 16;
    for (size_t i = tid; i < n16; i += nt)
      reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    for (size_t i = n16 * 16 + tid; i < bytes; i += nt) dst[i] = src[i];
  } else {
    for (size_t i = tid; i < bytes; i += nt) dst[i] = src[i];
  }
}

int launch_stage_pinned(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  size_t blocks = (bytes / 16 + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148) blocks = 148;
  note_launch(s, "k_stage_pinned", 0, (double)bytes);
  launch_pdl(k_stage_pinned, dim3((unsigned)blocks), dim3(256), 0, s, reinterpret_cast<uint8_t*>(dst),
             reinterpret_cast<const uint8_t*>(src), bytes);
  return (int)cudaGetLastError();
}

int launch_polyak_shadow(float* target, const float* online, int64_t n, float tau, const ShadowTable* t,
                         cudaStream_t s) {
  if (n == 0) return 0;
  ShadowTable none;
  memset(&none, 0, sizeof(none));
  int64_t blocks = (n / 4 + 255) / 256;
  if (blocks > 148 * 4) blocks = 148 * 4;
  note_launch(s, "k_polyak", 0, 12.0 * (double)n);
  launch_pdl(k_polyak_sh, dim3((unsigned)blocks), dim3(256), 0, s, reinterpret_cast<float4*>(target), reinterpret_cast<const float4*>(online),
                                               n / 4, tau, t ? *t : none);
  return (int)cudaGetLastError();
}

int launch_row_sums(const float* logp, const float* row_loss, int B, float* extras, cudaStream_t s) {
  note_launch(s, "k_row_sums", 0, 0); launch_pdl(k_row_sums, dim3(1), dim3(256), 0, s, logp, row_loss, B, extras);
  return (int)cudaGetLastError();
}

int launch_scalars(const ScalarsArgs& a, cudaStream_t s) {
  note_launch(s, "k_scalars", 0, 0); launch_pdl(k_scalars, dim3(1), dim3(256), 0, s, a);
  return (int)cudaGetLastError();
}

int launch_adam(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2, float eps,
                const float* c1, const float* c2, float* sumsq_part, cudaStream_t s) {
  note_launch(s, "k_adam", 0, 28.0 * (double)n); launch_pdl(k_adam, dim3(kAdamBlocks), dim3(256), 0, s, reinterpret_cast<float4*>(p), reinterpret_cast<const float4*>(g),
                                     reinterpret_cast<float4*>(m), reinterpret_cast<float4*>(v), n / 4, lr, b1, b2,
                                     eps, c1, c2, sumsq_part);
  return (int)cudaGetLastError();
}

int launch_polyak(float* target, const float* online, int64_t n, float tau, cudaStream_t s) {
  if (n == 0) return 0;
  int64_t blocks = (n / 4 + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 8) blocks = 148 * 8;
  note_launch(s, "k_polyak", 0, 12.0 * (double)n); launch_pdl(k_polyak, dim3((unsigned)blocks), dim3(256), 0, s, target, online, n, tau);
  return (int)cudaGetLastError();
}

int launch_metrics(const MetricsArgs& a, cudaStream_t s) {
  note_launch(s, "k_metrics", 0, 0); launch_pdl(k_metrics, dim3(1), dim3(256), 0, s, a);
  return (int)cudaGetLastError();
}

int launch_lpi_sums(const float* row_lpi, const float* row_q, int B, float* out2, cudaStream_t s) {
  note_launch(s, "k_lpi_sums", 0, 0); launch_pdl(k_lpi_sums, dim3(1), dim3(256), 0, s, row_lpi, row_q, B, out2);
  return (int)cudaGetLastError();
}

// ---- f1: peer-memory gradient all-reduce fused with a sharded Adam ----
// Cross-rank barrier: thread 0 adds 1 to its slot of every peer's arrival counters (release, system
// scope, over NVLink), then waits until every peer's arrival count in its own counters reaches its
// epoch + 1 (acquire).  One block; the next kernel on the stream starts after it completes.
namespace {
__device__ __forceinline__ void red_relaxed_sys(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__global__ void __launch_bounds__(256) k_dp_sync(const __grid_constant__ DpSync a) {
  grid_wait();
  grid_trigger();
  __shared__ float red[32];
  if (a.ra) {
    // this rank's row sums into its own tail (k_row_sums / k_lpi_sums, same block and order)
    float x = 0.f, y = 0.f;
    row_sums2(a.ra, a.rb, a.B, x, y);
    x = block_sum(x, red);
    y = block_sum(y, red);
    if (threadIdx.x == 0) {
      a.tail_mine[0] = x;
      a.tail_mine[1] = y;
    }
  }
  if (threadIdx.x == 0) {
    const unsigned e = a.own[kDpMaxRanks] + 1;
    // one release fence orders everything this rank wrote before (its gradients and tail, its
    // stores into the peers) ahead of the arrival counts; one acquire fence after the spin
    fence_acq_rel_sys();
    for (int q = 0; q < a.G; ++q) red_relaxed_sys(a.flag[q] + a.rank, 1u);
    for (int q = 0; q < a.G; ++q)
      while (ld_relaxed_sys(a.own + q) < e) {
      }
    fence_acq_rel_sys();
    a.own[kDpMaxRanks] = e;
  }
  __syncthreads();
  // the reduced row-sum tail (alpha step, metrics), summed in rank order
  for (int t = threadIdx.x; t < a.ntail; t += blockDim.x) {
    float acc = __ldcg(a.tail[0] + t);
    for (int q = 1; q < a.G; ++q) acc += __ldcg(a.tail[q] + t);
    a.tail_out[t] = acc;
  }
}

// This rank's slice [lo4, hi4) (float4 units) of one parameter group: g = sum over ranks (rank
// order, read from the peers' gradient buffers over NVLink), Adam (the arithmetic of k_adam_sh),
// the stepped parameters (and their bf16 shadow entries) stored into every rank's copy, sum(g^2)
// per block into every rank's
// partial buffer at [rank * gridDim.x + block].  m and v: this rank's slice only is ever touched.
__global__ void __launch_bounds__(256) k_dp_adam(const __grid_constant__ DpAdam d, float4* __restrict__ m,
                                                 float4* __restrict__ v, float lr, float b1, float b2, float eps,
                                                 const float* __restrict__ c1p, const float* __restrict__ c2p,
                                                 const __grid_constant__ ShadowTable t, int grad_perm) {
  grid_wait();
  grid_trigger();
  __shared__ float red[32];
  const float c1 = c1p[0], c2 = c2p[0];
  int pe = -1;
  int64_t plo = 0, phi = 0;
  if (grad_perm)
    for (int k = 0; k < t.n; ++k)
      if (t.e[k].perm_c > 0) {
        pe = k;
        plo = t.e[k].src;
        phi = plo + (int64_t)t.e[k].rows * t.e[k].cols;
      }
  float ss = 0.f;
  for (int64_t i = d.lo4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < d.hi4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 gg;
    float* gf = reinterpret_cast<float*>(&gg);
    if (pe >= 0 && 4 * i >= plo && 4 * i < phi) {
      const ShadowEnt& e = t.e[pe];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int l = (int)(4 * i + k - plo), row = l / e.cols, col = l - row * e.cols;
        const int ch = col / e.perm_p, pix = col - ch * e.perm_p;
        const int64_t j = plo + (int64_t)row * e.cols + pix * e.perm_c + ch;
        float acc = __ldcg(d.g[0] + j);
        for (int q = 1; q < d.G; ++q) acc += __ldcg(d.g[q] + j);
        gf[k] = acc;
      }
    } else {
      gg = __ldcg(reinterpret_cast<const float4*>(d.g[0]) + i);
      for (int q = 1; q < d.G; ++q) {
        const float4 o = __ldcg(reinterpret_cast<const float4*>(d.g[q]) + i);
        gg.x += o.x;
        gg.y += o.y;
        gg.z += o.z;
        gg.w += o.w;
      }
    }
    float4 mm = m[i], vv = v[i], pp = reinterpret_cast<const float4*>(d.p[d.rank])[i];
    float* mf = reinterpret_cast<float*>(&mm);
    float* vf = reinterpret_cast<float*>(&vv);
    float* pf = reinterpret_cast<float*>(&pp);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      ss = fmaf(gf[k], gf[k], ss);
      mf[k] = b1 * mf[k] + (1.f - b1) * gf[k];
      vf[k] = b2 * vf[k] + (1.f - b2) * gf[k] * gf[k];
      pf[k] = pf[k] - lr * (mf[k] * c1) / (sqrtf(vf[k] * c2) + eps);
    }
    m[i] = mm;
    v[i] = vv;
    for (int q = 0; q < d.G; ++q) reinterpret_cast<float4*>(d.p[q])[i] = pp;
    if (t.n)
      for (int q = 0; q < d.G; ++q) shadow_store4(t, d.sh[q], (int)(4 * i), pf);
  }
  ss = block_sum(ss, red);
  if (threadIdx.x == 0 && d.part[0])
    for (int q = 0; q < d.G; ++q) d.part[q][d.rank * gridDim.x + blockIdx.x] = ss;
}
}  // namespace

int launch_dp_sync(const DpSync& a, cudaStream_t s) {
  note_launch(s, "k_dp_sync", 0, 0);
  launch_pdl(k_dp_sync, dim3(1), dim3(256), 0, s, a);
  return (int)cudaGetLastError();
}

int launch_dp_adam(const DpAdam& d, float* m, float* v, float lr, float b1, float b2, float eps, const float* c1,
                   const float* c2, const ShadowTable* t, int grad_perm, cudaStream_t s) {
  ShadowTable none;
  memset(&none, 0, sizeof(none));
  note_launch(s, "k_dp_adam", 0, (16.0 + 10.0 * d.G) * 4.0 * (double)(d.hi4 - d.lo4));
  launch_pdl(k_dp_adam, dim3(kAdamBlocks), dim3(256), 0, s, d, reinterpret_cast<float4*>(m),
             reinterpret_cast<float4*>(v), lr, b1, b2, eps, c1, c2, t ? *t : none, grad_perm);
  return (int)cudaGetLastError();
}

}  // namespace sq
