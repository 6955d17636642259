// heads.cu -- distributional critic machinery (a9, a10, a12), warp per row.
//
//  k_target_ce: pbar = (softmax l1_bar + softmax l2_bar)/2 (Q20); categorical projection of
//      the atoms shifted by r + (1-d) gamma (z_j - alpha0 log pi') (Q21-Q23) in the
//      deterministic "hat" gather form m_k = sum_j pbar_j max(0, 1 - |b_j - k|), which is
//      the floor/ceil split of S:280 written without scatter (so no atomics, bitwise
//      reproducible); then CE of both online heads (Q24) and dL/dl = (softmax - m) s.
//  k_actor_q: Q_i = sum_k softmax(l_i^+)_k z_k (Q25), dL_pi/dl_i = -s/2 p (z - Q_i),
//      per-row terms of L_pi = s sum_b [alpha+ log pi_b - (Q1 + Q2)/2].
#include <cuda_runtime.h>

#include "common.cuh"
#include "heads.cuh"
#include "optim.cuh"

namespace sq {

namespace {

constexpr int kRows = 8;  // rows (warps) per block

// Row values live in registers: lane holds atoms k = lane + 32 i, i < NPL (all loads of a row are
// issued together; every reduction is a fixed-order warp butterfly).
template <int NPL>
__global__ void __launch_bounds__(256) k_target_ce(const __grid_constant__ TargetCEArgs a) {
  grid_wait();
  grid_trigger();
  extern __shared__ float sm[];
  const int N = a.N, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* pb = sm + w * 2 * N;  // pbar [N]
  float* bj = pb + N;          // b_j [N]
  const int row = blockIdx.x * kRows + w;
  if (a.step && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t tc = ++a.step[0], ta = ++a.step[1];
    a.scal[S_C1_CRITIC] = bias_corr(a.beta1, tc);
    a.scal[S_C2_CRITIC] = bias_corr(a.beta2, tc);
    a.scal[S_C1_ACTOR] = bias_corr(a.beta1, ta);
    a.scal[S_C2_ACTOR] = bias_corr(a.beta2, ta);
  }
  if (row >= a.B) return;
  const int64_t ridx = a.idx[row];
  float tl[2][NPL], ol[2][NPL];
#pragma unroll
  for (int hd = 0; hd < 2; ++hd)
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const int k = lane + 32 * i;
      tl[hd][i] = k < N ? a.tlogits[((int64_t)hd * a.B + row) * N + k] : -INFINITY;
      ol[hd][i] = k < N ? a.logits[((int64_t)hd * a.B + row) * N + k] : -INFINITY;
    }
  const float r = a.reward[ridx];
  const float nd = a.done[ridx] ? 0.f : 1.f;
  const float dz = (a.v_max - a.v_min) / (float)(N - 1);
  const float shift = expf(a.log_alpha[0]) * a.logp_next[row];
  // pbar = (softmax l1_bar + softmax l2_bar) / 2
  float pbar[NPL];
#pragma unroll
  for (int i = 0; i < NPL; ++i) pbar[i] = 0.f;
#pragma unroll
  for (int hd = 0; hd < 2; ++hd) {
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < NPL; ++i) mx = fmaxf(mx, tl[hd][i]);
    mx = warp_max(mx);
    float e[NPL], sum = 0.f;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      e[i] = (lane + 32 * i < N) ? expf(tl[hd][i] - mx) : 0.f;
      sum += e[i];
    }
    sum = warp_sum(sum);
    const float inv = 1.f / sum;
#pragma unroll
    for (int i = 0; i < NPL; ++i) pbar[i] += 0.5f * e[i] * inv;
  }
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    if (j < N) {
      const float zj = a.v_min + (float)j * dz;
      float g = r + nd * a.gamma * (zj - shift);
      g = fminf(fmaxf(g, a.v_min), a.v_max);
      const float b = (g - a.v_min) / dz;
      bj[j] = fminf(fmaxf(b, 0.f), (float)(N - 1));
      pb[j] = pbar[i];
    }
  }
  __syncwarp();
  // m_k = sum_j pbar_j max(0, 1 - |b_j - k|).  b_j is non-decreasing in j (g_j increases with z_j
  // and clipping preserves order), so the contributing j form a contiguous range: binary search
  // its start, then add the terms in ascending j as the full sum would.
  float m[NPL];
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int k = lane + 32 * i;
    float acc = 0.f;
    if (k < N) {
      const float kf = (float)k;
      int lo = 0, hi = N;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (bj[mid] - kf > -1.f) hi = mid;
        else lo = mid + 1;
      }
      for (int j = lo; j < N; ++j) {
        const float d = bj[j] - kf;
        if (d >= 1.f) break;
        const float wgt = 1.f - fabsf(d);
        if (wgt > 0.f) acc = fmaf(pb[j], wgt, acc);
      }
      a.m[(int64_t)row * N + k] = acc;
    }
    m[i] = acc;
  }
  // online heads: CE and dL/dl = (softmax - m) * scale
  float loss = 0.f;
#pragma unroll
  for (int hd = 0; hd < 2; ++hd) {
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < NPL; ++i) mx = fmaxf(mx, ol[hd][i]);
    mx = warp_max(mx);
    float e[NPL], sum = 0.f;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      e[i] = (lane + 32 * i < N) ? expf(ol[hd][i] - mx) : 0.f;
      sum += e[i];
    }
    sum = warp_sum(sum);
    const float lse = mx + logf(sum), inv = 1.f / sum;
    float ce = 0.f;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const int k = lane + 32 * i;
      if (k < N) {
        ce -= m[i] * (ol[hd][i] - lse);
        const float g = (e[i] * inv - m[i]) * a.scale;
        if (a.dlogits_bf) a.dlogits_bf[((int64_t)hd * a.B + row) * a.ld_dl + k] = __float2bfloat16_rn(g);
        else a.dlogits[((int64_t)hd * a.B + row) * N + k] = g;
      }
    }
    loss += warp_sum(ce);
  }
  if (lane == 0) a.row_loss[row] = loss * a.scale;
}

template <int NPL>
__global__ void __launch_bounds__(256) k_actor_q(const __grid_constant__ ActorQArgs a) {
  grid_wait();
  grid_trigger();
  const int N = a.N, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int row = blockIdx.x * kRows + w;
  if (row >= a.B) return;
  const float dz = (a.v_max - a.v_min) / (float)(N - 1);
  float l[2][NPL];
#pragma unroll
  for (int hd = 0; hd < 2; ++hd)
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const int k = lane + 32 * i;
      l[hd][i] = k < N ? a.logits[((int64_t)hd * a.B + row) * N + k] : -INFINITY;
    }
  float q0 = 0.f, q1 = 0.f;
#pragma unroll
  for (int hd = 0; hd < 2; ++hd) {
    float mx = -INFINITY;
#pragma unroll
    for (int i = 0; i < NPL; ++i) mx = fmaxf(mx, l[hd][i]);
    mx = warp_max(mx);
    float e[NPL], s = 0.f, sz = 0.f;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const int k = lane + 32 * i;
      e[i] = k < N ? expf(l[hd][i] - mx) : 0.f;
      s += e[i];
      sz += e[i] * (a.v_min + (float)k * dz);
    }
    s = warp_sum(s);
    sz = warp_sum(sz);
    const float inv = 1.f / s, q = sz * inv;
    if (hd == 0) q0 = q; else q1 = q;
    const float c = -0.5f * a.scale;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
      const int k = lane + 32 * i;
      if (k < N) {
        const float g = c * e[i] * inv * ((a.v_min + (float)k * dz) - q);
        if (a.dlogits_bf) a.dlogits_bf[((int64_t)hd * a.B + row) * a.ld_dl + k] = __float2bfloat16_rn(g);
        else a.dlogits[((int64_t)hd * a.B + row) * N + k] = g;
      }
    }
  }
  if (lane == 0) {
    const float qm = 0.5f * (q0 + q1);
    a.row_q[row] = qm;
    a.row_lpi[row] = (a.alpha1[0] * a.logp[row] - qm) * a.scale;
  }
}

}  // namespace

int launch_target_ce(const TargetCEArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(float) * 2 * a.N * kRows;
  const int npl = (a.N + 31) / 32;
  const dim3 grid((a.B + kRows - 1) / kRows);
  note_launch(s, "k_target_ce", 0, 0);
#define SQ_TCE(n)                                                                              \
  {                                                                                            \
    cudaFuncSetAttribute(k_target_ce<n>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    launch_pdl(k_target_ce<n>, grid, dim3(256), smem, s, a);                                                 \
  }
  if (npl <= 2) SQ_TCE(2) else if (npl <= 4) SQ_TCE(4) else if (npl <= 8) SQ_TCE(8) else SQ_TCE(16)
#undef SQ_TCE
  return (int)cudaGetLastError();
}

int launch_actor_q(const ActorQArgs& a, cudaStream_t s) {
  const int npl = (a.N + 31) / 32;
  const dim3 grid((a.B + kRows - 1) / kRows);
  note_launch(s, "k_actor_q", 0, 0);
  if (npl <= 2) launch_pdl(k_actor_q<2>, grid, dim3(256), 0, s, a);
  else if (npl <= 4) launch_pdl(k_actor_q<4>, grid, dim3(256), 0, s, a);
  else if (npl <= 8) launch_pdl(k_actor_q<8>, grid, dim3(256), 0, s, a);
  else launch_pdl(k_actor_q<16>, grid, dim3(256), 0, s, a);
  return (int)cudaGetLastError();
}

}  // namespace sq
