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

namespace sq {

namespace {

constexpr int kRows = 8;  // rows (warps) per block

__global__ void __launch_bounds__(256) k_target_ce(const __grid_constant__ TargetCEArgs a) {
  extern __shared__ float sm[];
  const int N = a.N, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* pb = sm + w * 2 * N;  // pbar [N]
  float* bj = pb + N;          // b_j [N]
  const int row = blockIdx.x * kRows + w;
  if (row >= a.B) return;
  const float dz = (a.v_max - a.v_min) / (float)(N - 1);
  const float alpha0 = expf(a.log_alpha[0]);
  const int64_t ridx = a.idx[row];
  const float r = a.reward[ridx];
  const float nd = a.done[ridx] ? 0.f : 1.f;
  const float shift = alpha0 * a.logp_next[row];
  // target heads -> pbar
  for (int hd = 0; hd < 2; ++hd) {
    const float* l = a.tlogits + ((int64_t)hd * a.B + row) * N;
    float mx = -INFINITY;
    for (int k = lane; k < N; k += 32) mx = fmaxf(mx, l[k]);
    mx = warp_max(mx);
    float s = 0.f;
    for (int k = lane; k < N; k += 32) s += expf(l[k] - mx);
    s = warp_sum(s);
    const float inv = 1.f / s;
    for (int k = lane; k < N; k += 32) {
      const float p = expf(l[k] - mx) * inv;
      pb[k] = (hd == 0) ? 0.5f * p : pb[k] + 0.5f * p;
    }
  }
  for (int j = lane; j < N; j += 32) {
    const float zj = a.v_min + (float)j * dz;
    float g = r + nd * a.gamma * (zj - shift);
    g = fminf(fmaxf(g, a.v_min), a.v_max);
    float b = (g - a.v_min) / dz;
    bj[j] = fminf(fmaxf(b, 0.f), (float)(N - 1));
  }
  __syncwarp();
  float* mrow = a.m + (int64_t)row * N;
  // b_j is non-decreasing in j (g_j is increasing in z_j and clipping preserves order), so the
  // atoms j with |b_j - k| < 1 form a contiguous range: binary search its start, then add the
  // same terms in the same (ascending j) order as the full sum.
  for (int k = lane; k < N; k += 32) {
    const float kf = (float)k;
    int lo = 0, hi = N;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (bj[mid] - kf > -1.f) hi = mid;
      else lo = mid + 1;
    }
    float acc = 0.f;
    for (int j = lo; j < N; ++j) {
      const float wgt = 1.f - fabsf(bj[j] - kf);
      if (bj[j] - kf >= 1.f) break;
      if (wgt > 0.f) acc = fmaf(pb[j], wgt, acc);
    }
    mrow[k] = acc;
  }
  __syncwarp();
  // online heads: CE and gradient
  float loss = 0.f;
  for (int hd = 0; hd < 2; ++hd) {
    const float* l = a.logits + ((int64_t)hd * a.B + row) * N;
    float* dl = a.dlogits_bf ? nullptr : a.dlogits + ((int64_t)hd * a.B + row) * N;
    __nv_bfloat16* dlb = a.dlogits_bf ? a.dlogits_bf + ((int64_t)hd * a.B + row) * a.ld_dl : nullptr;
    float mx = -INFINITY;
    for (int k = lane; k < N; k += 32) mx = fmaxf(mx, l[k]);
    mx = warp_max(mx);
    float s = 0.f;
    for (int k = lane; k < N; k += 32) s += expf(l[k] - mx);
    s = warp_sum(s);
    const float lse = mx + logf(s), inv = 1.f / s;
    float ce = 0.f;
    for (int k = lane; k < N; k += 32) {
      const float mk = mrow[k];
      ce -= mk * (l[k] - lse);
      const float g = (expf(l[k] - mx) * inv - mk) * a.scale;
      if (dlb) dlb[k] = __float2bfloat16_rn(g); else dl[k] = g;
    }
    loss += warp_sum(ce);
  }
  if (lane == 0) a.row_loss[row] = loss * a.scale;
}

__global__ void __launch_bounds__(256) k_actor_q(const __grid_constant__ ActorQArgs a) {
  const int N = a.N, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int row = blockIdx.x * kRows + w;
  if (row >= a.B) return;
  const float dz = (a.v_max - a.v_min) / (float)(N - 1);
  float q[2];
  for (int hd = 0; hd < 2; ++hd) {
    const float* l = a.logits + ((int64_t)hd * a.B + row) * N;
    float mx = -INFINITY;
    for (int k = lane; k < N; k += 32) mx = fmaxf(mx, l[k]);
    mx = warp_max(mx);
    float s = 0.f, sz = 0.f;
    for (int k = lane; k < N; k += 32) {
      const float e = expf(l[k] - mx);
      s += e;
      sz += e * (a.v_min + (float)k * dz);
    }
    s = warp_sum(s);
    sz = warp_sum(sz);
    const float inv = 1.f / s;
    q[hd] = sz * inv;
    float* dl = a.dlogits_bf ? nullptr : a.dlogits + ((int64_t)hd * a.B + row) * N;
    __nv_bfloat16* dlb = a.dlogits_bf ? a.dlogits_bf + ((int64_t)hd * a.B + row) * a.ld_dl : nullptr;
    const float c = -0.5f * a.scale;
    for (int k = lane; k < N; k += 32) {
      const float p = expf(l[k] - mx) * inv;
      const float g = c * p * ((a.v_min + (float)k * dz) - q[hd]);
      if (dlb) dlb[k] = __float2bfloat16_rn(g); else dl[k] = g;
    }
  }
  if (lane == 0) {
    const float qm = 0.5f * (q[0] + q[1]);
    a.row_q[row] = qm;
    a.row_lpi[row] = (a.alpha1[0] * a.logp[row] - qm) * a.scale;
  }
}

}  // namespace

int launch_target_ce(const TargetCEArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(float) * 2 * a.N * kRows;
  cudaFuncSetAttribute(k_target_ce, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  note_launch(s, "k_target_ce", 0, 0); k_target_ce<<<(a.B + kRows - 1) / kRows, 256, smem, s>>>(a);
  return (int)cudaGetLastError();
}

int launch_actor_q(const ActorQArgs& a, cudaStream_t s) {
  note_launch(s, "k_actor_q", 0, 0); k_actor_q<<<(a.B + kRows - 1) / kRows, 256, 0, s>>>(a);
  return (int)cudaGetLastError();
}

}  // namespace sq
