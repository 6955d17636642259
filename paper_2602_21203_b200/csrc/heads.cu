// heads.cu -- distributional critic machinery (a9, a10, a12), warp per row.
//
//  k_target_ce: pbar = (softmax l1_bar + softmax l2_bar)/2 (Q20); categorical projection of
//      the atoms shifted by r + (1-d) gamma (z_j - alpha0 log pi') (Q21-Q23) in the "hat" form
//      m_k = sum_j pbar_j max(0, 1 - |b_j - k|) (the floor/ceil split of S:280 with an integral
//      b_j landing whole), as a warp segmented scan over the sorted atoms (no atomics, bitwise
//      reproducible); then CE of both online heads (Q24) and dL/dl = (softmax - m) s.
//  k_actor_q: Q_i = sum_k softmax(l_i^+)_k z_k (Q25), dL_pi/dl_i = -s/2 p (z - Q_i),
//      per-row terms of L_pi = s sum_b [alpha+ log pi_b - (Q1 + Q2)/2].
//  k_target_mse / k_actor_q_mse: the scalar-critic variants (f3; Eqs. 1-2, Algorithm 1 lines
//      13, 15, 22), thread per row.
#include <cuda_runtime.h>

#include <cstdlib>

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
  auto stamp = [&](int k) {
    if (a.dbg && (threadIdx.x & 31) == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      a.dbg[(blockIdx.x * kRows + (threadIdx.x >> 5)) * 4 + k] = t;
    }
  };
  stamp(0);
  extern __shared__ float sm_acc[];
  const int N = a.N, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
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
  stamp(1);
  const float dz = (a.v_max - a.v_min) / (float)(N - 1);
  const float shift = expf(a.log_alpha[0]) * a.logp_next[row];
  // pbar = (softmax l1_bar + softmax l2_bar) / 2, or (CDQ, f3) the softmax of the head with the
  // smaller expected value sum_k p_k z_k (ties: head 1)
  float pbar[NPL];
#pragma unroll
  for (int i = 0; i < NPL; ++i) pbar[i] = 0.f;
  float phd[2][NPL], ev[2];
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
    if (a.cdq) {
      float q = 0.f;
#pragma unroll
      for (int i = 0; i < NPL; ++i) {
        phd[hd][i] = e[i] * inv;
        q += phd[hd][i] * (a.v_min + (float)(lane + 32 * i) * dz);
      }
      ev[hd] = warp_sum(q);
    } else {
#pragma unroll
      for (int i = 0; i < NPL; ++i) pbar[i] += 0.5f * e[i] * inv;
    }
  }
  if (a.cdq) {
    const int pick = ev[1] < ev[0] ? 1 : 0;
#pragma unroll
    for (int i = 0; i < NPL; ++i) pbar[i] = pick ? phd[1][i] : phd[0][i];
  }
  // Categorical projection (Q21-Q23) in the hat form m_k = sum_j pbar_j max(0, 1 - |b_j - k|):
  // atom j gives a_j = pbar_j (1 - f_j) to bin l_j = floor(b_j) and h_j = pbar_j f_j to bin
  // l_j + 1 (an integral b_j lands whole on l_j).  b_j is non-decreasing in j (g_j increases with
  // z_j; clipping keeps the order), so the atoms of one bin form a contiguous run: a segmented
  // scan over the atoms in j order (4 consecutive atoms per lane, then a warp scan of the lanes'
  // trailing runs as affine maps) yields every run's totals at its last atom; then
  // m_k = A(k) + H(k - 1).  Fixed-order fp32 sums (bitwise reproducible), O(log) depth however
  // many atoms pile up in one bin (clipped support).
  float* pbs = reinterpret_cast<float*>(sm_acc) + w * 3 * 32 * NPL;  // pbar | A | H, 32 NPL each
  float* As = pbs + 32 * NPL;
  float* Hs = As + 32 * NPL;
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = lane + 32 * i;
    pbs[j] = j < N ? pbar[i] : 0.f;
  }
  for (int k = lane; k < 32 * NPL; k += 32) As[k] = Hs[k] = 0.f;
  __syncwarp();
  int key[NPL];
  float sa[NPL], sh[NPL];
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int j = NPL * lane + i;
    float va = 0.f, vh = 0.f;
    key[i] = N + 1;  // padding atoms: a run past the support, never stored
    if (j < N) {
      const float zj = a.v_min + (float)j * dz;
      float g = r + nd * a.gamma * (zj - shift);
      g = fminf(fmaxf(g, a.v_min), a.v_max);
      const float b = fminf(fmaxf((g - a.v_min) / dz, 0.f), (float)(N - 1));
      const float fl = floorf(b);
      const float f = b - fl;
      key[i] = (int)fl;
      va = pbs[j] * (1.f - f);
      vh = pbs[j] * f;
    }
    // lane-local segmented inclusive scan
    const bool cont = i > 0 && key[i] == key[i - 1];
    sa[i] = va + (cont ? sa[i - 1] : 0.f);
    sh[i] = vh + (cont ? sh[i - 1] : 0.f);
  }
  // trailing-run totals across lanes: S(x) = tail(x) + c(x) S(x - 1), c(x) = [lane x is one run
  // continuing lane x - 1's last run]; composed as affine maps in a Hillis-Steele scan
  const int kprev = __shfl_up_sync(0xffffffffu, key[NPL - 1], 1);
  const int knext = __shfl_down_sync(0xffffffffu, key[0], 1);
  float Ba = sa[NPL - 1], Bh = sh[NPL - 1];
  int cc = (lane > 0 && key[0] == key[NPL - 1] && kprev == key[0]) ? 1 : 0;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float ua = __shfl_up_sync(0xffffffffu, Ba, off);
    const float uh = __shfl_up_sync(0xffffffffu, Bh, off);
    const int uc = __shfl_up_sync(0xffffffffu, cc, off);
    if (lane >= off) {
      if (cc) {
        Ba += ua;
        Bh += uh;
      }
      cc &= uc;
    }
  }
  // carry into this lane's first run from the lanes before it
  const float pa = __shfl_up_sync(0xffffffffu, Ba, 1), ph = __shfl_up_sync(0xffffffffu, Bh, 1);
  const bool carry = lane > 0 && kprev == key[0];
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const bool first_run = key[i] == key[0];
    const float ta = sa[i] + ((carry && first_run) ? pa : 0.f);
    const float th = sh[i] + ((carry && first_run) ? ph : 0.f);
    const bool run_end = i < NPL - 1 ? key[i + 1] != key[i] : (lane == 31 || knext != key[NPL - 1]);
    if (run_end && key[i] < N) {
      As[key[i]] = ta;
      Hs[key[i]] = th;
    }
  }
  __syncwarp();
  float m[NPL];
#pragma unroll
  for (int i = 0; i < NPL; ++i) {
    const int k = lane + 32 * i;
    float acc = 0.f;
    if (k < N) {
      acc = As[k] + (k > 0 ? Hs[k - 1] : 0.f);
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
  stamp(3);
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

// f3 scalar critic.  y = r + (1-d) gamma/2 sum_i (Qbar_i - alpha_0 log pi') (Algorithm 1 line 13,
// Q22 mask) or, CDQ, r + (1-d) gamma (min_i Qbar_i - alpha_0 log pi');
// L_Q = s sum_i sum_b (Q_i - y)^2, dL/dQ_i = 2 s (Q_i - y) (line 15, Eq. 2).
__global__ void __launch_bounds__(256) k_target_mse(const __grid_constant__ TargetCEArgs a) {
  grid_wait();
  grid_trigger();
  if (a.step && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t tc = ++a.step[0], ta = ++a.step[1];
    a.scal[S_C1_CRITIC] = bias_corr(a.beta1, tc);
    a.scal[S_C2_CRITIC] = bias_corr(a.beta2, tc);
    a.scal[S_C1_ACTOR] = bias_corr(a.beta1, ta);
    a.scal[S_C2_ACTOR] = bias_corr(a.beta2, ta);
  }
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= a.B) return;
  const int64_t ridx = a.idx[row];
  const float nd = a.done[ridx] ? 0.f : 1.f;
  const float sh = expf(a.log_alpha[0]) * a.logp_next[row];
  const float t0 = a.tlogits[row], t1 = a.tlogits[a.B + row];
  const float v = a.cdq ? fminf(t0, t1) - sh : 0.5f * ((t0 - sh) + (t1 - sh));
  const float y = a.reward[ridx] + nd * a.gamma * v;
  a.m[row] = y;
  float loss = 0.f;
#pragma unroll
  for (int hd = 0; hd < 2; ++hd) {
    const float e = a.logits[(int64_t)hd * a.B + row] - y;
    loss += e * e;
    const float g = 2.f * e * a.scale;
    if (a.dlogits_bf) a.dlogits_bf[((int64_t)hd * a.B + row) * a.ld_dl] = __float2bfloat16_rn(g);
    else a.dlogits[(int64_t)hd * a.B + row] = g;
  }
  a.row_loss[row] = loss * a.scale;
}

// L_pi = s sum_b [alpha+ log pi_b - (Q1 + Q2)/2] with Q_i the heads' outputs (line 22)
__global__ void __launch_bounds__(256) k_actor_q_mse(const __grid_constant__ ActorQArgs a) {
  grid_wait();
  grid_trigger();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= a.B) return;
  const float g = -0.5f * a.scale;
#pragma unroll
  for (int hd = 0; hd < 2; ++hd) {
    if (a.dlogits_bf) a.dlogits_bf[((int64_t)hd * a.B + row) * a.ld_dl] = __float2bfloat16_rn(g);
    else a.dlogits[(int64_t)hd * a.B + row] = g;
  }
  const float qm = 0.5f * (a.logits[row] + a.logits[a.B + row]);
  a.row_q[row] = qm;
  a.row_lpi[row] = (a.alpha1[0] * a.logp[row] - qm) * a.scale;
}

}  // namespace

static unsigned long long* g_tce_dbg = nullptr;
int launch_target_ce(const TargetCEArgs& a_in, cudaStream_t s) {
  TargetCEArgs a = a_in;
  if (a.mse) {
    if (a.N != 1) return (int)cudaErrorInvalidValue;
    note_launch(s, "k_target_mse", 0, 0);
    launch_pdl(k_target_mse, dim3((a.B + 255) / 256), dim3(256), 0, s, a);
    return (int)cudaGetLastError();
  }
  static const bool dbg = getenv("SQUINT_TCE_DBG") != nullptr;
  if (dbg) {
    if (!g_tce_dbg) cudaMalloc(&g_tce_dbg, 4096 * 4 * sizeof(unsigned long long));
    a.dbg = g_tce_dbg;
  }
  const size_t smem = sizeof(float) * 3 * 32 * ((a.N + 31) / 32 <= 2 ? 2 : (a.N + 31) / 32 <= 4 ? 4 : (a.N + 31) / 32 <= 8 ? 8 : 16) * kRows;
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
  if (a.mse) {
    if (a.N != 1) return (int)cudaErrorInvalidValue;
    note_launch(s, "k_actor_q_mse", 0, 0);
    launch_pdl(k_actor_q_mse, dim3((a.B + 255) / 256), dim3(256), 0, s, a);
    return (int)cudaGetLastError();
  }
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

extern "C" __attribute__((visibility("default"))) int squint_debug_tce(unsigned long long* host, int n) {
  if (!sq::g_tce_dbg) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(host, sq::g_tce_dbg, (size_t)n * 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return n;
}
