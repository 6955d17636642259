// dense_f32.cu -- fp32 SIMT grouped dense layers (the parity path, squint_dims.precision
// == SQUINT_FP32).  Full-row tiles (BM = 16 rows x BN >= N columns) so LayerNorm
// statistics (Q9) and the tanh-Gaussian head (Q13-Q14) are finished in the
// epilogue without another pass over HBM.  Reductions are fixed-order (no float atomics),
// so every result is bitwise reproducible run to run.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "dense.cuh"

namespace sq {

namespace {

constexpr float kLog2Pi = 1.8378770664093453f;
constexpr float kSquashEps = 1e-6f;  // Q14

SQ_DEV float a_at(const ASeg* A, int nA, int M, int m, int k) {
  if (m >= M) return 0.f;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    if (s >= nA) break;
    if (k < A[s].width) {
      int64_t row = A[s].rows ? A[s].rows[m] : (int64_t)m;
      return A[s].ptr[row * A[s].ld + k];
    }
    k -= A[s].width;
  }
  return 0.f;
}

SQ_DEV float b_at(const BSeg* B, int nB, int N, int n, int k) {
  if (n >= N) return 0.f;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    if (s >= nB) break;
    if (k < B[s].width) return B[s].kmajor ? B[s].ptr[(int64_t)n * B[s].ld + k] : B[s].ptr[(int64_t)k * B[s].ld + n];
    k -= B[s].width;
  }
  return 0.f;
}

// Sum v[i] over the 64 threads that share a row group (ty = tid / 64); fixed order.
template <int TM>
SQ_DEV void row_reduce(float (&v)[TM], float* red) {
  const int tid = threadIdx.x, lane = tid & 31, half = (tid >> 5) & 1, ty = tid >> 6;
#pragma unroll
  for (int i = 0; i < TM; ++i) v[i] = warp_sum(v[i]);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < TM; ++i) red[(ty * 2 + half) * TM + i] = v[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < TM; ++i) v[i] = red[(ty * 2) * TM + i] + red[(ty * 2 + 1) * TM + i];
  __syncthreads();
}

template <int TN>
__global__ void __launch_bounds__(256) k_dense_f32(const __grid_constant__ DenseBatch b) {
  constexpr int TM = 4, BM = 16, BN = 64 * TN, BK = 32;
  extern __shared__ float smem[];
  float* As = smem;                 // [BK][BM]
  float* Bs = As + BK * BM;         // [BK][BN + 1]
  float* red = Bs + BK * (BN + 1);  // [4 * 2 * TM]

  const int tile = blockIdx.x;
  int pi = 0;
  while (pi + 1 < b.nprob && tile >= b.p[pi + 1].tile0) ++pi;
  const DenseProb& P = b.p[pi];
  const int lt = tile - P.tile0;
  const int m0 = (lt / P.tiles_n) * BM, n0 = (lt % P.tiles_n) * BN;
  const int tid = threadIdx.x, tx = tid & 63, ty = tid >> 6;

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  const bool bk = P.B[0].kmajor;
  for (int k0 = 0; k0 < P.K; k0 += BK) {
    for (int e = tid; e < BM * BK; e += 256) {
      const int m = e / BK, k = e % BK;
      float av = (k0 + k < P.K) ? a_at(P.A, P.nA, P.M, m0 + m, k0 + k) : 0.f;
      if (b.emul & 1) av = __bfloat162float(__float2bfloat16_rn(av));
      As[k * BM + m] = av;
    }
    if (bk) {
      for (int e = tid; e < BN * BK; e += 256) {
        const int n = e / BK, k = e % BK;
        float bv = (k0 + k < P.K) ? b_at(P.B, P.nB, P.N, n0 + n, k0 + k) : 0.f;
        if (b.emul & 2) bv = __bfloat162float(__float2bfloat16_rn(bv));
        Bs[k * (BN + 1) + n] = bv;
      }
    } else {
      for (int e = tid; e < BN * BK; e += 256) {
        const int k = e / BN, n = e % BN;
        float bv = (k0 + k < P.K) ? b_at(P.B, P.nB, P.N, n0 + n, k0 + k) : 0.f;
        if (b.emul & 2) bv = __bfloat162float(__float2bfloat16_rn(bv));
        Bs[k * (BN + 1) + n] = bv;
      }
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < BK; ++kk) {
      float av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[kk * BM + ty * TM + i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[kk * (BN + 1) + tx + 64 * j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }

  const int epi = P.epi;
  const int N = P.N;
  auto row_of = [&](int i) { return m0 + ty * TM + i; };
  auto col_of = [&](int j) { return n0 + tx + 64 * j; };

  if (epi == EPI_STORE || epi == EPI_BIAS || epi == EPI_RELU_MASK) {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int r = row_of(i);
      if (r >= P.M) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int c = col_of(j);
        if (c >= N) continue;
        float v = acc[i][j];
        if (epi == EPI_BIAS) v += P.bias[c];
        if (epi == EPI_RELU_MASK) v = P.y[(int64_t)r * N + c] > 0.f ? v : 0.f;
        P.out[(int64_t)r * P.ldo + c] = v;
      }
    }
    return;
  }

  if (epi == EPI_LN_RELU || epi == EPI_LN_TANH) {
    float s[TM];
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      s[i] = 0.f;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int c = col_of(j);
        acc[i][j] = (c < N) ? acc[i][j] + P.bias[c] : 0.f;
        s[i] += acc[i][j];
      }
    }
    row_reduce<TM>(s, red);
    float mean[TM], ss[TM];
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      mean[i] = s[i] / (float)N;
      ss[i] = 0.f;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const float d = (col_of(j) < N) ? acc[i][j] - mean[i] : 0.f;
        acc[i][j] = d;
        ss[i] += d * d;
      }
    }
    row_reduce<TM>(ss, red);
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int r = row_of(i);
      const float rs = 1.0f / sqrtf(ss[i] / (float)N + P.ln_eps);
      if (r >= P.M) continue;
      if (tx == 0 && P.rstd) P.rstd[r] = rs;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int c = col_of(j);
        if (c >= N) continue;
        // option 4 bit 2 emulates the bf16 path's x_hat cache, which it also normalises with
        const float xh = (b.emul & 4) ? __bfloat162float(__float2bfloat16_rn(acc[i][j] * rs)) : acc[i][j] * rs;
        const float n = fmaf(xh, P.g[c], P.beta[c]);
        const float y = (epi == EPI_LN_RELU) ? fmaxf(n, 0.f) : tanhf(n);
        if (P.xh) P.xh[(int64_t)r * N + c] = xh;
        P.out[(int64_t)r * P.ldo + c] = y;
      }
    }
    return;
  }

  if (epi == EPI_BWD_LN_RELU || epi == EPI_BWD_LN_TANH) {
    float s1[TM], s2[TM], xhv[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int r = row_of(i);
      s1[i] = s2[i] = 0.f;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int c = col_of(j);
        float dxh = 0.f, xv = 0.f;
        if (r < P.M && c < N) {
          const float yv = P.y[(int64_t)r * N + c];
          const float dn = (epi == EPI_BWD_LN_RELU) ? (yv > 0.f ? acc[i][j] : 0.f) : acc[i][j] * (1.f - yv * yv);
          P.out2[(int64_t)r * N + c] = dn;
          xv = P.xh[(int64_t)r * N + c];
          dxh = dn * P.g[c];
        }
        acc[i][j] = dxh;
        xhv[i][j] = xv;
        s1[i] += dxh;
        s2[i] += dxh * xv;
      }
    }
    row_reduce<TM>(s1, red);
    row_reduce<TM>(s2, red);
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int r = row_of(i);
      if (r >= P.M) continue;
      const float rs = P.rstd[r];
      const float m1 = s1[i] / (float)N, m2 = s2[i] / (float)N;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int c = col_of(j);
        if (c >= N) continue;
        P.out[(int64_t)r * P.ldo + c] = rs * (acc[i][j] - m1 - xhv[i][j] * m2);
      }
    }
    return;
  }

  if (epi == EPI_TG_FWD) {
    // o = [mu | l] (N = 2A) -> smem, then one thread per row finishes the head.
    float* os = Bs;  // reuse: [BM][BN]
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int r = row_of(i);
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int c = col_of(j);
        if (c >= N) continue;
        const float v = acc[i][j] + P.bias[c];
        os[(ty * TM + i) * BN + c] = v;
        if (r < P.M && P.out) P.out[(int64_t)r * P.ldo + c] = v;
      }
    }
    __syncthreads();
    const int A = N / 2;
    if (tid < BM && m0 + tid < P.M) {
      const int r = m0 + tid;
      float lp = 0.f;
      for (int d = 0; d < A; ++d) {
        const float mu = os[tid * BN + d], l = os[tid * BN + A + d];
        const float tl = tanhf(l);
        const float log_std = P.lo + 0.5f * (P.hi - P.lo) * (tl + 1.f);
        const float sd = expf(log_std);
        const float e = P.eps ? P.eps[(int64_t)r * A + d] : 0.f;
        const float u = fmaf(sd, e, mu);
        P.act[(int64_t)r * A + d] = tanhf(u);
        lp += -0.5f * e * e - log_std - 0.5f * kLog2Pi - logf(sech2f(u) + kSquashEps);
      }
      if (P.logp) P.logp[r] = lp;
    }
    return;
  }

  if (epi == EPI_TG_BWD) {
    const int A = N;
    const float dlp = P.dlogp_scale[0] * P.dlogp_mult;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int r = row_of(i);
      if (r >= P.M) continue;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int d = col_of(j);
        if (d >= A) continue;
        const float mu = P.tg_o[(int64_t)r * 2 * A + d], l = P.tg_o[(int64_t)r * 2 * A + A + d];
        const float tl = tanhf(l);
        const float log_std = P.lo + 0.5f * (P.hi - P.lo) * (tl + 1.f);
        const float sd = expf(log_std);
        const float e = P.eps[(int64_t)r * A + d];
        const float u = fmaf(sd, e, mu);
        const float a = tanhf(u);
        const float om = sech2f(u);
        const float du = acc[i][j] * om + dlp * (2.f * a * om / (om + kSquashEps));
        const float dls = du * sd * e - dlp;
        P.out[(int64_t)r * P.ldo + d] = du;
        P.out[(int64_t)r * P.ldo + A + d] = dls * 0.5f * (P.hi - P.lo) * sech2f(l);
      }
    }
    return;
  }
}

// ---- weight gradients -----------------------------------------------------------------
__global__ void __launch_bounds__(256) k_dw_f32(const __grid_constant__ DwBatch b) {
  constexpr int BN = kDwBN, BK = kDwBK, BMc = 32;
  __shared__ float Ds[BMc][BN + 1];
  __shared__ float Xs[BMc][BK + 1];
  const int tile = blockIdx.x;
  int pi = 0;
  while (pi + 1 < b.nprob && tile >= b.p[pi + 1].tile0) ++pi;
  const DwProb& P = b.p[pi];
  const int lt = tile - P.tile0;
  const int n0 = (lt / P.tiles_k) * BN, k0 = (lt % P.tiles_k) * BK;
  const int tid = threadIdx.x, tn = tid >> 4, tk = tid & 15;

  float acc[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int mb = 0; mb < P.M; mb += BMc) {
    for (int e = tid; e < BMc * BN; e += 256) {
      const int m = e / BN, n = e % BN;
      float dv = (mb + m < P.M && n0 + n < P.N) ? P.D[(int64_t)(mb + m) * P.N + n0 + n] : 0.f;
      if (b.emul & 1) dv = __bfloat162float(__float2bfloat16_rn(dv));
      Ds[m][n] = dv;
    }
    for (int e = tid; e < BMc * BK; e += 256) {
      const int m = e / BK, k = e % BK;
      float xv = (k0 + k < P.K) ? a_at(P.A, P.nA, P.M, mb + m, k0 + k) : 0.f;
      if (b.emul & 1) xv = __bfloat162float(__float2bfloat16_rn(xv));
      Xs[m][k] = xv;
    }
    __syncthreads();
#pragma unroll 8
    for (int mm = 0; mm < BMc; ++mm) {
      const float d0 = Ds[mm][2 * tn], d1 = Ds[mm][2 * tn + 1];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float x = Xs[mm][tk + 16 * j];
        acc[0][j] = fmaf(d0, x, acc[0][j]);
        acc[1][j] = fmaf(d1, x, acc[1][j]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int n = n0 + 2 * tn + i;
    if (n >= P.N) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = k0 + tk + 16 * j;
      if (k < P.K) P.dW[(int64_t)n * P.K + k] = acc[i][j];
    }
  }
  if (k0 != 0) return;
  // column sums for this tile's 32 n: thread = (n_local = tid / 8, m-lane = tid % 8)
  const int nl = tid >> 3, ml = tid & 7, n = n0 + nl;
  float sb = 0.f, sg = 0.f, sbeta = 0.f;
  if (n < P.N) {
    for (int m = ml; m < P.M; m += 8) {
      sb += P.D[(int64_t)m * P.N + n];
      if (P.DN) {
        const float dn = P.DN[(int64_t)m * P.N + n];
        sg += dn * P.xh[(int64_t)m * P.N + n];
        sbeta += dn;
      }
    }
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) {
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
    sg += __shfl_xor_sync(0xffffffffu, sg, o);
    sbeta += __shfl_xor_sync(0xffffffffu, sbeta, o);
  }
  if (ml == 0 && n < P.N) {
    if (P.db) P.db[n] = sb;
    if (P.DN) {
      P.dg[n] = sg;
      P.dbeta[n] = sbeta;
    }
  }
}

}  // namespace

int plan_dense(DenseBatch& b) {
  int maxn = 1;
  for (int i = 0; i < b.nprob; ++i) maxn = b.p[i].N > maxn ? b.p[i].N : maxn;
  int tn = maxn <= 64 ? 1 : maxn <= 128 ? 2 : maxn <= 256 ? 4 : 8;
  const int BN = 64 * tn;
  int t = 0;
  for (int i = 0; i < b.nprob; ++i) {
    DenseProb& p = b.p[i];
    p.tiles_n = (p.N + BN - 1) / BN;
    p.tile0 = t;
    t += p.tiles_n * ((p.M + kDenseBM - 1) / kDenseBM);
  }
  b.ntiles = t;
  return tn;
}

void plan_dw(DwBatch& b) {
  int t = 0;
  for (int i = 0; i < b.nprob; ++i) {
    DwProb& p = b.p[i];
    p.tiles_k = (p.K + kDwBK - 1) / kDwBK;
    p.tile0 = t;
    t += p.tiles_k * ((p.N + kDwBN - 1) / kDwBN);
  }
  b.ntiles = t;
}

template <int TN>
static int launch_tn(const DenseBatch& b, cudaStream_t s) {
  constexpr int BN = 64 * TN;
  const size_t smem = sizeof(float) * (32 * 16 + 32 * (BN + 1) + 64);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_dense_f32<TN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  note_launch(s, "k_dense_f32", 0, 0); k_dense_f32<TN><<<b.ntiles, 256, smem, s>>>(b);
  return (int)cudaGetLastError();
}

int launch_dense_f32(const DenseBatch& b, int tn, cudaStream_t s) {
  if (b.ntiles == 0) return 0;
  switch (tn) {
    case 1: return launch_tn<1>(b, s);
    case 2: return launch_tn<2>(b, s);
    case 4: return launch_tn<4>(b, s);
    default: return launch_tn<8>(b, s);
  }
}

int launch_dw_f32(const DwBatch& b, cudaStream_t s) {
  if (b.ntiles == 0) return 0;
  note_launch(s, "k_dw_f32", 0, 0); k_dw_f32<<<b.ntiles, 256, 0, s>>>(b);
  return (int)cudaGetLastError();
}

}  // namespace sq
