// dense_tc.cu -- bf16 tensor-core (tcgen05) grouped dense layers for the bf16 path.
//
// Same problem semantics and epilogues as dense_f32.cu (LayerNorm P:159 / Q9, tanh-Gaussian
// Q13-Q14 and their backward), but the contraction runs on the 5th-gen tensor cores:
//   * 128 threads per CTA, one 128-row output tile (UMMA M = 128) x BN columns (N <= 512;
//     two N = 256 MMAs when N > 256), fp32 accumulator in TMEM;
//   * operands are fp32 in global memory (master weights, fp32 activations); the fill
//     threads convert to bf16 and write 128B-swizzled K-major tiles, so no bf16 shadow copy
//     of the weights is ever needed; 2-stage smem ring, tcgen05.commit -> mbarrier;
//   * epilogue: one thread per tile row reads its TMEM lane (tcgen05.ld 32x32b), so the
//     LayerNorm row statistics are register-local -- no cross-thread reduction.
// Weight gradients dW = D^T X run through the same kernel with both operands read
// "row-contiguous" (the batch is the reduction dim); db / dg / dbeta are fixed-order column
// sums in k_colsums.  Nothing uses float atomics: results are bitwise reproducible.
#include <cuda_runtime.h>

#include "common.cuh"
#include "dense.cuh"
#include "dense_tc.cuh"
#include "tc.cuh"

namespace sq {

namespace {

constexpr float kLog2Pi = 1.8378770664093453f;
constexpr float kSquashEps = 1e-6f;

__device__ __forceinline__ float op_at(const TcOp& op, int r, int k) {
  if (r >= op.rows) return 0.f;
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    if (s >= op.nseg) break;
    const TcSeg& g = op.s[s];
    if (k < g.width) {
      if (g.kcontig) {
        const int64_t row = g.gather ? g.gather[r] : (int64_t)r;
        return g.ptr[row * g.ld + k];
      } else {
        const int64_t kk = g.gather ? g.gather[k] : (int64_t)k;
        return g.ptr[kk * g.ld + r];
      }
    }
    k -= g.width;
  }
  return 0.f;
}

// out[j] = src[(row0 + lane) * ld + c0 + j] for j < ncv, rows < nrow (0 elsewhere): coalesced
// 128-byte row reads into the warp's smem tile, then a transposed register read.
__device__ __forceinline__ void warp_load_tile(const float* src, int ld, int row0, int nrow, int c0, int ncv,
                                               float* T, float (&out)[32]) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
#pragma unroll 4
  for (int i = 0; i < 32; ++i) T[i * 33 + lane] = (i < nrow && lane < ncv) ? src[(int64_t)(row0 + i) * ld + c0 + lane] : 0.f;
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 32; ++j) out[j] = T[lane * 33 + j];
}
// dst[(row0 + lane) * ld + c0 + j] = in[j], through the smem tile (coalesced stores).
__device__ __forceinline__ void warp_store_tile(float* dst, int ld, int row0, int nrow, int c0, int ncv, float* T,
                                                const float (&in)[32]) {
  const int lane = threadIdx.x & 31;
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 32; ++j) T[lane * 33 + j] = in[j];
  __syncwarp();
#pragma unroll 4
  for (int i = 0; i < 32; ++i)
    if (i < nrow && lane < ncv) dst[(int64_t)(row0 + i) * ld + c0 + lane] = T[i * 33 + lane];
}

constexpr int kNT = 256;  // threads per CTA (8 warps)
constexpr int kG = 4;     // 16-byte chunks a thread loads before it converts/stores (MLP)

// 8 consecutive-k elements (r = gr, k = kb .. kb+7) of an operand.  The segment is resolved
// once per chunk; a chunk that straddles a segment boundary or the K tail takes the
// element-wise path.
__device__ __forceinline__ void load_chunk(const TcOp& op, int gr, int kb, int K, float (&f)[8]) {
  if (gr >= op.rows || kb >= K) {
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = 0.f;
    return;
  }
  int kl = kb, s = 0;
  while (s + 1 < op.nseg && kl >= op.s[s].width) kl -= op.s[s++].width;
  const TcSeg& g = op.s[s];
  if (kl + 8 <= g.width && kb + 8 <= K) {
    if (g.kcontig) {
      const int64_t row = g.gather ? __ldg(g.gather + gr) : (int64_t)gr;
      const float* p = g.ptr + row * g.ld + kl;
      if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(p)), y = __ldg(reinterpret_cast<const float4*>(p) + 1);
        f[0] = x.x; f[1] = x.y; f[2] = x.z; f[3] = x.w;
        f[4] = y.x; f[5] = y.y; f[6] = y.z; f[7] = y.w;
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = __ldg(p + i);
      }
    } else if (g.gather) {
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = __ldg(g.ptr + __ldg(g.gather + kl + i) * g.ld + gr);
    } else {
      const float* p = g.ptr + (int64_t)kl * g.ld + gr;
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = __ldg(p + (int64_t)i * g.ld);
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = (kb + i < K) ? op_at(op, gr, kb + i) : 0.f;
}

// Fill one 128B-swizzled K-major tile: rows [r0, r0 + nrows) of `op`, K block [k0, k0 + 64).
// Thread order follows the source's contiguous dimension so warps read whole lines; each
// thread issues the loads of kG chunks before converting and storing any of them.
__device__ __forceinline__ void fill_tile(uint8_t* tile, const TcOp& op, int r0, int nrows, int k0, int K) {
  const int tid = threadIdx.x;
  const int items = nrows * 8;
  const bool kc = op.s[0].kcontig;
  for (int base = tid; base < items; base += kNT * kG) {
    float f[kG][8];
#pragma unroll
    for (int g = 0; g < kG; ++g) {
      const int e = base + g * kNT;
      const int r = kc ? (e >> 3) : (e % nrows), c = kc ? (e & 7) : (e / nrows);
      if (e < items) {
        load_chunk(op, r0 + r, k0 + 8 * c, K, f[g]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) f[g][i] = 0.f;
      }
    }
#pragma unroll
    for (int g = 0; g < kG; ++g) {
      const int e = base + g * kNT;
      if (e >= items) break;
      const int r = kc ? (e >> 3) : (e % nrows), c = kc ? (e & 7) : (e / nrows);
      *reinterpret_cast<uint4*>(tile + tc::sw128_off(r, c)) = tc::pack_bf16x8(f[g]);
    }
  }
}

__global__ void __launch_bounds__(kNT, 1) k_dense_tc(const __grid_constant__ TcBatch b, int stage_bytes) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bars[2];
  __shared__ uint32_t tmem_slot;
  __shared__ float red[2][2][128];  // [stat][column half][tile row]
  __shared__ float xt[8][32][33];    // per-warp transpose tile

  const int tile = blockIdx.x;
  int pi = 0;
  while (pi + 1 < b.nprob && tile >= b.p[pi + 1].tile0) ++pi;
  const TcProb& P = b.p[pi];
  const int lt = tile - P.tile0;
  const int m0 = (lt / P.tiles_n) * 128, n0 = (lt % P.tiles_n) * P.bn;
  const int nreal = min(P.bn, P.N - n0);        // real columns of this tile
  const int nt = (nreal + 15) & ~15;            // MMA N (multiple of 16)
  const int n1 = nt > 256 ? 256 : nt, n2 = nt - n1;
  uint32_t ncols = 32;
  while ((int)ncols < nt) ncols <<= 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (warp == 0) tc::tmem_alloc(&tmem_slot, ncols);
  if (tid == 0) {
    tc::mbar_init(&bars[0], 1);
    tc::mbar_init(&bars[1], 1);
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_slot;

  const int nkb = (P.K + 63) / 64;
  const uint32_t id1 = tc::idesc_bf16(128, n1), id2 = tc::idesc_bf16(128, n2 > 0 ? n2 : 16);
  for (int kb = 0; kb < nkb; ++kb) {
    const int s = kb & 1;
    if (kb >= 2) tc::mbar_wait(&bars[s], ((kb - 2) >> 1) & 1);
    uint8_t* As = smem + s * stage_bytes;
    uint8_t* Bs = As + 16384;
    fill_tile(As, P.A, m0, 128, kb * 64, P.K);
    fill_tile(Bs, P.B, n0, nt, kb * 64, P.K);
    tc::fence_async_smem();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after_sync();
      const uint32_t a0 = tc::smem_u32(As), b0 = tc::smem_u32(Bs);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = tc::sdesc_k128(a0 + 32 * k);
        tc::mma_bf16(tmem, ad, tc::sdesc_k128(b0 + 32 * k), id1, (kb | k) != 0);
        if (n2 > 0) tc::mma_bf16(tmem + 256, ad, tc::sdesc_k128(b0 + 256 * 128 + 32 * k), id2, (kb | k) != 0);
      }
      tc::mma_commit(&bars[s]);
    }
  }
  tc::mbar_wait(&bars[(nkb - 1) & 1], ((nkb - 1) >> 1) & 1);
  tc::fence_after_sync();

  // ---- epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 (= tile rows), column half w / 4.
  // Row-per-thread values are exchanged through a per-warp 32x33 smem tile so that every
  // global load/store of y, xh, out is a coalesced 128-byte row segment.
  const int q = warp & 3, hh = warp >> 2, rl = q * 32 + lane;
  const int row0 = m0 + q * 32;  // first tile row of this warp
  const int r = row0 + lane;
  const bool rv = r < P.M;
  const int nrow = min(32, P.M - row0);
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
  const int epi = P.epi;
  const int N = P.N;
  const int nch = (nreal + 31) / 32;
  float* T = &xt[warp][0][0];
  float v[32], a[32], bb[32];

  if (epi == EPI_STORE || epi == EPI_BIAS || epi == EPI_RELU_MASK) {
    for (int ch = hh; ch < nch; ch += 2) {
      const int c0 = n0 + ch * 32, ncv = min(32, n0 + nreal - c0);
      tc::tmem_ld32(trow + ch * 32, v);
      if (epi == EPI_RELU_MASK) warp_load_tile(P.y, N, row0, nrow, c0, ncv, T, a);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int c = c0 + j;
        if (epi == EPI_BIAS && j < ncv) v[j] += P.bias[c];
        if (epi == EPI_RELU_MASK) v[j] = a[j] > 0.f ? v[j] : 0.f;
      }
      warp_store_tile(P.out + P.out_col0, P.ldo, row0, nrow, c0, ncv, T, v);
    }
  } else if (epi == EPI_LN_RELU || epi == EPI_LN_TANH) {
    float s1 = 0.f;
    for (int ch = hh; ch < nch; ch += 2) {
      tc::tmem_ld32(trow + ch * 32, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int c = ch * 32 + j;
        if (c < N) s1 += v[j] + P.bias[c];
      }
    }
    red[0][hh][rl] = s1;
    __syncthreads();
    const float mean = (red[0][0][rl] + red[0][1][rl]) / (float)N;
    float s2 = 0.f;
    for (int ch = hh; ch < nch; ch += 2) {
      tc::tmem_ld32(trow + ch * 32, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int c = ch * 32 + j;
        if (c < N) {
          const float d = v[j] + P.bias[c] - mean;
          s2 += d * d;
        }
      }
    }
    red[1][hh][rl] = s2;
    __syncthreads();
    const float rs = 1.0f / sqrtf((red[1][0][rl] + red[1][1][rl]) / (float)N + P.ln_eps);
    if (rv && hh == 0 && P.rstd) P.rstd[r] = rs;
    for (int ch = hh; ch < nch; ch += 2) {
      const int c0 = ch * 32, ncv = min(32, N - c0);
      tc::tmem_ld32(trow + ch * 32, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int c = c0 + j < N ? c0 + j : N - 1;
        const float xh = (v[j] + P.bias[c] - mean) * rs;
        const float n = fmaf(xh, P.g[c], P.beta[c]);
        a[j] = xh;
        v[j] = (epi == EPI_LN_RELU) ? fmaxf(n, 0.f) : tanhf(n);
      }
      if (P.xh) warp_store_tile(P.xh, N, row0, nrow, c0, ncv, T, a);
      warp_store_tile(P.out, P.ldo, row0, nrow, c0, ncv, T, v);
    }
  } else if (epi == EPI_BWD_LN_RELU || epi == EPI_BWD_LN_TANH) {
    float s1 = 0.f, s2 = 0.f;
    for (int ch = hh; ch < nch; ch += 2) {
      const int c0 = ch * 32, ncv = min(32, N - c0);
      tc::tmem_ld32(trow + ch * 32, v);
      warp_load_tile(P.y, N, row0, nrow, c0, ncv, T, a);
      warp_load_tile(P.xh, N, row0, nrow, c0, ncv, T, bb);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int c = c0 + j < N ? c0 + j : N - 1;
        const float dn = (epi == EPI_BWD_LN_RELU) ? (a[j] > 0.f ? v[j] : 0.f) : v[j] * (1.f - a[j] * a[j]);
        const float dxh = (c0 + j < N) ? dn * P.g[c] : 0.f;
        s1 += dxh;
        s2 += dxh * bb[j];
        v[j] = dn;
      }
      warp_store_tile(P.out2, N, row0, nrow, c0, ncv, T, v);
    }
    red[0][hh][rl] = s1;
    red[1][hh][rl] = s2;
    __syncthreads();
    const float m1 = (red[0][0][rl] + red[0][1][rl]) / (float)N, m2 = (red[1][0][rl] + red[1][1][rl]) / (float)N;
    const float rs = rv ? P.rstd[r] : 0.f;
    for (int ch = hh; ch < nch; ch += 2) {
      const int c0 = ch * 32, ncv = min(32, N - c0);
      tc::tmem_ld32(trow + ch * 32, v);
      warp_load_tile(P.y, N, row0, nrow, c0, ncv, T, a);
      warp_load_tile(P.xh, N, row0, nrow, c0, ncv, T, bb);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int c = c0 + j < N ? c0 + j : N - 1;
        const float dn = (epi == EPI_BWD_LN_RELU) ? (a[j] > 0.f ? v[j] : 0.f) : v[j] * (1.f - a[j] * a[j]);
        v[j] = rs * (dn * P.g[c] - m1 - bb[j] * m2);
      }
      warp_store_tile(P.out, P.ldo, row0, nrow, c0, ncv, T, v);
    }
  } else if (epi == EPI_TG_FWD) {
    if (hh == 0) {
      tc::tmem_ld32(trow, v);  // N = 2A <= 32
      if (rv) {
        const int A = N / 2;
        float lp = 0.f;
        for (int d = 0; d < A; ++d) {
          const float mu = v[d] + P.bias[d], l = v[A + d] + P.bias[A + d];
          if (P.out) {
            P.out[(int64_t)r * P.ldo + d] = mu;
            P.out[(int64_t)r * P.ldo + A + d] = l;
          }
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
    }
  } else if (epi == EPI_TG_BWD) {
    if (hh == 0) {
      tc::tmem_ld32(trow, v);  // N = A <= 32
      if (rv) {
        const int A = N;
        const float dlp = P.dlogp_scale[0] * P.dlogp_mult;
        for (int d = 0; d < A; ++d) {
          const float mu = P.tg_o[(int64_t)r * 2 * A + d], l = P.tg_o[(int64_t)r * 2 * A + A + d];
          const float tl = tanhf(l);
          const float log_std = P.lo + 0.5f * (P.hi - P.lo) * (tl + 1.f);
          const float sd = expf(log_std);
          const float e = P.eps[(int64_t)r * A + d];
          const float u = fmaf(sd, e, mu);
          const float a1 = tanhf(u);
          const float om = sech2f(u);
          const float du = v[d] * om + dlp * (2.f * a1 * om / (om + kSquashEps));
          const float dls = du * sd * e - dlp;
          P.out[(int64_t)r * P.ldo + d] = du;
          P.out[(int64_t)r * P.ldo + A + d] = dls * 0.5f * (P.hi - P.lo) * sech2f(l);
        }
      }
    }
  }

  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}

// db[n] = sum_m D[m][n]; dg[n] = sum_m DN[m][n] xh[m][n]; dbeta[n] = sum_m DN[m][n]
// One warp per column n, fixed lane-strided order + shuffle tree.
__global__ void __launch_bounds__(256) k_colsums(const __grid_constant__ DwBatch b) {
  const int lane = threadIdx.x & 31;
  int gw = blockIdx.x * 8 + (threadIdx.x >> 5);
  int pi = 0;
  for (; pi < b.nprob; ++pi) {
    if (gw < b.p[pi].N) break;
    gw -= b.p[pi].N;
  }
  if (pi >= b.nprob) return;
  const DwProb& P = b.p[pi];
  const int n = gw;
  float sb = 0.f, sg = 0.f, sbeta = 0.f;
  for (int m = lane; m < P.M; m += 32) {
    sb += P.D[(int64_t)m * P.N + n];
    if (P.DN) {
      const float dn = P.DN[(int64_t)m * P.N + n];
      sg += dn * P.xh[(int64_t)m * P.N + n];
      sbeta += dn;
    }
  }
  sb = warp_sum(sb);
  sg = warp_sum(sg);
  sbeta = warp_sum(sbeta);
  if (lane == 0) {
    if (P.db) P.db[n] = sb;
    if (P.DN) {
      P.dg[n] = sg;
      P.dbeta[n] = sbeta;
    }
  }
}

TcSeg seg_from_a(const ASeg& a) { return TcSeg{a.ptr, a.rows, a.ld, a.width, 1}; }

}  // namespace

void plan_tc(TcBatch& b) {
  int t = 0;
  for (int i = 0; i < b.nprob; ++i) {
    TcProb& p = b.p[i];
    const int npad = (p.N + 15) & ~15;
    if (epi_row_complete(p.epi))
      p.bn = npad;  // full row in one tile (N <= 512)
    else
      p.bn = npad > 128 ? 128 : npad;  // more CTAs for the plain epilogues
    p.tiles_n = (p.N + p.bn - 1) / p.bn;
    p.tile0 = t;
    t += p.tiles_n * ((p.M + 127) / 128);
  }
  b.ntiles = t;
}

int launch_tc(const TcBatch& b, cudaStream_t s) {
  if (b.ntiles == 0) return 0;
  int maxbn = 16;
  for (int i = 0; i < b.nprob; ++i) maxbn = b.p[i].bn > maxbn ? b.p[i].bn : maxbn;
  const int stage_bytes = 16384 + maxbn * 128;
  const size_t smem = 2 * (size_t)stage_bytes + 1024;
  cudaFuncSetAttribute(k_dense_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  note_launch();
  k_dense_tc<<<b.ntiles, kNT, smem, s>>>(b, stage_bytes);
  return (int)cudaGetLastError();
}

// DenseBatch (fp32-path problem description) -> TcBatch: same operands, same epilogues.
int launch_dense_bf16(const DenseBatch& d, cudaStream_t s) {
  TcBatch b;
  b.nprob = d.nprob;
  for (int i = 0; i < d.nprob; ++i) {
    const DenseProb& q = d.p[i];
    TcProb& p = b.p[i];
    memset(&p, 0, sizeof(p));
    p.M = q.M;
    p.N = q.N;
    p.K = q.K;
    p.A.rows = q.M;
    p.A.nseg = q.nA;
    for (int k = 0; k < q.nA; ++k) p.A.s[k] = seg_from_a(q.A[k]);
    p.B.rows = q.N;
    p.B.nseg = q.nB;
    for (int k = 0; k < q.nB; ++k) p.B.s[k] = TcSeg{q.B[k].ptr, nullptr, q.B[k].ld, q.B[k].width, q.B[k].kmajor};
    p.epi = q.epi;
    p.bias = q.bias;
    p.g = q.g;
    p.beta = q.beta;
    p.out = q.out;
    p.ldo = q.ldo;
    p.out_col0 = 0;
    p.out2 = q.out2;
    p.xh = q.xh;
    p.rstd = q.rstd;
    p.y = q.y;
    p.eps = q.eps;
    p.act = q.act;
    p.logp = q.logp;
    p.tg_o = q.tg_o;
    p.dlogp_scale = q.dlogp_scale;
    p.dlogp_mult = q.dlogp_mult;
    p.lo = q.lo;
    p.hi = q.hi;
    p.ln_eps = q.ln_eps;
  }
  plan_tc(b);
  return launch_tc(b, s);
}

// DwBatch -> one TcProb per segment of the layer input X (dW column blocks), + column sums.
int launch_dw_bf16(const DwBatch& d, cudaStream_t s) {
  TcBatch b;
  b.nprob = 0;
  for (int i = 0; i < d.nprob; ++i) {
    const DwProb& q = d.p[i];
    int col0 = 0;
    for (int k = 0; k < q.nA; ++k) {
      TcProb& p = b.p[b.nprob++];
      memset(&p, 0, sizeof(p));
      p.M = q.N;  // output rows = layer out features
      p.N = q.A[k].width;
      p.K = q.M;  // reduction over the batch
      p.A.rows = q.N;
      p.A.nseg = 1;
      p.A.s[0] = TcSeg{q.D, nullptr, q.N, q.M, 0};  // A(n, m) = D[m][n]
      p.B.rows = q.A[k].width;
      p.B.nseg = 1;
      p.B.s[0] = TcSeg{q.A[k].ptr, q.A[k].rows, q.A[k].ld, q.M, 0};  // B(kx, m) = X[gather(m)][kx]
      p.epi = EPI_STORE;
      p.out = q.dW;
      p.ldo = q.K;
      p.out_col0 = col0;
      col0 += q.A[k].width;
    }
  }
  plan_tc(b);
  int e = launch_tc(b, s);
  if (e) return e;
  int ncol = 0;
  for (int i = 0; i < d.nprob; ++i) ncol += d.p[i].N;
  note_launch();
  k_colsums<<<(ncol + 7) / 8, 256, 0, s>>>(d);
  return (int)cudaGetLastError();
}

}  // namespace sq
