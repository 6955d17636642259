// rowchain.cu -- row-complete fused MLP chains (k_rowchain): one CTA owns one 128-row tile of one
// problem and runs every layer of the chain on whole rows, so a LayerNorm layer's row statistics,
// its normalisation and the next layer's input never leave the SM.
//
// Why: in the 4-CTA cluster chain (chain.cu) each 256-wide layer spends ~2 us all-gathering the
// next layer's 64 KB input through distributed shared memory (~20 B/clk per SM) and ~1 us on the
// cross-CTA row statistics; here the epilogue writes the next layer's bf16 input straight into
// this CTA's shared memory (K-major, 128-byte swizzle: the layout TMA would have produced) and the
// tensor core reads it from there.  A 128 x 256 x 256 layer is 2048 tensor-core cycles (~1 us) on
// one SM; the weights (up to 128 KB per layer) stream through a 2-stage TMA ring behind the MMAs.
//
// Roles (320 threads): warps 0-7 epilogue (warp w: TMEM lanes 32 (w % 4) .. +31 = tile rows, columns
// half w / 4 of the layer), warp 8 TMA producer (first input, weight ring), warp 9 MMA issuer.
// Layers: forward LayerNorm (+ReLU / tanh) -- y = act(g x_hat + beta), x_hat and 1/sigma cached for
// the backward; backward LayerNorm dX = dY W with the LayerNorm (+ReLU / tanh) backward of the layer
// below and its bias / affine column partials; last layers: fp32 logits (GE_BIAS_F32) or the
// tanh-Gaussian head (GE_TG_FWD, Q13-Q14).  Each layer's bf16 output can also be stored to global
// memory (TMA store of the shared-memory tile) for the weight-gradient GEMMs.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "chain.cuh"
#include "common.cuh"
#include "gemm_dev.cuh"
#include "tc.cuh"

namespace sq {

namespace {

using namespace gd;
constexpr int kThr = 320;                   // 8 epilogue warps + producer + MMA issuer
constexpr int kEpi = 256;                   // epilogue threads
constexpr int kStages = 2;                  // weight ring depth
constexpr uint32_t kStage = 32768;          // one K block of a <= 256-wide weight: 256 x 64 bf16
constexpr uint32_t kA = 0;                  // 64 KB: the current layer's input (4 K blocks)
constexpr uint32_t kW = 65536;              // weight ring
constexpr uint32_t kX = kW + kStages * kStage;  // 64 KB: x_hat of a backward LayerNorm layer
constexpr float kLog2Pi = 1.8378770664093453f;
constexpr float kSquashEps = 1e-6f;

__device__ __forceinline__ bool is_bwd(int epi) { return epi == GE_BWD_LN_RELU || epi == GE_BWD_LN_TANH; }
__device__ __forceinline__ bool is_ln(int epi) {
  return epi == GE_LN_RELU || epi == GE_LN_TANH || is_bwd(epi);
}
__device__ __forceinline__ uint32_t w_bytes(const CLayer& L) {
  return L.b_mn ? (uint32_t)((L.slice + 63) / 64) * 8192u : (uint32_t)L.slice * 128u;
}

// 32 consecutive bf16 columns [col0, col0 + 32) of tile row `row` of a K-major SW128 tile set
// (K block kb = col / 64 at kb * 16384)
__device__ __forceinline__ void tile_put32(uint8_t* base, int row, int col0, const float (&v)[32]) {
  uint8_t* blk = base + (col0 >> 6) * 16384;
  const int c0 = (col0 & 63) >> 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float f[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = v[8 * i + k];
    *reinterpret_cast<uint4*>(blk + tc::sw128_off(row, c0 + i)) = tc::pack_bf16x8(f);
  }
}
__device__ __forceinline__ void tile_get32(const uint8_t* base, int row, int col0, float (&v)[32]) {
  const uint8_t* blk = base + (col0 >> 6) * 16384;
  const int c0 = (col0 & 63) >> 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint4 u = *reinterpret_cast<const uint4*>(blk + tc::sw128_off(row, c0 + i));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(h[k]);
      v[8 * i + 2 * k] = f.x, v[8 * i + 2 * k + 1] = f.y;
    }
  }
}

__global__ void __launch_bounds__(kThr, 1) k_rowchain(const __grid_constant__ CBatch b) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t a_load, a_epi, acc_full, x_full, w_full[kStages], w_empty[kStages];
  __shared__ uint32_t tmem_slot;
  __shared__ float red[2][2][2][128];                   // [layer parity][statistic][column half][row]
  __shared__ float colacc[4][3][256];                   // backward LayerNorm column partials per row quarter
  __shared__ __align__(16) float s_par[kChainMaxLayers][3][256];  // bias, g, beta of every layer

  int pi = 0;
  while (pi + 1 < b.nprob && (int)blockIdx.x >= b.p[pi + 1].c0) ++pi;
  const CProb& P = b.p[pi];
  const int mt = blockIdx.x - P.c0, m0 = mt * 128;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nl = P.nlayers;
  uint8_t* A = sm + kA;
  uint8_t* X = sm + kX;
  // instrumentation (SQUINT_CHAIN_DBG): globaltimer stamps, 32 per CTA
  auto stamp = [&](int k) {
    if (b.dbg) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      b.dbg[blockIdx.x * 32 + k] = t;
    }
  };
  if (tid == 0) stamp(0);

  if (warp == 0) tc::tmem_alloc(&tmem_slot, 256);
  if (tid == 256) {
    tc::mbar_init(&a_load, 1);
    tc::mbar_init(&a_epi, kEpi / 32);
    tc::mbar_init(&acc_full, 1);
    tc::mbar_init(&x_full, 1);
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&w_full[s], 1);
      tc::mbar_init(&w_empty[s], 1);
    }
    tc::fence_mbar_init();
  }
  if (tid == 288) {
    tc::tma_prefetch_desc(&b.maps[P.amap]);
    for (int l = 0; l < nl; ++l) tc::tma_prefetch_desc(&b.maps[P.L[l].bmap]);
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_slot;
  if (tid == 0) stamp(1);

  if (warp == 8) {
    // ---- TMA producer: the first input, x_hat of a leading backward layer, the weight ring ---------
    if (lane == 0) {
      int it = 0, issued = 0;
      int wl[kChainMaxLayers * 4], wk[kChainMaxLayers * 4], nw = 0;
      for (int l = 0; l < nl; ++l)
        for (int kb = 0; kb < P.L[l].nkb; ++kb) wl[nw] = l, wk[nw++] = kb;
      auto issue_w = [&](int e) {
        const CLayer& L = P.L[wl[e]];
        const int kb = wk[e], st = it % kStages;
        if (it >= kStages) tc::mbar_wait(&w_empty[st], ((it / kStages) - 1) & 1);
        uint8_t* dst = sm + kW + st * kStage;
        tc::mbar_expect_tx(&w_full[st], w_bytes(L));
        if (L.b_mn) {
          for (int j = 0; j * 64 < L.slice; ++j) tc::tma_load_2d(dst + j * 8192, &b.maps[L.bmap], 64 * j, 64 * kb, &w_full[st]);
        } else {
          tc::tma_load_2d(dst, &b.maps[L.bmap], 64 * kb, 0, &w_full[st]);
        }
        ++it;
      };
      // weights are never written by the immediately preceding kernel (b.prefetch_b): the ring's
      // first blocks load before the dependency wait
      if (b.prefetch_b)
        for (; issued < nw && issued < kStages; ++issued) issue_w(issued);
      tc::pdl_wait();
      tc::mbar_expect_tx(&a_load, (uint32_t)P.L[0].nkb * 16384u);
      for (int kb = 0; kb < P.L[0].nkb; ++kb) tc::tma_load_2d(A + kb * 16384, &b.maps[P.amap], 64 * kb, m0, &a_load);
      if (is_bwd(P.L[0].epi)) {
        const CLayer& L = P.L[0];
        tc::mbar_expect_tx(&x_full, (uint32_t)(L.N / 64) * 16384u);
        for (int j = 0; j < L.N / 64; ++j) tc::tma_load_2d(X + j * 16384, &b.maps[L.xmap], 64 * j, m0, &x_full);
      }
      stamp(24);
      for (; issued < nw; ++issued) issue_w(issued);
      stamp(25);
    }
  } else if (warp == 9) {
    // ---- MMA issuer (whole warp, one elected lane issues) -----------------------------------------
    int it = 0;
    const uint32_t a0 = tc::smem_u32(A), w0 = tc::smem_u32(sm + kW);
    for (int l = 0; l < nl; ++l) {
      const CLayer& L = P.L[l];
      if (l == 0)
        tc::mbar_wait(&a_load, 0);
      else
        tc::mbar_wait(&a_epi, (l - 1) & 1);
      tc::fence_after_sync();
      if (lane == 0) stamp(16 + 2 * l);
      const uint32_t id = tc::idesc_bf16_major(128, L.slice, 0, L.b_mn);
      for (int kb = 0; kb < L.nkb; ++kb) {
        const int st = it % kStages;
        tc::mbar_wait(&w_full[st], (it / kStages) & 1);
        tc::fence_after_sync();
        const uint32_t bs = w0 + st * kStage;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = tc::sdesc_sw128(a0 + kb * 16384 + 32 * k, 16, 1024);
          const uint64_t bd = L.b_mn ? tc::sdesc_sw128(bs + 2048 * k, 8192, 1024) : tc::sdesc_sw128(bs + 32 * k, 16, 1024);
          tc::mma_bf16_e(tmem, ad, bd, id, (kb | k) != 0);
        }
        tc::mma_commit_e(&w_empty[st]);
        ++it;
      }
      tc::mma_commit_e(&acc_full);
      if (lane == 0) stamp(17 + 2 * l);
    }
  } else {
    // ---- epilogue warps ------------------------------------------------------------------------------
    const int q = warp & 3, hf = warp >> 2, rl = q * 32 + lane, r = m0 + rl;
    const bool rv = r < P.M;
    const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
    tc::pdl_wait();
    tc::pdl_trigger();
    for (int e = tid; e < nl * 3 * 256; e += kEpi) {
      const int l = e / 768, k = (e / 256) % 3, c = e & 255;
      const CLayer& L = P.L[l];
      const float* src = k == 0 ? L.bias : (k == 1 ? L.g : L.beta);
      s_par[l][k][c] = (src && c < L.N) ? src[c] : 0.f;
    }
    float rs_in[kChainMaxLayers];
#pragma unroll
    for (int l = 0; l < kChainMaxLayers; ++l) rs_in[l] = (l < nl && is_bwd(P.L[l].epi) && rv) ? P.L[l].rstd[r] : 0.f;
    tc::named_bar(1, kEpi);
    if (tid == 0) stamp(2);
    int nbwd = 0;        // backward layers done (x_full phase)
    bool store_pending = false;  // tid 0: a TMA store out of A not yet known to have read it
    for (int l = 0; l < nl; ++l) {
      const CLayer& L = P.L[l];
      const int epi = L.epi;
      const float* bias = s_par[l][0];
      const float* gg = s_par[l][1];
      const float* bb = s_par[l][2];
      const bool last = l == nl - 1;
      tc::mbar_wait(&acc_full, l & 1);
      tc::fence_after_sync();
      if (tid == 0) stamp(3 + 4 * l);
      // A may be rewritten once the previous layer's TMA store has read it
      auto a_free = [&]() {
        if (tid == 0) stamp(4 + 4 * l);
        if (tid == 0 && store_pending) tc::bulk_wait_read<0>();
        store_pending = false;
        tc::named_bar(1, kEpi);
      };
      float v[32], a[32];
      if (epi == GE_LN_RELU || epi == GE_LN_TANH) {
        const int half = L.N / 2, nch = half / 32;
        float s1 = 0.f, s2 = 0.f;
        for (int c = 0; c < nch; ++c) {
          const int col0 = hf * half + 32 * c;
          tc::tmem_ld32(trow + col0, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float u = v[j] + bias[col0 + j];
            s1 += u;
            s2 = fmaf(u, u, s2);
          }
        }
        red[l & 1][0][hf][rl] = s1;
        red[l & 1][1][hf][rl] = s2;
        tc::named_bar(2 + q, 64);
        const float t1 = red[l & 1][0][0][rl] + red[l & 1][0][1][rl];
        const float t2 = red[l & 1][1][0][rl] + red[l & 1][1][1][rl];
        const float mean = t1 / (float)L.N;
        const float rs = rsqrtf(fmaxf(t2 / (float)L.N - mean * mean, 0.f) + L.ln_eps);
        if (rv && hf == 0 && L.rstd) L.rstd[r] = rs;
        a_free();
        for (int c = 0; c < nch; ++c) {
          const int col0 = hf * half + 32 * c;
          tc::tmem_ld32(trow + col0, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float x = (v[j] + bias[col0 + j] - mean) * rs;
            const float n = fmaf(x, gg[col0 + j], bb[col0 + j]);
            a[j] = x;
            v[j] = (epi == GE_LN_RELU) ? fmaxf(n, 0.f) : tanh_fast(n);
          }
          tile_put32(A, rl, col0, v);
          if (L.xh_out && rv) row_st_bf16(L.xh_out + (int64_t)r * L.ld_xh + col0, 32, a);
        }
      } else if (is_bwd(epi)) {
        const int half = L.N / 2, nch = half / 32;
        tc::mbar_wait(&x_full, nbwd & 1);
        float s1 = 0.f, s2 = 0.f;
        for (int c = 0; c < nch; ++c) {
          const int col0 = hf * half + 32 * c;
          tc::tmem_ld32(trow + col0, v);
          tile_get32(X, rl, col0, a);
          float pg[32], pb[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float x = rv ? a[j] : 0.f;
            const float n = fmaf(x, gg[col0 + j], bb[col0 + j]);
            const float dn = rv ? ((epi == GE_BWD_LN_RELU) ? (n > 0.f ? v[j] : 0.f) : v[j] * sech2_fast(n)) : 0.f;
            const float dxh = dn * gg[col0 + j];
            s1 += dxh;
            s2 = fmaf(dxh, x, s2);
            pg[j] = dn * x;
            pb[j] = dn;
          }
          const float cg = colsum32(pg);
          const float cb = colsum32(pb);
          colacc[q][1][col0 + lane] = cg;
          colacc[q][2][col0 + lane] = cb;
        }
        red[l & 1][0][hf][rl] = s1;
        red[l & 1][1][hf][rl] = s2;
        tc::named_bar(2 + q, 64);
        const float m1 = (red[l & 1][0][0][rl] + red[l & 1][0][1][rl]) / (float)L.N;
        const float m2 = (red[l & 1][1][0][rl] + red[l & 1][1][1][rl]) / (float)L.N;
        const float rs = rs_in[l];
        a_free();
        for (int c = 0; c < nch; ++c) {
          const int col0 = hf * half + 32 * c;
          tc::tmem_ld32(trow + col0, v);
          tile_get32(X, rl, col0, a);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float x = rv ? a[j] : 0.f;
            const float n = fmaf(x, gg[col0 + j], bb[col0 + j]);
            const float dn = rv ? ((epi == GE_BWD_LN_RELU) ? (n > 0.f ? v[j] : 0.f) : v[j] * sech2_fast(n)) : 0.f;
            v[j] = rv ? rs * (dn * gg[col0 + j] - m1 - x * m2) : 0.f;
          }
          tile_put32(A, rl, col0, v);
          const float cx = colsum32(v);
          colacc[q][0][col0 + lane] = cx;
        }
        ++nbwd;
      } else if (epi == GE_BIAS_F32) {
        // logits: staged row-major [128][N] fp32 in A (free: the last MMA is done), then stored with
        // consecutive threads on consecutive addresses
        a_free();
        float* T = reinterpret_cast<float*>(A);
        const int half = ((L.slice + 63) / 64) * 32, nch = half / 32;
        for (int c = 0; c < nch; ++c) {
          const int col0 = hf * half + 32 * c;
          tc::tmem_ld32(trow + col0, v);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col0 + j < L.N) T[rl * L.N + col0 + j] = v[j] + bias[col0 + j];
        }
        tc::named_bar(1, kEpi);
        const int rows = min(128, P.M - m0), tot = rows * L.N;
        for (int e = tid; e < tot; e += kEpi) {
          const int rr = e / L.N, cc = e - rr * L.N;
          L.outf[(int64_t)(m0 + rr) * L.ldf + cc] = T[e];
        }
      } else if (epi == GE_TG_FWD) {
        if (hf == 0) {
          float v16[16];
          tc::tmem_ld16(trow, v16);
          if (rv) {
            const int Ad = L.N / 2;
            float lp = 0.f;
            for (int d = 0; d < Ad; ++d) {
              const float mu = v16[d] + bias[d], lg = v16[Ad + d] + bias[Ad + d];
              if (L.tgo) {
                L.tgo[(int64_t)r * 2 * Ad + d] = mu;
                L.tgo[(int64_t)r * 2 * Ad + Ad + d] = lg;
              }
              const float log_std = L.lo + 0.5f * (L.hi - L.lo) * (tanhf(lg) + 1.f);
              const float sd = expf(log_std);
              const float e = L.eps ? L.eps[(int64_t)r * Ad + d] : 0.f;
              const float u = fmaf(sd, e, mu);
              const float at = tanhf(u);
              if (L.act) L.act[(int64_t)r * Ad + d] = at;
              if (L.act_bf) L.act_bf[(int64_t)r * L.ld_act_bf + d] = __float2bfloat16_rn(at);
              lp += -0.5f * e * e - log_std - 0.5f * kLog2Pi - logf(sech2f(u) + kSquashEps);
            }
            if (L.logp) L.logp[r] = lp;
          }
        }
      }
      if (tid == 0) stamp(5 + 4 * l);
      if (!last) {
        // the next layer's input is in A: generic-proxy writes -> visible to the tensor core
        tc::fence_async_smem();
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&a_epi);
      }
      if (is_ln(epi)) {
        tc::named_bar(1, kEpi);  // every epilogue thread finished writing A / x_hat reads / colacc
        if (tid == 0) {
          if (L.omap >= 0) {
            for (int kb = 0; kb < L.N / 64; ++kb) tc::tma_store_2d(&b.maps[L.omap], A + kb * 16384, 64 * kb, m0);
            tc::bulk_commit();
            store_pending = true;
          }
          // x_hat of the next backward layer (the buffer is free now)
          if (l + 1 < nl && is_bwd(P.L[l + 1].epi)) {
            const CLayer& Ln = P.L[l + 1];
            tc::mbar_expect_tx(&x_full, (uint32_t)(Ln.N / 64) * 16384u);
            for (int j = 0; j < Ln.N / 64; ++j) tc::tma_load_2d(X + j * 16384, &b.maps[Ln.xmap], 64 * j, m0, &x_full);
          }
        }
        if (is_bwd(epi) && L.part) {
          for (int e = tid; e < 3 * L.N; e += kEpi) {
            const int kk = e / L.N, c = e - kk * L.N;
            L.part[((int64_t)mt * 3 + kk) * L.N + c] = ((colacc[0][kk][c] + colacc[1][kk][c]) + colacc[2][kk][c]) + colacc[3][kk][c];
          }
          tc::named_bar(1, kEpi);  // colacc is rewritten by the next backward layer
        }
      }
    }
    if (tid == 0) stamp(14);
    if (tid == 0) tc::bulk_wait_all();  // shared memory stays valid until every TMA store read it
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}

}  // namespace

bool rowchain_supported(int hidden) { return hidden % 64 == 0 && hidden <= 256; }

int rowchain_launch(ChainBuilder& cb, cudaStream_t s) {
  CBatch& b = cb.b;
  if (cb.err || b.nprob == 0) return cb.err ? -1 : 0;
  int nm = 0, nt = 0;
  bool any_bwd = false;
  double flops = 0;
  for (int i = 0; i < b.nprob; ++i) {
    CProb& p = b.p[i];
    if (p.nlayers < 1) return -1;
    p.c0 = nt;
    nt += (p.M + 127) / 128;
    if (nm + 1 > kChainMaxMaps || tmap_get(cb.amat[i], 128, &b.maps[nm])) return -1;
    p.amap = nm++;
    for (int l = 0; l < p.nlayers; ++l) {
      CLayer& L = p.L[l];
      const bool bwd = L.epi == GE_BWD_LN_RELU || L.epi == GE_BWD_LN_TANH;
      const bool ln = L.epi == GE_LN_RELU || L.epi == GE_LN_TANH || bwd;
      if (L.nkb > 4 || L.slice > 256 || (ln && (L.N % 64 || L.N > 256)) || (L.epi == GE_BIAS_F32 && L.N > 128) ||
          (L.epi == GE_TG_FWD && (L.N > 16 || l != p.nlayers - 1)) || (l > 0 && p.L[l - 1].N != L.K))
        return -1;
      if (l + 1 < p.nlayers && !ln) return -1;  // only LayerNorm layers feed a next layer
      if (bwd && !L.rstd) return -1;
      if (nm + 3 > kChainMaxMaps) return -1;
      if (tmap_get(cb.wmat[i][l], L.b_mn ? 64 : L.slice, &b.maps[nm])) return -1;
      L.bmap = nm++;
      L.omap = L.xmap = -1;
      L.xh_out = nullptr;
      if (cb.omat[i][l].ptr) {
        if (!ln || tmap_get(cb.omat[i][l], 128, &b.maps[nm])) return -1;
        L.omap = nm++;
      }
      if (bwd) {
        if (!cb.xmat[i][l].ptr || tmap_get(cb.xmat[i][l], 128, &b.maps[nm])) return -1;
        L.xmap = nm++;
        any_bwd = true;
      } else if (cb.xmat[i][l].ptr) {
        L.xh_out = reinterpret_cast<__nv_bfloat16*>(const_cast<void*>(cb.xmat[i][l].ptr));
        L.ld_xh = cb.xmat[i][l].ld;
      }
      flops += 2.0 * p.M * (double)L.N * L.K;
    }
  }
  b.nclusters = nt;
  b.dbg = chain_dbg_for_launch(nt);
  const size_t smem = kX + (any_bwd ? 65536 : 0) + 1024;
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(k_rowchain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kX + 65536 + 1024));
    if (e != cudaSuccess) return (int)e;
    attr = kX + 65536 + 1024;
  }
  note_launch(s, "k_rowchain", flops, 0);
  return (int)launch_pdl(k_rowchain, dim3(nt), dim3(kThr), smem, s, b);
}

}  // namespace sq
