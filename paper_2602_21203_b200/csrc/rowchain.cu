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
constexpr int kEpiWarps = 16;               // epilogue warps: 4 TMEM lane quarters x kParts column parts
constexpr int kParts = kEpiWarps / 4;
constexpr int kEpi = 32 * kEpiWarps;        // epilogue threads
constexpr int kThr = kEpi + 64;             // + TMA producer warp + MMA issuer warp
constexpr int kStages = 2;                  // weight ring depth with a backward layer (X holds x_hat) ...
constexpr int kStagesFwd = 4;               // ... and in forward-only chains (X is two more stages)
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

// Per-layer epilogue state of one thread: row rl of the tile, columns [cp * N / kParts, +N / kParts).
struct EpiCtx {
  const CLayer& L;
  const float* bias;
  const float* g;
  const float* beta;
  uint8_t* A;
  const uint8_t* X;
  uint8_t* Xw;     // forward layers: x_hat staging (the X buffer) stored by TMA, or NULL: staged in A
  const void* xmap;  // forward layers: the x_hat tensor map
  int m0;
  uint32_t trow;
  int rl, r;
  bool rv;
  int q, cp, tid, l;
  bool& store_pending;
  float* red;      // [2 statistics][kParts][128] of this layer parity
  float* colacc;   // [4][3][256]
  float rs = 0.f;  // backward: 1/sigma of the row (forward cache)
};

// A may be rewritten once the previous layer's TMA store has read it
__device__ __forceinline__ void a_free(EpiCtx& E) {
  if (E.tid == 0 && E.store_pending) tc::bulk_wait_read<0>();
  E.store_pending = false;
  tc::named_bar(1, kEpi);
}

// row totals of two statistics over the kParts warps sharing the row (fixed order)
__device__ __forceinline__ void row_total2(EpiCtx& E, float s1, float s2, float& t1, float& t2) {
  E.red[(0 * kParts + E.cp) * 128 + E.rl] = s1;
  E.red[(1 * kParts + E.cp) * 128 + E.rl] = s2;
  tc::named_bar(2 + E.q, 32 * kParts);
  t1 = 0.f, t2 = 0.f;
#pragma unroll
  for (int k = 0; k < kParts; ++k) {
    t1 += E.red[(0 * kParts + k) * 128 + E.rl];
    t2 += E.red[(1 * kParts + k) * 128 + E.rl];
  }
}

__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }

// TMEM -> registers: PART consecutive fp32 columns of this warp's 32 lanes, one wait
template <int PART>
__device__ __forceinline__ void tmem_ld_part(uint32_t taddr, float (&v)[PART]) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
#pragma unroll
  for (int c = 0; c < PART / 32; ++c)
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[32 * c + 0]), "=r"(r[32 * c + 1]), "=r"(r[32 * c + 2]), "=r"(r[32 * c + 3]), "=r"(r[32 * c + 4]),
          "=r"(r[32 * c + 5]), "=r"(r[32 * c + 6]), "=r"(r[32 * c + 7]), "=r"(r[32 * c + 8]), "=r"(r[32 * c + 9]),
          "=r"(r[32 * c + 10]), "=r"(r[32 * c + 11]), "=r"(r[32 * c + 12]), "=r"(r[32 * c + 13]), "=r"(r[32 * c + 14]),
          "=r"(r[32 * c + 15]), "=r"(r[32 * c + 16]), "=r"(r[32 * c + 17]), "=r"(r[32 * c + 18]), "=r"(r[32 * c + 19]),
          "=r"(r[32 * c + 20]), "=r"(r[32 * c + 21]), "=r"(r[32 * c + 22]), "=r"(r[32 * c + 23]), "=r"(r[32 * c + 24]),
          "=r"(r[32 * c + 25]), "=r"(r[32 * c + 26]), "=r"(r[32 * c + 27]), "=r"(r[32 * c + 28]), "=r"(r[32 * c + 29]),
          "=r"(r[32 * c + 30]), "=r"(r[32 * c + 31])
        : "r"(taddr + 32 * c)
        : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// forward LayerNorm layer (one TMEM pass; the row slice stays in registers): y = act(g x_hat + beta),
// x_hat = (u - mean) / sigma, u = acc + bias (Q9, Q10).  y -> A (the next layer's input), x_hat -> X
// (stored to global memory by TMA for the backward), 1/sigma -> global.
template <bool RELU, int PART>
__device__ __forceinline__ void ln_fwd(EpiCtx& E) {
  const CLayer& L = E.L;
  const int c0 = E.cp * PART;
  float u[PART];
  tmem_ld_part<PART>(E.trow + c0, u);
  float s1 = 0.f, s2 = 0.f;
#pragma unroll
  for (int j = 0; j < PART; j += 4) {
    const float4 b4 = ld4(E.bias + c0 + j);
    u[j] += b4.x, u[j + 1] += b4.y, u[j + 2] += b4.z, u[j + 3] += b4.w;
    s1 += (u[j] + u[j + 1]) + (u[j + 2] + u[j + 3]);
    s2 = fmaf(u[j], u[j], fmaf(u[j + 1], u[j + 1], fmaf(u[j + 2], u[j + 2], fmaf(u[j + 3], u[j + 3], s2))));
  }
  float t1, t2;
  row_total2(E, s1, s2, t1, t2);
  const float mean = t1 / (float)L.N;
  const float rs = rsqrtf(fmaxf(t2 / (float)L.N - mean * mean, 0.f) + L.ln_eps);
  const float nmr = -mean * rs;
  if (E.rv && E.cp == 0 && L.rstd) L.rstd[E.r] = rs;
  a_free(E);
  if (L.xmap >= 0 && !E.Xw) {
    // x_hat through A: staged, stored by TMA, and A released before y is written
#pragma unroll
    for (int c8 = 0; c8 < PART / 8; ++c8) {
      float x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fmaf(u[8 * c8 + k], rs, nmr);
      const int col = c0 + 8 * c8;
      *reinterpret_cast<uint4*>(E.A + (uint32_t)(col >> 6) * 16384u + tc::sw128_off(E.rl, (col & 63) >> 3)) =
          tc::pack_bf16x8(x);
    }
    tc::fence_async_smem();
    tc::named_bar(1, kEpi);
    if (E.tid == 0) {
      for (int kb = 0; kb < L.N / 64; ++kb) tc::tma_store_2d(E.xmap, E.A + kb * 16384, 64 * kb, E.m0);
      tc::bulk_commit();
      tc::bulk_wait_read<0>();
    }
    tc::named_bar(1, kEpi);
  }
  // 8 columns (one 16-byte chunk of the swizzled row) at a time
#pragma unroll
  for (int c8 = 0; c8 < PART / 8; ++c8) {
    const int col = c0 + 8 * c8;
    const float4 ga = ld4(E.g + col), gb = ld4(E.g + col + 4), ea = ld4(E.beta + col), eb = ld4(E.beta + col + 4);
    const float gj[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
    const float ej[8] = {ea.x, ea.y, ea.z, ea.w, eb.x, eb.y, eb.z, eb.w};
    float y[8], x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float xx = fmaf(u[8 * c8 + k], rs, nmr);
      const float n = fmaf(xx, gj[k], ej[k]);
      x[k] = xx;
      y[k] = RELU ? fmaxf(n, 0.f) : tanh_fast(n);
    }
    const uint32_t off = (uint32_t)(col >> 6) * 16384u + tc::sw128_off(E.rl, (col & 63) >> 3);
    *reinterpret_cast<uint4*>(E.A + off) = tc::pack_bf16x8(y);
    if (L.xmap >= 0 && E.Xw) *reinterpret_cast<uint4*>(E.Xw + off) = tc::pack_bf16x8(x);
  }
}

// backward LayerNorm layer: acc = dL/dy of y = act(g x_hat + beta) -> dL/du (u = the pre-LN input)
// into A, plus the column partials (sum du, sum dn x_hat, sum dn) of the bias / g / beta gradients.
// x_hat (bf16) comes from X; the accumulator is read twice (pass 2 recomputes dn).
template <bool RELU, int PART>
__device__ __forceinline__ void ln_bwd(EpiCtx& E) {
  const CLayer& L = E.L;
  const int c0 = E.cp * PART;
  const int lane = E.tid & 31;
  float s1 = 0.f, s2 = 0.f;
#pragma unroll 1
  for (int c = 0; c < PART / 32; ++c) {
    const int col0 = c0 + 32 * c;
    float v[32], a[32];
    tc::tmem_ld32(E.trow + col0, v);
    tile_get32(E.X, E.rl, col0, a);
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      const float4 g4 = ld4(E.g + col0 + j), e4 = ld4(E.beta + col0 + j);
      const float gj[4] = {g4.x, g4.y, g4.z, g4.w}, ej[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float x = E.rv ? a[j + k] : 0.f;
        const float n = fmaf(x, gj[k], ej[k]);
        const float d = E.rv ? (RELU ? (n > 0.f ? v[j + k] : 0.f) : v[j + k] * sech2_fast(n)) : 0.f;
        const float dxh = d * gj[k];
        s1 += dxh;
        s2 = fmaf(dxh, x, s2);
        a[j + k] = d * x;
        v[j + k] = d;
      }
    }
    const float cg = colsum32(a);
    const float cb = colsum32(v);
    E.colacc[(E.q * 3 + 1) * 256 + col0 + lane] = cg;
    E.colacc[(E.q * 3 + 2) * 256 + col0 + lane] = cb;
  }
  float m1, m2;
  row_total2(E, s1, s2, m1, m2);
  m1 /= (float)L.N;
  m2 /= (float)L.N;
  const float rs = E.rs;
  a_free(E);
#pragma unroll 1
  for (int c = 0; c < PART / 32; ++c) {
    const int col0 = c0 + 32 * c;
    float v[32], a[32];
    tc::tmem_ld32(E.trow + col0, v);
    tile_get32(E.X, E.rl, col0, a);
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
      const float4 g4 = ld4(E.g + col0 + j), e4 = ld4(E.beta + col0 + j);
      const float gj[4] = {g4.x, g4.y, g4.z, g4.w}, ej[4] = {e4.x, e4.y, e4.z, e4.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float x = E.rv ? a[j + k] : 0.f;
        const float n = fmaf(x, gj[k], ej[k]);
        const float d = E.rv ? (RELU ? (n > 0.f ? v[j + k] : 0.f) : v[j + k] * sech2_fast(n)) : 0.f;
        v[j + k] = E.rv ? rs * (d * gj[k] - m1 - x * m2) : 0.f;
      }
    }
    tile_put32(E.A, E.rl, col0, v);
    const float cx = colsum32(v);
    E.colacc[(E.q * 3 + 0) * 256 + col0 + lane] = cx;
  }
}

__global__ void __launch_bounds__(kThr, 1) k_rowchain(const __grid_constant__ CBatch b) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t a_load, a_epi, acc_full[2], x_full, w_full[kStagesFwd], w_empty[kStagesFwd];
  __shared__ uint32_t tmem_slot;
  __shared__ float red[2][2][kParts][128];              // [layer parity][statistic][column part][row]
  __shared__ float colacc[4 * 3 * 256];                 // backward LayerNorm column partials [row quarter][3][col]
  __shared__ __align__(16) float s_par[kChainMaxLayers][3][256];  // bias, g, beta of every layer

  int pi = 0;
  while (pi + 1 < b.nprob && (int)blockIdx.x >= b.p[pi + 1].c0) ++pi;
  const CProb& P = b.p[pi];
  const int mt = blockIdx.x - P.c0, m0 = mt * 128;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nl = P.nlayers;
  uint8_t* A = sm + kA;
  uint8_t* X = sm + kX;
  bool any_bwd = false;
  for (int l = 0; l < nl; ++l) any_bwd = any_bwd || is_bwd(P.L[l].epi);
  // forward-only chains: a whole 256 x 256 layer of weights in flight (X becomes ring stages 2, 3;
  // x_hat is staged through A); with a backward layer X holds its x_hat
  const int ns = any_bwd ? kStages : kStagesFwd;
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
  if (tid == kEpi) {
    tc::mbar_init(&a_load, 1);
    tc::mbar_init(&a_epi, kEpi / 32);
    tc::mbar_init(&acc_full[0], 1);
    tc::mbar_init(&acc_full[1], 1);
    tc::mbar_init(&x_full, 1);
    for (int s = 0; s < kStagesFwd; ++s) {
      tc::mbar_init(&w_full[s], 1);
      tc::mbar_init(&w_empty[s], 1);
    }
    tc::fence_mbar_init();
  }
  if (tid == kEpi + 32) {
    tc::tma_prefetch_desc(&b.maps[P.amap]);
    for (int l = 0; l < nl; ++l) tc::tma_prefetch_desc(&b.maps[P.L[l].bmap]);
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_slot;
  if (tid == 0) stamp(1);

  if (warp == kEpiWarps) {
    // ---- TMA producer: the first input, x_hat of a leading backward layer, the weight ring ---------
    if (lane == 0) {
      int it = 0, issued = 0;
      int wl[kChainMaxLayers * 4], wk[kChainMaxLayers * 4], nw = 0;
      for (int l = 0; l < nl; ++l)
        for (int kb = 0; kb < P.L[l].nkb; ++kb) wl[nw] = l, wk[nw++] = kb;
      auto issue_w = [&](int e) {
        const CLayer& L = P.L[wl[e]];
        const int kb = wk[e], st = it % ns;
        if (it >= ns) tc::mbar_wait(&w_empty[st], ((it / ns) - 1) & 1);
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
        for (; issued < nw && issued < ns; ++issued) issue_w(issued);
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
  } else if (warp == kEpiWarps + 1) {
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
      // 256-wide LayerNorm layers whose weights are all in flight: the two 128-column halves are issued
      // one after the other and committed separately, so the epilogue warps of half 0 start while the
      // tensor core computes half 1
      const bool split = is_ln(L.epi) && L.slice == 256 && L.nkb <= ns;
      const int nh = split ? 2 : 1, wn = split ? 128 : L.slice;
      const uint32_t id = tc::idesc_bf16_major(128, wn, 0, L.b_mn);
      const int it0 = it;
      for (int h = 0; h < nh; ++h) {
        it = it0;
        for (int kb = 0; kb < L.nkb; ++kb) {
          const int st = it % ns;
          if (h == 0) {
            tc::mbar_wait(&w_full[st], (it / ns) & 1);
            tc::fence_after_sync();
          }
          const uint32_t bs = w0 + st * kStage + (uint32_t)h * (L.b_mn ? 2 * 8192 : 128 * 128);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = tc::sdesc_sw128(a0 + kb * 16384 + 32 * k, 16, 1024);
            const uint64_t bd = L.b_mn ? tc::sdesc_sw128(bs + 2048 * k, 8192, 1024) : tc::sdesc_sw128(bs + 32 * k, 16, 1024);
            tc::mma_bf16_e(tmem + (uint32_t)(h * 128), ad, bd, id, (kb | k) != 0);
          }
          if (h == nh - 1) tc::mma_commit_e(&w_empty[st]);
          ++it;
        }
        tc::mma_commit_e(&acc_full[h]);
      }
      if (nh == 1) tc::mma_commit_e(&acc_full[1]);
      if (lane == 0) stamp(17 + 2 * l);
    }
  } else {
    // ---- epilogue warps ------------------------------------------------------------------------------
    // warp w: TMEM lane quarter q = w % 4 (tile rows 32 q .. 32 q + 31), column part cp = w / 4 of kParts
    const int q = warp & 3, cp = warp >> 2, rl = q * 32 + lane, r = m0 + rl;
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
    float rs_in0 = 0.f, rs_in1 = 0.f, rs_in2 = 0.f;
    if (rv) {
      if (nl > 0 && is_bwd(P.L[0].epi)) rs_in0 = P.L[0].rstd[r];
      if (nl > 1 && is_bwd(P.L[1].epi)) rs_in1 = P.L[1].rstd[r];
      if (nl > 2 && is_bwd(P.L[2].epi)) rs_in2 = P.L[2].rstd[r];
    }
    tc::named_bar(1, kEpi);
    if (tid == 0) stamp(2);
    int nbwd = 0;        // backward layers done (x_full phase)
    bool store_pending = false;  // tid 0: a TMA store out of A not yet known to have read it
    for (int l = 0; l < nl; ++l) {
      const CLayer& L = P.L[l];
      const int epi = L.epi;
      const bool last = l == nl - 1;
      // LayerNorm layers: the warp's column part lies in half cp / (kParts / 2) of the accumulator
      tc::mbar_wait(&acc_full[is_ln(epi) ? cp / (kParts / 2) : 1], l & 1);
      tc::fence_after_sync();
      if (tid == 0) stamp(3 + 4 * l);
      EpiCtx E{L, s_par[l][0], s_par[l][1], s_par[l][2], A, X, any_bwd ? X : nullptr,
               L.xmap >= 0 ? (const void*)&b.maps[L.xmap] : nullptr, m0, trow, rl, r, rv, q, cp, tid, l, store_pending,
               &red[l & 1][0][0][0], colacc};
      const bool p64 = L.N / kParts == 64;
      if (epi == GE_LN_RELU) {
        if (p64) ln_fwd<true, 64>(E); else ln_fwd<true, 32>(E);
      } else if (epi == GE_LN_TANH) {
        if (p64) ln_fwd<false, 64>(E); else ln_fwd<false, 32>(E);
      } else if (is_bwd(epi)) {
        tc::mbar_wait(&x_full, nbwd & 1);
        E.rs = l == 0 ? rs_in0 : (l == 1 ? rs_in1 : rs_in2);
        if (epi == GE_BWD_LN_RELU) {
          if (p64) ln_bwd<true, 64>(E); else ln_bwd<true, 32>(E);
        } else {
          if (p64) ln_bwd<false, 64>(E); else ln_bwd<false, 32>(E);
        }
        ++nbwd;
      } else if (epi == GE_BIAS_F32) {
        // logits: staged row-major [128][N] fp32 in A (free: the last MMA is done), then stored with
        // consecutive threads on consecutive addresses
        a_free(E);
        float* T = reinterpret_cast<float*>(A);
        const int part = ((L.slice + 32 * kParts - 1) / (32 * kParts)) * 32;
        float v[32];
        for (int c = 0; c < part / 32; ++c) {
          const int col0 = cp * part + 32 * c;
          tc::tmem_ld32(trow + col0, v);
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (col0 + j < L.N) T[rl * L.N + col0 + j] = v[j] + E.bias[col0 + j];
        }
        tc::named_bar(1, kEpi);
        const int rows = min(128, P.M - m0);
        if (L.ldf == L.N) {  // the tile's rows are one contiguous block
          float* dst = L.outf + (int64_t)m0 * L.N;
          const int tot = rows * L.N;
          for (int e = tid; e < tot; e += kEpi) dst[e] = T[e];
        } else {
          for (int rr = warp; rr < rows; rr += kEpiWarps)
            for (int cc = lane; cc < L.N; cc += 32) L.outf[(int64_t)(m0 + rr) * L.ldf + cc] = T[rr * L.N + cc];
        }
      } else if (epi == GE_TG_FWD) {
        if (cp == 0) {
          float v16[16];
          tc::tmem_ld16(trow, v16);
          if (rv) {
            const int Ad = L.N / 2;
            float lp = 0.f;
            for (int d = 0; d < Ad; ++d) {
              const float mu = v16[d] + E.bias[d], lg = v16[Ad + d] + E.bias[Ad + d];
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
          if (L.omap >= 0 || (!is_bwd(epi) && L.xmap >= 0 && any_bwd)) {
            if (L.omap >= 0)
              for (int kb = 0; kb < L.N / 64; ++kb) tc::tma_store_2d(&b.maps[L.omap], A + kb * 16384, 64 * kb, m0);
            if (!is_bwd(epi) && L.xmap >= 0 && any_bwd)  // forward x_hat cache staged in X
              for (int kb = 0; kb < L.N / 64; ++kb) tc::tma_store_2d(&b.maps[L.xmap], X + kb * 16384, 64 * kb, m0);
            tc::bulk_commit();
            store_pending = true;
          }
          // x_hat of the next backward layer (the buffer is free now)
          if (l + 1 < nl && is_bwd(P.L[l + 1].epi)) {
            const CLayer& Ln = P.L[l + 1];
            tc::mbar_expect_tx(&x_full, (uint32_t)(Ln.N / 64) * 16384u);
            for (int j2 = 0; j2 < Ln.N / 64; ++j2) tc::tma_load_2d(X + j2 * 16384, &b.maps[Ln.xmap], 64 * j2, m0, &x_full);
          }
        }
        if (is_bwd(epi) && L.part) {
          for (int e = tid; e < 3 * L.N; e += kEpi) {
            const int kk = e / L.N, c = e - kk * L.N;
            float sacc = 0.f;
#pragma unroll
            for (int qq = 0; qq < 4; ++qq) sacc += colacc[(qq * 3 + kk) * 256 + c];
            L.part[((int64_t)mt * 3 + kk) * L.N + c] = sacc;
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

bool rowchain_supported(int hidden) { return hidden % (32 * kParts) == 0 && hidden <= 256; }

int rowchain_launch(ChainBuilder& cb, cudaStream_t s) {
  CBatch& b = cb.b;
  if (cb.err || b.nprob == 0) return cb.err ? -1 : 0;
  int nm = 0, nt = 0;
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
      if (L.nkb > 4 || L.slice > 256 || (ln && (L.N % (32 * kParts) || L.N > 256)) || (L.epi == GE_BIAS_F32 && L.N > 128) ||
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
      if (bwd && !cb.xmat[i][l].ptr) return -1;
      if (cb.xmat[i][l].ptr) {  // backward: x_hat loaded; forward: x_hat stored (both by TMA, 128-row boxes)
        if (!ln || tmap_get(cb.xmat[i][l], 128, &b.maps[nm])) return -1;
        L.xmap = nm++;
      }
      flops += 2.0 * p.M * (double)L.N * L.K;
    }
  }
  b.nclusters = nt;
  b.dbg = chain_dbg_for_launch(nt);
  const size_t smem = kX + 65536 + 1024;
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
