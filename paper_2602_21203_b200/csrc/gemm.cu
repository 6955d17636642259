// gemm.cu -- grouped bf16 GEMM on tcgen05 fed by TMA, with the layers' epilogues fused.
// See gemm.cuh for the problem semantics.
//
// CTA = one 128-row x bn-column output tile, 256 threads:
//   warp 0 lane 0  TMA producer: per 64-wide K block, one A box (K-major 64x128 or two
//                  MN-major 64x64 boxes) and the B boxes into a stage of an S-deep ring,
//                  completion counted in bytes on the stage's "full" mbarrier;
//   warp 1 lane 0  MMA issuer: 4 x tcgen05.mma (K = 16 each, two when bn > 256) per stage,
//                  tcgen05.commit -> the stage's "empty" mbarrier; last commit -> "done";
//   all 8 warps    epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 (= tile rows) for the
//                  column chunks of parity w / 4; row statistics (LayerNorm) are combined
//                  through shared memory; global stores go through a per-warp 32 x 33
//                  transpose tile so each store instruction writes a contiguous row segment.
// Launched with programmatic dependent launch: setup (barrier init, TMEM allocation,
// tensor-map prefetch) overlaps the previous kernel's tail; griddepcontrol.wait precedes
// every read of data a predecessor wrote.  No float atomics: results are deterministic.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "gemm.cuh"
#include "tc.cuh"
#include "gemm_dev.cuh"

namespace sq {

namespace {

using namespace gd;
constexpr int kThreads = 256;
constexpr int kMaxStages = 8;
constexpr int kABytes = 16384;  // 128 x 64 bf16
constexpr float kLog2Pi = 1.8378770664093453f;
constexpr float kSquashEps = 1e-6f;
constexpr int kColaccOff = 4 * 4 * 4096;                  // after the 4 warp pairs' box rings
constexpr int kEpiBytes = kColaccOff + 4 * 3 * 512 * 4;    // + LN-bwd column partials [4][3][512]

int g_pdl = 1;

struct TileGeo {
  int nt, nbox_b, bbytes, bnb;
};
__device__ __forceinline__ TileGeo tile_geo(const GProb& P, int nreal, int b_mn) {
  TileGeo g;
  g.nt = round16(nreal);
  const int bn16 = round16(P.bn);
  if (b_mn) {
    g.bnb = 64;
    g.nbox_b = (g.nt + 63) / 64;
    g.bbytes = g.nbox_b * 8192;
  } else {
    g.bnb = bn16 > 256 ? 256 : bn16;
    g.nbox_b = (g.nt + g.bnb - 1) / g.bnb;
    g.bbytes = g.nbox_b * g.bnb * 128;
  }
  return g;
}

// One template instance per epilogue: each kernel carries only its own epilogue code, which
// keeps the executed instruction footprint inside the instruction caches.
template <int EPI>
__global__ void __launch_bounds__(kThreads, 1) k_gemm(const __grid_constant__ GBatch b) {
  extern __shared__ uint8_t smem_raw[];
  // pointer arithmetic on the __shared__ array (not integer casts) keeps the address space
  // known to the compiler (LDS/STS, no aliasing with global accesses)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full_bar[kMaxStages], empty_bar[kMaxStages], done_bar, ld_bar[8];
  __shared__ uint32_t tmem_slot;
  __shared__ float red[2][2][128];
  __shared__ float cl_red[2][4][128];  // per-row partials of each cluster CTA, pushed by the CTAs
  __shared__ __align__(16) float s_bias[512], s_g[512], s_beta[512];  // per-column epilogue params

  const int tile = blockIdx.x;
  int pi = 0;
  while (pi + 1 < b.nprob && tile >= b.p[pi + 1].tile0) ++pi;
  const GProb& P = b.p[pi];
  const int lt = tile - P.tile0;
  const int mt = lt / P.tiles_n;
  const int m0 = mt * 128, n0 = (lt % P.tiles_n) * P.bn;
  const int nreal = min(P.bn, P.N - n0);
  const int nt = round16(nreal);
  const int n1 = nt > 256 ? 256 : nt, n2 = nt - n1;
  uint32_t ncols = 32;
  while ((int)ncols < nt) ncols <<= 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = b.nstages;
  auto stamp = [&](int k) {
    if (b.dbg && tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      b.dbg[blockIdx.x * 8 + k] = t;
    }
  };
  stamp(0);

  if (warp == 0) tc::tmem_alloc(&tmem_slot, ncols);
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < S; ++i) {
      tc::mbar_init(&full_bar[i], 1);
      tc::mbar_init(&empty_bar[i], 1);
    }
    tc::mbar_init(&done_bar, 1);
    for (int i = 0; i < 8; ++i) tc::mbar_init(&ld_bar[i], 1);
    tc::fence_mbar_init();
  }
  if (warp == 2 && lane < P.nseg) {
    tc::tma_prefetch_desc(&b.maps[P.seg[lane].amap]);
    tc::tma_prefetch_desc(&b.maps[P.seg[lane].bmap]);
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_slot;
  stamp(1);
  int npre = 0;  // stages whose B (weights / long-finished activations) was loaded before the wait
  if (b.prefetch_b && warp == 0 && lane == 0) {
    // B never comes from the immediately preceding kernel (host contract), and every earlier
    // kernel has completed: the preceding kernel triggers its dependents only after its own wait.
    int kb = 0;
    for (int s = 0; s < P.nseg && kb < S; ++s) {
      const GSeg& G = P.seg[s];
      const TileGeo geo = tile_geo(P, nreal, G.b_mn);
      for (int l = 0; l < G.nkb && kb < S; ++l, ++kb) {
        uint8_t* Bs = smem + kb * b.stage_bytes + kABytes;
        tc::mbar_expect_tx(&full_bar[kb], kABytes + geo.bbytes);
        for (int i = 0; i < geo.nbox_b; ++i) {
          if (!G.b_mn)
            tc::tma_load_2d(Bs + i * geo.bnb * 128, &b.maps[G.bmap], G.b_k + 64 * l, P.b_n + n0 + geo.bnb * i, &full_bar[kb]);
          else
            tc::tma_load_2d(Bs + i * 8192, &b.maps[G.bmap], P.b_n + n0 + 64 * i, G.b_k + 64 * l, &full_bar[kb]);
        }
      }
    }
    npre = kb;
  }
  tc::pdl_wait();
  tc::pdl_trigger();
  stamp(2);
  // per-column epilogue parameters -> smem (overlaps the main loop; read after the done barrier)
  if (warp >= 2) {
    for (int c = tid - 64; c < nt; c += kThreads - 64) {
      const int gc = n0 + c;
      const bool ok = gc < P.N;
      s_bias[c] = (ok && P.bias) ? P.bias[gc] : 0.f;
      s_g[c] = (ok && P.g) ? P.g[gc] : 0.f;
      s_beta[c] = (ok && P.beta) ? P.beta[gc] : 0.f;
    }
  }

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    int kb = 0;
    for (int s = 0; s < P.nseg; ++s) {
      const GSeg& G = P.seg[s];
      const TileGeo geo = tile_geo(P, nreal, G.b_mn);
      const void* am = &b.maps[G.amap];
      const void* bm = &b.maps[G.bmap];
      for (int l = 0; l < G.nkb; ++l, ++kb) {
        const int st = kb % S;
        if (kb >= S) tc::mbar_wait(&empty_bar[st], ((kb / S) - 1) & 1);
        uint8_t* As = smem + st * b.stage_bytes;
        uint8_t* Bs = As + kABytes;
        const bool pre = kb < npre;  // B already in flight, transaction bytes already expected
        if (!pre) tc::mbar_expect_tx(&full_bar[st], kABytes + geo.bbytes);
        const int kc = 64 * l;
        if (!G.a_mn) {
          tc::tma_load_2d(As, am, G.a_k + kc, P.a_m + m0, &full_bar[st]);
        } else {
          tc::tma_load_2d(As, am, P.a_m + m0, G.a_k + kc, &full_bar[st]);
          tc::tma_load_2d(As + 8192, am, P.a_m + m0 + 64, G.a_k + kc, &full_bar[st]);
        }
        for (int i = 0; i < geo.nbox_b && !pre; ++i) {
          if (!G.b_mn)
            tc::tma_load_2d(Bs + i * geo.bnb * 128, bm, G.b_k + kc, P.b_n + n0 + geo.bnb * i, &full_bar[st]);
          else
            tc::tma_load_2d(Bs + i * 8192, bm, P.b_n + n0 + 64 * i, G.b_k + kc, &full_bar[st]);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    int kb = 0;
    for (int s = 0; s < P.nseg; ++s) {
      const GSeg& G = P.seg[s];
      const uint32_t id1 = tc::idesc_bf16_major(128, n1, G.a_mn, G.b_mn);
      const uint32_t id2 = tc::idesc_bf16_major(128, n2 > 0 ? n2 : 16, G.a_mn, G.b_mn);
      for (int l = 0; l < G.nkb; ++l, ++kb) {
        const int st = kb % S;
        tc::mbar_wait(&full_bar[st], (kb / S) & 1);
        tc::fence_after_sync();
        const uint32_t a0 = tc::smem_u32(smem + st * b.stage_bytes), b0 = a0 + kABytes;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = G.a_mn ? tc::sdesc_sw128(a0 + 2048 * k, 8192, 1024) : tc::sdesc_sw128(a0 + 32 * k, 16, 1024);
          const uint64_t bd = G.b_mn ? tc::sdesc_sw128(b0 + 2048 * k, 8192, 1024) : tc::sdesc_sw128(b0 + 32 * k, 16, 1024);
          const uint32_t acc = (kb | k) != 0;
          tc::mma_bf16(tmem, ad, bd, id1, acc);
          if (n2 > 0) {
            const uint64_t bd2 = G.b_mn ? tc::sdesc_sw128(b0 + 32768 + 2048 * k, 8192, 1024)
                                        : tc::sdesc_sw128(b0 + 32768 + 32 * k, 16, 1024);
            tc::mma_bf16(tmem + 256, ad, bd2, id2, acc);
          }
        }
        tc::mma_commit(&empty_bar[st]);
      }
    }
    tc::mma_commit(&done_bar);
  }
  __syncwarp();
  tc::mbar_wait(&done_bar, 0);
  tc::fence_after_sync();
  __syncthreads();  // s_bias / s_g / s_beta visible
  stamp(3);

  // ---------------- epilogue ----------------
  const int q = warp & 3, hh = warp >> 2, rl = q * 32 + lane;
  const int row0 = m0 + q * 32;
  const int r = row0 + lane;
  const bool rv = r < P.M;
  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
  const int N = P.N;
  const int nch = (nreal + 31) / 32;       // 32-column chunks of the tile
  const int ngrp = (nreal + 63) / 64;      // 64-column groups (TMA boxes); warp hh owns groups hh, hh+2, ...
  uint8_t* pslots = smem + q * 4 * kSlotBytes;  // the warp pair's ring of 4 boxes
  float v[32], a[32];
  // per-row totals over the whole LayerNorm row: the two column halves of this CTA (smem), then
  // the CTAs of the cluster (distributed shared memory, summed in rank order: every CTA gets the
  // same bits)
  // per-row totals over the whole LayerNorm row: the two column halves of this CTA (smem), then
  // the CTAs of the cluster.  Push model: every CTA stores its row partials into each peer's
  // cl_red[k][rank] (distributed shared memory), one cluster barrier, then local reads summed in
  // rank order (every CTA gets the same bits; no remote access after the barrier).
  auto row_total2 = [&](float p1, float p2, float& t1, float& t2) {
    red[0][hh][rl] = p1;
    red[1][hh][rl] = p2;
    __syncthreads();
    t1 = red[0][0][rl] + red[0][1][rl];
    t2 = red[1][0][rl] + red[1][1][rl];
    if (b.cs > 1) {
      const uint32_t me = (uint32_t)(blockIdx.x % b.cs);
      if (hh == 0)
        for (int rk = 0; rk < b.cs; ++rk) {
          tc::dsmem_st(&cl_red[0][me][rl], (uint32_t)rk, t1);
          tc::dsmem_st(&cl_red[1][me][rl], (uint32_t)rk, t2);
        }
      tc::cluster_sync();
      t1 = t2 = 0.f;
      for (int rk = 0; rk < b.cs; ++rk) {
        t1 += cl_red[0][rk][rl];
        t2 += cl_red[1][rk][rl];
      }
    }
  };

  if constexpr (EPI == GE_BIAS_F32 || EPI == GE_DW) {
    for (int ch = hh; ch < nch; ch += 2) {
      const int c0 = n0 + ch * 32, ncv = min(32, n0 + nreal - c0);
      tc::tmem_ld32(trow + ch * 32, v);
      if constexpr (EPI == GE_BIAS_F32) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += s_bias[ch * 32 + j];
        if (rv) row_st_f32(P.outf + (int64_t)r * P.ldf + c0, ncv, v);
      } else {
        if (rv) {
          if (P.perm_c == 0) {
            row_st_f32(P.outf + (int64_t)r * P.ldf + c0, ncv, v);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int c = c0 + j, pix = c / P.perm_c, chn = c - pix * P.perm_c;
              if (j < ncv) P.outf[(int64_t)r * P.ldf + chn * P.perm_p + pix] = v[j];
            }
          }
        }
      }
    }
    if constexpr (EPI == GE_DW) {
      if (n0 == 0 && hh == 0 && rv) {
        float db = 0.f, dg = 0.f, dbe = 0.f;
        if (P.part_in) {
          for (int t = 0; t < P.part_tiles; ++t) {
            const float* pp = P.part_in + (int64_t)t * 3 * P.M;
            db += pp[r];
            dg += pp[P.M + r];
            dbe += pp[2 * P.M + r];
          }
        } else if (P.colsum) {
          float acc4[4] = {0.f, 0.f, 0.f, 0.f};
          int i = 0;
          for (; i + 4 <= P.colsum_rows; i += 4)
#pragma unroll
            for (int u = 0; u < 4; ++u) acc4[u] += __bfloat162float(P.colsum[(int64_t)(i + u) * P.ld_colsum + r]);
          for (; i < P.colsum_rows; ++i) acc4[0] += __bfloat162float(P.colsum[(int64_t)i * P.ld_colsum + r]);
          db = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);
        }
        if (P.db) P.db[r] = db;
        if (P.dg) P.dg[r] = dg;
        if (P.dbeta) P.dbeta[r] = dbe;
      }
    }
  } else if constexpr (EPI == GE_RELU_MASK) {
    // mask-source boxes by TMA (loaded once per warp pair), masked gradient written in place,
    // stored by TMA; warp hh of pair q owns the 32-column half hh of each 64-column box
    for (int g = 0; g < ngrp; ++g) {
      uint8_t* sl = pslots + (g & 3) * kSlotBytes;
      if (g >= 4) {
        if (hh == 0 && lane == 0) tc::bulk_wait_read<3>();
        tc::named_bar(1 + q, 64);
      }
      if (hh == 0 && lane == 0) {
        tc::mbar_expect_tx(&ld_bar[q], kSlotBytes);
        tc::tma_load_2d(sl, &b.maps[P.ymap], n0 + g * 64, row0, &ld_bar[q]);
      }
      tc::mbar_wait(&ld_bar[q], g & 1);
      const int ch = 2 * g + hh;
      if (ch < nch) {
        tc::tmem_ld32(trow + ch * 32, v);
        box_get(sl, hh, a);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = a[j] > 0.f ? v[j] : 0.f;
        box_put(sl, hh, v);
      }
      pair_store(sl, &b.maps[P.omap], n0 + g * 64, row0, q, hh);
    }
  } else if constexpr (EPI == GE_LN_RELU || EPI == GE_LN_TANH) {
    // one pass for the row moments (bf16 outputs: E[u^2] - mean^2 in fp32 is ample), one pass to
    // normalise and store
    float s1 = 0.f, s2 = 0.f;
    for (int ch = hh; ch < nch; ch += 2) {
      tc::tmem_ld32(trow + ch * 32, v);
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int cc = ch * 32 + j;
        const float u = v[j] + s_bias[cc];
        if (cc < nreal) s1 += u, s2 += u * u;
      }
    }
    stamp(5);
    float t1, t2;
    row_total2(s1, s2, t1, t2);
    stamp(6);
    const float mean = t1 / (float)N;
    const float rs = rsqrtf(fmaxf(t2 / (float)N - mean * mean, 0.f) + P.ln_eps);
    if (rv && hh == 0 && n0 == 0 && P.rstd) P.rstd[r] = rs;
    const bool tma_out = (N & 7) == 0;
    for (int g = 0; g < ngrp; ++g) {
      uint8_t* sy = pslots + ((2 * g) & 3) * kSlotBytes;
      uint8_t* sx = pslots + ((2 * g + 1) & 3) * kSlotBytes;
      if (g >= 2) {  // the pair's slots of group g-2 must have been read by the TMA unit
        if (hh == 0 && lane == 0) tc::bulk_wait_read<2>();
        tc::named_bar(1 + q, 64);
      }
      const int ch = 2 * g + hh;
      if (ch < nch) {
        tc::tmem_ld32(trow + ch * 32, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int cc = ch * 32 + j;
          const float x = (v[j] + s_bias[cc] - mean) * rs;
          const float n = fmaf(x, s_g[cc], s_beta[cc]);
          a[j] = x;
          v[j] = (EPI == GE_LN_RELU) ? fmaxf(n, 0.f) : tanh_fast(n);
        }
        // TMA stores are masked at 16-byte granularity: an output block whose last column is
        // not 8-aligned (the projection's z inside [z | s | a]) is stored directly instead.
        if (tma_out) box_put(sy, hh, v);
        else if (rv) row_st_bf16(P.out + (int64_t)r * P.ldo + n0 + ch * 32, min(32, nreal - ch * 32), v);
        if (P.xh) box_put(sx, hh, a);
      }
      if (tma_out) pair_store(sy, &b.maps[P.omap], n0 + g * 64, row0, q, hh);
      if (P.xh) pair_store(sx, &b.maps[P.xmap], n0 + g * 64, row0, q, hh);
    }
  } else if constexpr (EPI == GE_BWD_LN_RELU || EPI == GE_BWD_LN_TANH) {
    float* colacc = reinterpret_cast<float*>(smem + kColaccOff);  // [4][3][512]
    // the pair's x_hat boxes (<= 4) by TMA on one transaction barrier
    if (hh == 0 && lane == 0) {
      tc::mbar_expect_tx(&ld_bar[q], ngrp * kSlotBytes);
      for (int g = 0; g < ngrp; ++g)
        tc::tma_load_2d(pslots + g * kSlotBytes, &b.maps[P.xmap], n0 + g * 64, row0, &ld_bar[q]);
    }
    tc::mbar_wait(&ld_bar[q], 0);
    float s1 = 0.f, s2 = 0.f;
    for (int g = 0; g < ngrp; ++g) {
      const int ch = 2 * g + hh;
      if (ch < nch) {
        const int c0 = ch * 32, ncv = min(32, nreal - c0);
        tc::tmem_ld32(trow + ch * 32, v);
        box_get(pslots + g * kSlotBytes, hh, a);
        float pg[32], pb[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int cc = c0 + j;
          const bool ok = rv && (j < ncv);
          const float x = ok ? a[j] : 0.f;
          const float n = fmaf(x, s_g[cc], s_beta[cc]);
          const float dn = ok ? ((EPI == GE_BWD_LN_RELU) ? (n > 0.f ? v[j] : 0.f) : v[j] * sech2_fast(n)) : 0.f;
          const float dxh = dn * s_g[cc];
          s1 += dxh;
          s2 += dxh * x;
          pg[j] = dn * x;
          pb[j] = dn;
        }
        const float cg = colsum32(pg);
        const float cb = colsum32(pb);
        colacc[(q * 3 + 1) * 512 + c0 + lane] = cg;
        colacc[(q * 3 + 2) * 512 + c0 + lane] = cb;
      }
    }
    float m1, m2;
    row_total2(s1, s2, m1, m2);
    m1 /= (float)N;
    m2 /= (float)N;
    const float rs = rv ? P.rstd[r] : 0.f;
    for (int g = 0; g < ngrp; ++g) {
      uint8_t* sl = pslots + g * kSlotBytes;
      const int ch = 2 * g + hh;
      if (ch < nch) {
        const int c0 = ch * 32, ncv = min(32, nreal - c0);
        tc::tmem_ld32(trow + ch * 32, v);
        box_get(sl, hh, a);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int cc = c0 + j;
          const bool ok = rv && (j < ncv);
          const float x = ok ? a[j] : 0.f;
          const float n = fmaf(x, s_g[cc], s_beta[cc]);
          const float dn = ok ? ((EPI == GE_BWD_LN_RELU) ? (n > 0.f ? v[j] : 0.f) : v[j] * sech2_fast(n)) : 0.f;
          v[j] = ok ? rs * (dn * s_g[cc] - m1 - x * m2) : 0.f;
          a[j] = v[j];
        }
        box_put(sl, hh, v);
        const float cx = colsum32(a);
        colacc[(q * 3 + 0) * 512 + c0 + lane] = cx;
      }
      pair_store(sl, &b.maps[P.omap], n0 + g * 64, row0, q, hh);
    }
    __syncthreads();
    if (P.part) {
      for (int e = tid; e < 3 * nreal; e += kThreads) {
        const int kk = e / nreal, c = e - kk * nreal;
        float s = 0.f;
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) s += colacc[(qq * 3 + kk) * 512 + c];
        P.part[((int64_t)mt * 3 + kk) * N + n0 + c] = s;
      }
    }
  } else if constexpr (EPI == GE_TG_FWD) {
    float* T = reinterpret_cast<float*>(smem) + warp * 32 * 33;
    if (hh == 0) {
      tc::tmem_ld32(trow, v);  // N = 2A <= 32
      // row -> smem so [mu | l] can be indexed by the runtime A (no local-memory arrays)
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; ++j) T[lane * 33 + j] = v[j];
      __syncwarp();
      const float* o = T + lane * 33;
      if (rv) {
        const int A = N / 2;
        float lp = 0.f;
        for (int d = 0; d < A; ++d) {
          const float mu = o[d] + s_bias[d], l = o[A + d] + s_bias[A + d];
          if (P.tgo) {
            P.tgo[(int64_t)r * 2 * A + d] = mu;
            P.tgo[(int64_t)r * 2 * A + A + d] = l;
          }
          const float tl = tanhf(l);
          const float log_std = P.lo + 0.5f * (P.hi - P.lo) * (tl + 1.f);
          const float sd = expf(log_std);
          const float e = P.eps ? P.eps[(int64_t)r * A + d] : 0.f;
          const float u = fmaf(sd, e, mu);
          const float at = tanhf(u);
          if (P.act) P.act[(int64_t)r * A + d] = at;
          if (P.act_bf) P.act_bf[(int64_t)r * P.ld_act_bf + d] = __float2bfloat16_rn(at);
          lp += -0.5f * e * e - log_std - 0.5f * kLog2Pi - logf(sech2f(u) + kSquashEps);
        }
        if (P.logp) P.logp[r] = lp;
      }
    }
  } else if constexpr (EPI == GE_TG_BWD) {
    float* T = reinterpret_cast<float*>(smem) + warp * 32 * 33;
    if (hh == 0) {
      tc::tmem_ld32(trow, v);  // acc_col0 + A <= 32
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; ++j) T[lane * 33 + j] = v[j];
      __syncwarp();
      const float* o = T + lane * 33 + P.acc_col0;
      if (rv) {
        const int A = N - P.acc_col0;
        const float dlp = P.dlogp_scale[0];
        for (int d = 0; d < A; ++d) {
          const float mu = P.tgo[(int64_t)r * 2 * A + d], l = P.tgo[(int64_t)r * 2 * A + A + d];
          const float tl = tanhf(l);
          const float log_std = P.lo + 0.5f * (P.hi - P.lo) * (tl + 1.f);
          const float sd = expf(log_std);
          const float e = P.eps[(int64_t)r * A + d];
          const float u = fmaf(sd, e, mu);
          const float a1 = tanhf(u);
          const float om = sech2f(u);
          const float du = o[d] * om + dlp * (2.f * a1 * om / (om + kSquashEps));
          const float dls = du * sd * e - dlp;
          P.out[(int64_t)r * P.ldo + d] = __float2bfloat16_rn(du);
          P.out[(int64_t)r * P.ldo + A + d] = __float2bfloat16_rn(dls * 0.5f * (P.hi - P.lo) * sech2f(l));
        }
      }
    }
  }

  stamp(7);
  if (lane == 0) tc::bulk_wait_read<0>();  // TMA stores have finished reading this CTA's smem
  tc::fence_before_sync();
  __syncthreads();
  stamp(4);
  if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}

typedef void (*GemmKernel)(GBatch);
GemmKernel kernel_for(int epi) {
  switch (epi) {
    case GE_LN_RELU: return k_gemm<GE_LN_RELU>;
    case GE_LN_TANH: return k_gemm<GE_LN_TANH>;
    case GE_BIAS_F32: return k_gemm<GE_BIAS_F32>;
    case GE_TG_FWD: return k_gemm<GE_TG_FWD>;
    case GE_BWD_LN_RELU: return k_gemm<GE_BWD_LN_RELU>;
    case GE_BWD_LN_TANH: return k_gemm<GE_BWD_LN_TANH>;
    case GE_RELU_MASK: return k_gemm<GE_RELU_MASK>;
    case GE_TG_BWD: return k_gemm<GE_TG_BWD>;
    case GE_DW: return k_gemm<GE_DW>;
  }
  return nullptr;
}

bool row_complete(int e) {
  return e == GE_LN_RELU || e == GE_LN_TANH || e == GE_BWD_LN_RELU || e == GE_BWD_LN_TANH || e == GE_TG_FWD ||
         e == GE_TG_BWD;
}

int host_bbytes(const GProb& p, int b_mn) {
  const int bn16 = (p.bn + 15) & ~15;
  if (b_mn) return ((bn16 + 63) / 64) * 8192;
  const int bnb = bn16 > 256 ? 256 : bn16;
  return ((bn16 + bnb - 1) / bnb) * bnb * 128;
}

}  // namespace

void gemm_set_pdl(int on) { g_pdl = on; }

static unsigned long long* g_dbg_dev = nullptr;
static int g_dbg_tiles = 0;
int gemm_debug_times(unsigned long long* host, int max_entries) {
  if (!g_dbg_dev) return 0;
  cudaDeviceSynchronize();
  const int n = g_dbg_tiles * 8 < max_entries ? g_dbg_tiles * 8 : max_entries;
  cudaMemcpy(host, g_dbg_dev, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return n;
}

GProb& GemmBuilder::add(int M, int N, int epi) {
  if (b.nprob >= kGemmMaxProb) {
    err = 1;
    return b.p[kGemmMaxProb - 1];
  }
  GProb& p = b.p[b.nprob++];
  memset(&p, 0, sizeof(p));
  p.M = M;
  p.N = N;
  p.epi = epi;
  p.ln_eps = 1e-5f;
  return p;
}

void GemmBuilder::seg(GProb& p, const Mat& A, int a_mn, int a_k, const Mat& Bm, int b_mn, int b_k, int K) {
  if (p.nseg >= 3) {
    err = 2;
    return;
  }
  const int pi = (int)(&p - b.p);
  GSeg& s = p.seg[p.nseg];
  segA[pi][p.nseg] = A;
  segB[pi][p.nseg] = Bm;
  s.a_mn = a_mn;
  s.b_mn = b_mn;
  s.a_k = a_k;
  s.b_k = b_k;
  s.nkb = (K + 63) / 64;
  s.k = K;
  p.nseg++;
}

int gemm_launch(GemmBuilder& gb, cudaStream_t s) {
  GBatch& b = gb.b;
  if (gb.err) return -1;
  if (b.nprob == 0) return 0;
  // plan tiles.  LayerNorm epilogues need whole rows: with N >= 128 the row is split over a
  // cluster of cs CTAs of 64-column multiples (more SMs share the epilogue work).
  const int epi0 = b.p[0].epi;
  const bool ln_launch = epi0 == GE_LN_RELU || epi0 == GE_LN_TANH || epi0 == GE_BWD_LN_RELU || epi0 == GE_BWD_LN_TANH;
  b.cs = 1;
  if (ln_launch) {
    int cs = 8;
    for (int i = 0; i < b.nprob; ++i) {
      const int n = b.p[i].N;
      const int c = n >= 256 && n % 256 == 0 ? 4 : (n >= 128 && n % 128 == 0 ? 2 : 1);
      cs = c < cs ? c : cs;
    }
    static const bool no_cluster = getenv("SQUINT_NO_CLUSTER") != nullptr;
    b.cs = no_cluster ? 1 : cs;
  }
  int t = 0, bmax = 0;
  for (int i = 0; i < b.nprob; ++i) {
    GProb& p = b.p[i];
    if (p.M < 1 || p.N < 1 || p.nseg < 1) return -1;
    for (int k = 0; k < p.nseg; ++k)  // TMA box starts along a contiguous dim: 16-byte aligned
      if ((p.seg[k].a_mn && (p.a_m & 7)) || (p.seg[k].b_mn && (p.b_n & 7)) || (p.seg[k].a_k & 63) ||
          (p.seg[k].b_k & 63))
        return -1;
    const int n16 = (p.N + 15) & ~15;
    if (row_complete(p.epi)) {
      if (n16 > 512) return -1;
      p.bn = b.cs > 1 ? p.N / b.cs : n16;
    } else if (p.epi == GE_DW) {
      p.bn = n16 >= 256 ? 64 : (n16 > 128 ? 128 : n16);
    } else {
      p.bn = n16 > 128 ? 128 : n16;
    }
    p.tiles_n = (p.N + p.bn - 1) / p.bn;
    p.tile0 = t;
    t += p.tiles_n * ((p.M + 127) / 128);
    for (int k = 0; k < p.nseg; ++k) {
      const int bb = host_bbytes(p, p.seg[k].b_mn);
      bmax = bb > bmax ? bb : bmax;
    }
  }
  b.ntiles = t;
  b.stage_bytes = kABytes + bmax;
  int S = (200 * 1024) / b.stage_bytes;
  S = S > kMaxStages ? kMaxStages : S;
  int maxkb = 0;  // no more stages than K blocks
  for (int i = 0; i < b.nprob; ++i) {
    int k = 0;
    for (int j = 0; j < b.p[i].nseg; ++j) k += b.p[i].seg[j].nkb;
    maxkb = k > maxkb ? k : maxkb;
  }
  S = S > maxkb ? maxkb : S;
  S = S < 2 ? 2 : S;
  if ((size_t)S * b.stage_bytes > 200 * 1024) return -1;
  b.nstages = S;
  // tensor maps
  b.nmaps = 0;
  for (int i = 0; i < b.nprob; ++i) {
    GProb& p = b.p[i];
    const int bn16 = (p.bn + 15) & ~15;
    for (int k = 0; k < p.nseg; ++k) {
      GSeg& g = p.seg[k];
      if (b.nmaps + 2 > kGemmMaxMaps) return -1;
      if (tmap_get(gb.segA[i][k], g.a_mn ? 64 : 128, &b.maps[b.nmaps])) return -1;
      g.amap = b.nmaps++;
      if (tmap_get(gb.segB[i][k], g.b_mn ? 64 : (bn16 > 256 ? 256 : bn16), &b.maps[b.nmaps])) return -1;
      g.bmap = b.nmaps++;
    }
  }
  // epilogue tensor maps (64-column x 32-row bf16 boxes)
  for (int i = 0; i < b.nprob; ++i) {
    GProb& p = b.p[i];
    p.omap = p.xmap = p.ymap = -1;
    const bool ln = p.epi == GE_LN_RELU || p.epi == GE_LN_TANH;
    const bool bwd = p.epi == GE_BWD_LN_RELU || p.epi == GE_BWD_LN_TANH;
    if (ln || bwd || p.epi == GE_RELU_MASK) {
      if (b.nmaps + 3 > kGemmMaxMaps || !p.out) return -1;
      if (tmap_get(Mat{p.out, p.M, p.N, p.ldo}, 32, &b.maps[b.nmaps])) return -1;
      p.omap = b.nmaps++;
    }
    if ((ln && p.xh) || bwd) {
      if (!p.xh || tmap_get(Mat{p.xh, p.M, p.N, p.ldx}, 32, &b.maps[b.nmaps])) return -1;
      p.xmap = b.nmaps++;
    }
    if (p.epi == GE_RELU_MASK) {
      if (!p.y || tmap_get(Mat{p.y, p.M, p.N, p.ldy}, 32, &b.maps[b.nmaps])) return -1;
      p.ymap = b.nmaps++;
    }
  }
  size_t smem = (size_t)S * b.stage_bytes;
  if (smem < (size_t)kEpiBytes) smem = kEpiBytes;
  smem += 1024;
  const int epi = b.p[0].epi;
  for (int i = 1; i < b.nprob; ++i)
    if (b.p[i].epi != epi) return -1;  // one epilogue kind per launch (template instance)
  GemmKernel kern = kernel_for(epi);
  if (!kern) return -1;
  static size_t attr_smem[16] = {0};  // opt-in limit set so far per instance
  if (smem > attr_smem[epi]) {
    cudaError_t ae = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ae != cudaSuccess) return (int)ae;
    attr_smem[epi] = smem;
  }
  b.dbg = nullptr;
  {
    // SQUINT_GEMM_DBG=k: only launch k records; SQUINT_GEMM_DBG=all: every launch gets its own
    // 64-tile slot (launch i at slot i % 256), for whole-update kernel-span timelines.
    static const char* dbg_env = getenv("SQUINT_GEMM_DBG");
    static int launch_no = 0;
    if (dbg_env) {
      const int me = launch_no++;
      const bool all = dbg_env[0] == 'a';
      if (!g_dbg_dev) {
        cudaMalloc(&g_dbg_dev, 256 * 64 * 8 * sizeof(unsigned long long));
        cudaMemset(g_dbg_dev, 0, 256 * 64 * 8 * sizeof(unsigned long long));
      }
      if (all) {
        b.dbg = g_dbg_dev + (size_t)(me % 256) * 64 * 8;
        g_dbg_tiles = 256 * 64;
      } else if (me == atoi(dbg_env)) {
        g_dbg_tiles = b.ntiles < 4096 ? b.ntiles : 4096;
        b.dbg = g_dbg_dev;
      }
    }
  }
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(b.ntiles);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  static const bool no_pdl = getenv("SQUINT_NO_PDL") != nullptr;
  if (g_pdl && !no_pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (b.cs > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = b.cs;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  {
    static const char* names[9] = {"k_gemm<ln_relu>", "k_gemm<ln_tanh>", "k_gemm<bias>", "k_gemm<tg_fwd>",
                                   "k_gemm<bwd_ln_relu>", "k_gemm<bwd_ln_tanh>", "k_gemm<relu_mask>",
                                   "k_gemm<tg_bwd>", "k_gemm<dw>"};
    double flops = 0;
    for (int i = 0; i < b.nprob; ++i)
      for (int k = 0; k < b.p[i].nseg; ++k) flops += 2.0 * b.p[i].M * (double)(b.p[i].N - b.p[i].acc_col0) * b.p[i].seg[k].k;
    note_launch(s, names[epi], flops, 0);
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, b);
  static const bool dbg = getenv("SQUINT_DEBUG_SYNC") != nullptr;
  if (dbg) {
    cudaError_t se = cudaStreamSynchronize(s);
    fprintf(stderr, "[squint] k_gemm nprob=%d tiles=%d stages=%d stage_bytes=%d -> %s\n", b.nprob, b.ntiles, S,
            b.stage_bytes, cudaGetErrorString(se));
    for (int i = 0; i < b.nprob; ++i) {
      const GProb& p = b.p[i];
      fprintf(stderr, "   p%d epi=%d M=%d N=%d bn=%d nseg=%d", i, p.epi, p.M, p.N, p.bn, p.nseg);
      for (int k = 0; k < p.nseg; ++k)
        fprintf(stderr, " [a_mn=%d b_mn=%d nkb=%d]", p.seg[k].a_mn, p.seg[k].b_mn, p.seg[k].nkb);
      fprintf(stderr, "\n");
    }
    if (se != cudaSuccess) return (int)se;
  }
  return (int)e;
}

}  // namespace sq
