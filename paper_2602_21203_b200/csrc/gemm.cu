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
constexpr int kDbgSlots = 16;  // globaltimer stamps per CTA (SQUINT_GEMM_DBG); slot 15 = EPI (+64 split-K) | grid << 8
constexpr int kABytes = 16384;  // 128 x 64 bf16
constexpr float kLog2Pi = 1.8378770664093453f;
constexpr float kSquashEps = 1e-6f;
constexpr int kColaccOff = 4 * 4 * 4096;                  // after the 4 warp pairs' box rings
constexpr int kEpiBytes = kColaccOff + 4 * 3 * 512 * 4;    // + LN-bwd column partials [4][3][512]
constexpr int kStaticSmem = 17 * 1024;  // static __shared__ of k_gemm (~14.6 KB) / k_gemm_ln16 (~16.6 KB), inside the 227 KB per CTA

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
  __shared__ uint64_t full_bar[kMaxStages], empty_bar[kMaxStages], done_bar, ld_bar[8], stats_bar;
  __shared__ uint32_t tmem_slot;
  __shared__ float red[2][2][128];
  // per-row (sum, sum of squares) of each cluster CTA, pushed by the CTAs (8-CTA clusters only for the
  // LayerNorm backward; 4 rows of partials keep the forward LayerNorm CTA small enough for two per SM)
  __shared__ float2 cl_red[(EPI == GE_BWD_LN_RELU || EPI == GE_BWD_LN_TANH) ? 8 : 4][128];
  __shared__ __align__(16) float s_bias[512], s_g[512], s_beta[512];  // per-column epilogue params
  // (the problem descriptor is read from the parameter block: a shared-memory copy of it, once
  // needed by a producer loop that re-read it per iteration, measured 2 % slower at c2 since the
  // loop invariants are hoisted)

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
  // weight gradient with a plain bias: column sums of D from an N = 16 MMA against ones
  const bool ones = EPI == GE_DW && P.bias_ones && n0 == 0;
  const uint32_t ones_col = ncols;
  if (ones) ncols *= 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = b.nstages;
  uint8_t* ones_tile = smem + (S * b.stage_bytes > kEpiBytes ? S * b.stage_bytes : kEpiBytes);  // 16 x 64 bf16
  auto stamp = [&](int k) {
    if (b.dbg && tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      b.dbg[blockIdx.x * kDbgSlots + k] = t;
    }
  };
  auto stamp_any = [&](int k) {  // recorded by the calling thread
    if (b.dbg) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      b.dbg[blockIdx.x * kDbgSlots + k] = t;
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
    tc::mbar_init(&stats_bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 2 && lane < P.nseg) {
    tc::tma_prefetch_desc(&b.maps[P.seg[lane].amap]);
    tc::tma_prefetch_desc(&b.maps[P.seg[lane].bmap]);
  }
  if (warp == 2 && lane >= 8 && lane < 11) {  // epilogue maps: a descriptor fetch on first use stalls the TMA queue
    const int m = lane == 8 ? P.omap : (lane == 9 ? P.xmap : P.ymap);
    if (m >= 0) tc::tma_prefetch_desc(&b.maps[m]);
  }
  if (ones && warp == 3) {
    // all elements 1.0 (so the swizzle is irrelevant); visible to the tensor core (async proxy)
    for (int i = lane; i < 2048 / 16; i += 32)
      reinterpret_cast<uint4*>(ones_tile)[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    tc::fence_async_smem();
  }
  tc::fence_before_sync();
  if (b.cs > 1) tc::cluster_sync_init();  // peers' stats_bar initialised before any st.async reaches it
  else __syncthreads();
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
  if (warp == 0) npre = __shfl_sync(0xffffffffu, npre, 0);  // the producer loop runs warp-wide
  // The producer (warp 0) waits for the preceding kernel right before its first load, with its
  // loop invariants computed; everything else below (x_hat / 1/sigma prefetches, epilogue
  // parameters) is issued by the other warps, off the path to the first operand load.
  if (warp != 0) {
    tc::pdl_wait();
    tc::pdl_trigger();
  }
  stamp(2);
  // LayerNorm backward: the pair's x_hat boxes (TMA, by warps 4-7) and the row's 1/sigma, fetched
  // while the main loop runs (b.xpre_off: their shared-memory home past the operand ring)
  float rs_pre = 0.f;
  const int q0 = warp & 3, r0 = m0 + q0 * 32 + lane;
  if constexpr (EPI == GE_BWD_LN_RELU || EPI == GE_BWD_LN_TANH) {
    if (warp >= 2 && r0 < P.M) rs_pre = P.rstd[r0];  // warps 0 / 1: after their role loops
    if (b.xpre_off && warp >= 4 && lane == 0) {
      const int ng = (nreal + 63) / 64;
      uint8_t* xs = smem + b.xpre_off + q0 * 4 * kSlotBytes;
      tc::mbar_expect_tx(&ld_bar[q0], ng * kSlotBytes);
      for (int g = 0; g < ng; ++g) tc::tma_load_2d(xs + g * kSlotBytes, &b.maps[P.xmap], n0 + g * 64, m0 + q0 * 32, &ld_bar[q0]);
      stamp(10);
    }
  }
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

  // Producer and MMA issuer: single threads running tight loops.  Everything loop-invariant
  // (tensor-map addresses, tile coordinates, byte counts) is hoisted per segment and the stage
  // index advances without divisions: the TMA and MMA instructions take uniform-register operands,
  // and per-iteration operand conversions had made issuing ~3x slower than the TMA unit.
  const bool wide = EPI == GE_DW && b.wide > 1;
  if (wide && warp == 0) {
    // ---------------- wide producer (weight gradients: both operands MN-major) ----------------
    // one TMA box covers KW = b.wide K blocks (64 MN x 64 KW K rows): 4x fewer, larger boxes;
    // stage = [A rows 0-63 | A rows 64-127 | B column groups], each KW x 8 KB
    const int KW = b.wide, sbytes = b.stage_bytes;
    const GSeg G = P.seg[0];
    const TileGeo geo = tile_geo(P, nreal, 1);
    const void* am = &b.maps[G.amap];
    const void* bm = &b.maps[G.bmap];
    const int am0 = P.a_m + m0, bn0 = P.b_n + n0, nsb = (G.nkb + KW - 1) / KW;
    const uint32_t tx = (uint32_t)((2 + geo.nbox_b) * KW * 8192);
    int st = 0, ph = 0;
    tc::pdl_wait();
    tc::pdl_trigger();
    for (int sb = 0; sb < nsb; ++sb) {
      if (sb >= S) tc::mbar_wait(&empty_bar[st], ph ^ 1);
      uint8_t* As = smem + st * sbytes;
      const int kc = G.a_k + 64 * KW * sb, kcb = G.b_k + 64 * KW * sb;
      tc::mbar_expect_tx_e(&full_bar[st], tx);
      tc::tma_load_2d_e(As, am, am0, kc, &full_bar[st]);
      tc::tma_load_2d_e(As + KW * 8192, am, am0 + 64, kc, &full_bar[st]);
      for (int i = 0; i < geo.nbox_b; ++i)
        tc::tma_load_2d_e(As + (2 + i) * KW * 8192, bm, bn0 + 64 * i, kcb, &full_bar[st]);
      if (++st == S) st = 0, ph ^= 1;
    }
    if (lane == 0) stamp_any(11);
  } else if (wide && warp == 1) {
    // ---------------- wide MMA issuer ----------------
    const int KW = b.wide;
    const GSeg G = P.seg[0];
    const uint32_t id1 = tc::idesc_bf16_major(128, n1, 1, 1), id_ones = tc::idesc_bf16_major(128, 16, 1, 0);
    const uint32_t smem0 = tc::smem_u32(smem), sbytes = (uint32_t)b.stage_bytes, lbo = (uint32_t)KW * 8192u;
    const uint32_t ones0 = tc::smem_u32(ones_tile);
    const int nsb = (G.nkb + KW - 1) / KW;
    int st = 0, ph = 0, kb = 0;
    for (int sb = 0; sb < nsb; ++sb) {
      tc::mbar_wait(&full_bar[st], ph);
      if (lane == 0 && sb == 0) stamp_any(8);
      if (lane == 0) stamp_any(9);
      tc::fence_after_sync();
      const uint32_t a0 = smem0 + st * sbytes, b0 = a0 + 2 * lbo;
      for (int j = 0; j < KW && kb < G.nkb; ++j, ++kb) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = tc::sdesc_sw128(a0 + j * 8192 + 2048 * k, lbo, 1024);
          const uint32_t acc = (kb | k) != 0;
          tc::mma_bf16_e(tmem, ad, tc::sdesc_sw128(b0 + j * 8192 + 2048 * k, lbo, 1024), id1, acc);
          if (ones) tc::mma_bf16_e(tmem + ones_col, ad, tc::sdesc_sw128(ones0 + 32 * k, 16, 1024), id_ones, acc);
        }
      }
      tc::mma_commit_e(&empty_bar[st]);
      if (++st == S) st = 0, ph ^= 1;
    }
    tc::mma_commit_e(&done_bar);
  } else if (warp == 0) {
    // ---------------- TMA producer (whole warp, one elected lane issues) ----------------
    const int sbytes = b.stage_bytes, rank = b.mcast ? (int)(blockIdx.x % b.cs) : 0, cs = b.cs;
    const uint16_t mask = (uint16_t)((1u << cs) - 1u);
    int kb = 0, st = 0, ph = 0;
    for (int s = 0; s < P.nseg; ++s) {
      const GSeg G = P.seg[s];
      const TileGeo geo = tile_geo(P, nreal, G.b_mn);
      const void* am = &b.maps[G.amap];
      const void* bm = &b.maps[G.bmap];
      const int am0 = P.a_m + m0, bn0 = P.b_n + n0;
      const uint32_t tx = kABytes + geo.bbytes;
      if (s == 0) {
        tc::pdl_wait();
        tc::pdl_trigger();
      }
      for (int l = 0; l < G.nkb; ++l, ++kb) {
        if (kb >= S) tc::mbar_wait(&empty_bar[st], ph ^ 1);
        uint8_t* As = smem + st * sbytes;
        uint8_t* Bs = As + kABytes;
        const bool pre = kb < npre;  // B already in flight, transaction bytes already expected
        const int kc = G.a_k + 64 * l, kcb = G.b_k + 64 * l;
        if (!pre) tc::mbar_expect_tx_e(&full_bar[st], tx);
        if (b.mcast) {
          // the cluster's CTAs share the A tile: K block kb is fetched once, by rank kb % cs, for all
          if ((kb & (cs - 1)) == rank) {
            if (!G.a_mn) {
              tc::tma_load_2d_mc_e(As, am, kc, am0, &full_bar[st], mask);
            } else {
              tc::tma_load_2d_mc_e(As, am, am0, kc, &full_bar[st], mask);
              tc::tma_load_2d_mc_e(As + 8192, am, am0 + 64, kc, &full_bar[st], mask);
            }
          }
        } else if (!G.a_mn) {
          tc::tma_load_2d_e(As, am, kc, am0, &full_bar[st]);
        } else {
          tc::tma_load_2d_e(As, am, am0, kc, &full_bar[st]);
          tc::tma_load_2d_e(As + 8192, am, am0 + 64, kc, &full_bar[st]);
        }
        if (!pre) {
          if (!G.b_mn)
            for (int i = 0; i < geo.nbox_b; ++i)
              tc::tma_load_2d_e(Bs + i * geo.bnb * 128, bm, kcb, bn0 + geo.bnb * i, &full_bar[st]);
          else
            for (int i = 0; i < geo.nbox_b; ++i) tc::tma_load_2d_e(Bs + i * 8192, bm, bn0 + 64 * i, kcb, &full_bar[st]);
        }
        if (++st == S) st = 0, ph ^= 1;
      }
    }
    if (lane == 0) stamp_any(11);
  } else if (warp == 1) {
    // ---------------- MMA issuer (whole warp, one elected lane issues) ----------------
    const uint32_t smem0 = tc::smem_u32(smem), sbytes = (uint32_t)b.stage_bytes;
    const uint32_t ones0 = tc::smem_u32(ones_tile);
    int kb = 0, st = 0, ph = 0;
    for (int s = 0; s < P.nseg; ++s) {
      const GSeg& G = P.seg[s];
      const uint32_t id1 = tc::idesc_bf16_major(128, n1, G.a_mn, G.b_mn);
      const uint32_t id2 = tc::idesc_bf16_major(128, n2 > 0 ? n2 : 16, G.a_mn, G.b_mn);
      const uint32_t id_ones = tc::idesc_bf16_major(128, 16, G.a_mn, 0);
      // K-advance per 16-wide step: 2 KB through an MN-major operand's rows, 32 B inside a K-major row
      const uint32_t astep = G.a_mn ? 2048u : 32u, bstep = G.b_mn ? 2048u : 32u;
      const uint32_t albo = G.a_mn ? 8192u : 16u, blbo = G.b_mn ? 8192u : 16u;
      for (int l = 0; l < G.nkb; ++l, ++kb) {
        tc::mbar_wait(&full_bar[st], ph);
        if (lane == 0 && kb == 0) stamp_any(8);
        if (lane == 0) stamp_any(9);
        tc::fence_after_sync();
        const uint32_t a0 = smem0 + st * sbytes, b0 = a0 + kABytes;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t ad = tc::sdesc_sw128(a0 + astep * k, albo, 1024);
          const uint32_t acc = (kb | k) != 0;
          tc::mma_bf16_e(tmem, ad, tc::sdesc_sw128(b0 + bstep * k, blbo, 1024), id1, acc);
          if (n2 > 0) tc::mma_bf16_e(tmem + 256, ad, tc::sdesc_sw128(b0 + 32768 + bstep * k, blbo, 1024), id2, acc);
          if (ones) tc::mma_bf16_e(tmem + ones_col, ad, tc::sdesc_sw128(ones0 + 32 * k, 16, 1024), id_ones, acc);
        }
        tc::mma_commit_e(&empty_bar[st]);
        if (++st == S) st = 0, ph ^= 1;
      }
    }
    tc::mma_commit_e(&done_bar);
  }
  __syncwarp();
  if constexpr (EPI == GE_BWD_LN_RELU || EPI == GE_BWD_LN_TANH)
    if (warp < 2 && r0 < P.M) rs_pre = P.rstd[r0];
  // one poller: 256 threads spinning in try_wait compete with the TMA's complete_tx traffic on
  // the shared-memory barrier unit; the rest wait in bar.sync
  if (tid == 0) tc::mbar_wait(&done_bar, 0);
  __syncthreads();  // MMAs done; s_bias / s_g / s_beta visible
  tc::fence_after_sync();
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
  // (st.async into every cluster CTA's cl_red[rank], completion counted on its stats_bar; the
  // receiver sums the cs entries in rank order: every CTA gets the same bits, no cluster barrier)
  // (split in two so that independent work can run while the partials travel: row_push, then
  // row_pull for the totals)
  auto row_push = [&](float p1, float p2, float& t1, float& t2) {
    if (b.cs > 1 && tid == 0) tc::mbar_expect_tx(&stats_bar, b.cs * 128 * 8);
    red[0][hh][rl] = p1;
    red[1][hh][rl] = p2;
    __syncthreads();
    stamp(14);
    t1 = red[0][0][rl] + red[0][1][rl];
    t2 = red[1][0][rl] + red[1][1][rl];
    if (b.cs > 1) {
      const uint32_t me = (uint32_t)(blockIdx.x % b.cs);
      if (hh == 0)
        for (int rk = 0; rk < b.cs; ++rk)
          tc::st_async_v2(tc::mapa(&cl_red[me][rl], (uint32_t)rk), t1, t2, tc::mapa(&stats_bar, (uint32_t)rk));
    }
  };
  auto row_pull = [&](float& t1, float& t2) {
    if (b.cs > 1) {
      tc::mbar_wait(&stats_bar, 0);
      t1 = t2 = 0.f;
      for (int rk = 0; rk < b.cs; ++rk) {
        t1 += cl_red[rk][rl].x;
        t2 += cl_red[rk][rl].y;
      }
    }
  };
  auto row_total2 = [&](float p1, float p2, float& t1, float& t2) {
    row_push(p1, p2, t1, t2);
    row_pull(t1, t2);
  };

  if constexpr (EPI == GE_BIAS_F32 || EPI == GE_DW) {
    // fp32 rows through a per-warp 32 x 33 transpose tile: each store instruction writes 32
    // consecutive floats of one row (coalesced for any row pitch)
    float* T = reinterpret_cast<float*>(smem) + warp * 32 * 33;
    const int nvr = min(32, P.M - row0);
    for (int ch = hh; ch < nch; ch += 2) {
      const int c0 = n0 + ch * 32, ncv = min(32, n0 + nreal - c0);
      tc::tmem_ld32(trow + ch * 32, v);
      if constexpr (EPI == GE_BIAS_F32) {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] += s_bias[ch * 32 + j];
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; ++j) T[lane * 33 + j] = v[j];
      __syncwarp();
      if (lane < ncv)
        for (int i = 0; i < nvr; ++i) P.outf[(int64_t)(row0 + i) * P.ldf + c0 + lane] = T[i * 33 + lane];
    }
    if constexpr (EPI == GE_DW) {
      if (n0 == 0 && hh == 0) {
        float db = 0.f, dg = 0.f, dbe = 0.f;
        if (ones) {
          float o[16];
          tc::tmem_ld16(trow + ones_col, o);
          db = o[0];
        }
        if (rv) {
          if (P.part_in) {
            for (int t = 0; t < P.part_tiles; ++t) {
              const float* pp = P.part_in + (int64_t)t * 3 * P.M;
              db += pp[r];
              dg += pp[P.M + r];
              dbe += pp[2 * P.M + r];
            }
          }
          if (P.db) P.db[r] = db;
          if (P.dg) P.dg[r] = dg;
          if (P.dbeta) P.dbeta[r] = dbe;
        }
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
        uint32_t yp[16], xp[16];
        ln_fwd32<EPI == GE_LN_RELU>(v, s_bias + ch * 32, s_g + ch * 32, s_beta + ch * 32, mean, rs, yp, xp);
        // TMA stores are masked at 16-byte granularity: an output block whose last column is
        // not 8-aligned (the projection's z inside [z | s | a]) is stored directly instead.
        if (tma_out) {
          box_put_pk(sy, hh, yp);
        } else if (rv) {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[2 * j] = bf2_lo(yp[j]), v[2 * j + 1] = bf2_hi(yp[j]);
          row_st_bf16(P.out + (int64_t)r * P.ldo + n0 + ch * 32, min(32, nreal - ch * 32), v);
        }
        if (P.xh) box_put_pk(sx, hh, xp);
      }
      if (tma_out) pair_store(sy, &b.maps[P.omap], n0 + g * 64, row0, q, hh);
      if (P.xh) pair_store(sx, &b.maps[P.xmap], n0 + g * 64, row0, q, hh);
    }
  } else if constexpr (EPI == GE_BWD_LN_RELU || EPI == GE_BWD_LN_TANH) {
    float* colacc = reinterpret_cast<float*>(smem + kColaccOff);  // [4][3][512]
    if (P.bn == 32) {
      // 8-CTA clusters (32 columns per CTA): warp (q, hh) takes columns 16 hh .. 16 hh + 15 of the
      // slice, so each thread handles 16 values; outputs go straight to global memory (a 64-column
      // TMA box would overlap the neighbour CTA's columns)
      uint8_t* xs = b.xpre_off ? smem + b.xpre_off + q * 4 * kSlotBytes : pslots;
      if (!b.xpre_off && hh == 0 && lane == 0) {
        tc::mbar_expect_tx(&ld_bar[q], kSlotBytes);
        tc::tma_load_2d(xs, &b.maps[P.xmap], n0, row0, &ld_bar[q]);
      }
      tc::mbar_wait(&ld_bar[q], 0);
      stamp(5);
      const int c0 = hh * 16;
      float dn[16], xh[16], pg[16], pb[16];
      tc::tmem_ld16(trow + c0, dn);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const uint4 u = *reinterpret_cast<const uint4*>(xs + gd::box_off(lane, 2 * hh + j));
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(h2[k]);
          xh[8 * j + 2 * k] = f.x, xh[8 * j + 2 * k + 1] = f.y;
        }
      }
      float s1 = 0.f, s2 = 0.f;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int cc = c0 + j;
        const bool ok = rv && (cc < nreal);
        const float x = ok ? xh[j] : 0.f;
        const float n = fmaf(x, s_g[cc], s_beta[cc]);
        const float d = ok ? ((EPI == GE_BWD_LN_RELU) ? (n > 0.f ? dn[j] : 0.f) : dn[j] * sech2_fast(n)) : 0.f;
        const float dxh = d * s_g[cc];
        s1 += dxh;
        s2 += dxh * x;
        pg[j] = d * x;
        pb[j] = d;
        dn[j] = d;
        xh[j] = x;
      }
      float m1, m2;
      row_push(s1, s2, m1, m2);
      // the column partials while the row partials travel through the cluster
      const float cg = gd::colsum16(pg), cb = gd::colsum16(pb);
      if (lane < 16) {
        colacc[(q * 3 + 1) * 512 + c0 + lane] = cg;
        colacc[(q * 3 + 2) * 512 + c0 + lane] = cb;
      }
      row_pull(m1, m2);
      stamp(6);
      m1 /= (float)N;
      m2 /= (float)N;
      const float rs = rv ? rs_pre : 0.f;
      float o[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const bool ok = rv && (c0 + j < nreal);
        o[j] = ok ? rs * (dn[j] * s_g[c0 + j] - m1 - xh[j] * m2) : 0.f;
        pg[j] = o[j];
      }
      if (rv && c0 < nreal) {
        bf16* dst = P.out + (int64_t)r * P.ldo + n0 + c0;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          float f[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) f[k] = o[8 * j + k];
          reinterpret_cast<uint4*>(dst)[j] = tc::pack_bf16x8(f);
        }
      }
      const float cx = gd::colsum16(pg);
      if (lane < 16) colacc[(q * 3 + 0) * 512 + c0 + lane] = cx;
      __syncthreads();
      if (P.part) {
        for (int e = tid; e < 3 * nreal; e += kThreads) {
          const int kk = e / nreal, c = e - kk * nreal;
          float sacc = 0.f;
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) sacc += colacc[(qq * 3 + kk) * 512 + c];
          P.part[((int64_t)mt * 3 + kk) * N + n0 + c] = sacc;
        }
      }
    } else {
    // the pair's x_hat boxes (<= 4) by TMA on one transaction barrier (prefetched when possible)
    uint8_t* xs = b.xpre_off ? smem + b.xpre_off + q * 4 * kSlotBytes : pslots;
    if (!b.xpre_off && hh == 0 && lane == 0) {
      tc::mbar_expect_tx(&ld_bar[q], ngrp * kSlotBytes);
      for (int g = 0; g < ngrp; ++g)
        tc::tma_load_2d(xs + g * kSlotBytes, &b.maps[P.xmap], n0 + g * 64, row0, &ld_bar[q]);
    }
    tc::mbar_wait(&ld_bar[q], 0);
    stamp(5);
    // pass 1: dn = dL/d(g x_hat + beta) through the activation, the row sums of dxh = dn g and
    // dxh x_hat, column partials of dn x_hat and dn.  With one 64-column group the warp keeps
    // (dn, x_hat) in v / a for pass 2.
    float s1 = 0.f, s2 = 0.f;
    for (int g = 0; g < ngrp; ++g) {
      const int ch = 2 * g + hh;
      if (ch < nch) {
        const int c0 = ch * 32, ncv = min(32, nreal - c0);
        tc::tmem_ld32(trow + ch * 32, v);
        box_get(xs + g * kSlotBytes, hh, a);
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
          v[j] = dn;
          a[j] = x;
        }
        const float cg = colsum32(pg);
        const float cb = colsum32(pb);
        colacc[(q * 3 + 1) * 512 + c0 + lane] = cg;
        colacc[(q * 3 + 2) * 512 + c0 + lane] = cb;
      }
    }
    float m1, m2;
    stamp(13);
    row_total2(s1, s2, m1, m2);
    stamp(6);
    m1 /= (float)N;
    m2 /= (float)N;
    const float rs = rv ? rs_pre : 0.f;
    for (int g = 0; g < ngrp; ++g) {
      uint8_t* sl = xs + g * kSlotBytes;
      const int ch = 2 * g + hh;
      if (ch < nch) {
        const int c0 = ch * 32, ncv = min(32, nreal - c0);
        if (ngrp > 1) {  // recompute (dn, x_hat) of this group
          tc::tmem_ld32(trow + ch * 32, v);
          box_get(sl, hh, a);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int cc = c0 + j;
            const bool ok = rv && (j < ncv);
            const float x = ok ? a[j] : 0.f;
            const float n = fmaf(x, s_g[cc], s_beta[cc]);
            v[j] = ok ? ((EPI == GE_BWD_LN_RELU) ? (n > 0.f ? v[j] : 0.f) : v[j] * sech2_fast(n)) : 0.f;
            a[j] = x;
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const bool ok = rv && (j < ncv);
          v[j] = ok ? rs * (v[j] * s_g[c0 + j] - m1 - a[j] * m2) : 0.f;
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
    }  // bn == 64
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
  if (b.dbg && tid == 0) b.dbg[blockIdx.x * kDbgSlots + 15] = (unsigned long long)EPI | ((unsigned long long)gridDim.x << 8);
  if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}

// ---------------------------------------------------------------------------------------------
// LayerNorm backward over wide whole tiles (c3: 128 x 256 tiles of 512-wide rows in 2-CTA
// clusters): the same producer / MMA roles as k_gemm, and an epilogue run by 16 warps instead of
// 8.  The k_gemm epilogue of such a tile was issue- and latency-bound at two warps per SM
// sub-partition (~6.5 us per pass over the tile, ncu: 6.9-8.7 cycles per issued instruction);
// here warp w takes TMEM lane quarter w % 4 and column quarter w / 4, in 8-column steps (TMEM
// loads one step ahead) with 8-value shuffle column sums, so each thread holds ~40 live values.
// Host contract (gemm_launch): ks == 1, every problem's slice bn a multiple of 64 and <= 256,
// N % bn == 0, M % 128 == 0 (no ragged rows or columns).
constexpr int kBlnThreads = 512;

// column sums of 8 values per lane over the warp's 32 rows: lane l returns column l % 8 (fixed
// butterfly order: bitwise reproducible)
__device__ __forceinline__ float colsum8(float (&v)[8]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 4; s >= 1; s >>= 1) {
    const bool up = (lane & s) != 0;
#pragma unroll
    for (int j = 0; j < s; ++j) {
      const float send = up ? v[j] : v[j + s];
      const float keep = up ? v[j + s] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  float t = v[0] + __shfl_xor_sync(0xffffffffu, v[0], 8);
  return t + __shfl_xor_sync(0xffffffffu, t, 16);
}

template <int EPI>
__global__ void __launch_bounds__(kBlnThreads, 1) k_gemm_ln16(const __grid_constant__ GBatch b) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full_bar[kMaxStages], empty_bar[kMaxStages], done_bar, ld_bar[8], stats_bar;
  __shared__ uint32_t tmem_slot;
  __shared__ float red[2][4][128];
  __shared__ float2 cl_red[8][128];
  __shared__ __align__(16) float s_g[512], s_beta[512];
  constexpr bool BWD = EPI == GE_BWD_LN_RELU || EPI == GE_BWD_LN_TANH;
  static_assert(BWD, "k_gemm_ln16: LayerNorm backward only");

  const int tile = blockIdx.x;
  int pi = 0;
  while (pi + 1 < b.nprob && tile >= b.p[pi + 1].tile0) ++pi;
  const GProb& P = b.p[pi];
  const int lt = tile - P.tile0;
  const int mt = lt / P.tiles_n;
  const int m0 = mt * 128, n0 = (lt % P.tiles_n) * P.bn;
  const int nreal = P.bn;  // host contract: whole slices
  const uint32_t ncols = nreal <= 32 ? 32u : (nreal <= 64 ? 64u : (nreal <= 128 ? 128u : 256u));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = b.nstages;
  auto stamp = [&](int k) {
    if (b.dbg && tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      b.dbg[blockIdx.x * kDbgSlots + k] = t;
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
    tc::mbar_init(&stats_bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 2 && lane < P.nseg) {
    tc::tma_prefetch_desc(&b.maps[P.seg[lane].amap]);
    tc::tma_prefetch_desc(&b.maps[P.seg[lane].bmap]);
  }
  if (warp == 2 && lane >= 8 && lane < 10) tc::tma_prefetch_desc(&b.maps[lane == 8 ? P.omap : P.xmap]);
  tc::fence_before_sync();
  if (b.cs > 1) tc::cluster_sync_init();
  else __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_slot;
  stamp(1);
  int npre = 0;
  if (b.prefetch_b && warp == 0 && lane == 0) {
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
  if (warp == 0) npre = __shfl_sync(0xffffffffu, npre, 0);
  if (warp != 0) {  // the producer waits right before its first load (see k_gemm)
    tc::pdl_wait();
    tc::pdl_trigger();
  }
  stamp(2);
  // epilogue geometry: warp (q, hq): TMEM lanes / tile rows 32 q .., column quarter hq; the pair
  // p = hq / 2 owns the 64-column boxes g = p, p + 2 (half hh = hq % 2 of each)
  const int q = warp & 3, hq = warp >> 2, pp = hq >> 1, hh = hq & 1, rl = q * 32 + lane;
  const int row0 = m0 + q * 32, r = row0 + lane;
  const int ngrp = nreal / 64;
  float rs_pre = (BWD && warp >= 2) ? P.rstd[r] : 0.f;  // warps 0 / 1: after their role loops
  uint8_t* xs = (b.xpre_off ? smem + b.xpre_off : smem) + (q * 2 + pp) * 2 * kSlotBytes;  // the pair's <= 2 boxes
  if (BWD && b.xpre_off && hh == 1 && lane == 0) {  // (the pair's second warp: warp 0 is the producer)
    const int nb = (ngrp - pp + 1) / 2;
    if (nb > 0) {
      tc::mbar_expect_tx(&ld_bar[q * 2 + pp], nb * kSlotBytes);
      for (int j = 0; j < nb; ++j)
        tc::tma_load_2d(xs + j * kSlotBytes, &b.maps[P.xmap], n0 + (pp + 2 * j) * 64, row0, &ld_bar[q * 2 + pp]);
    }
  }
  if (warp >= 2)
    for (int c = tid - 64; c < nreal; c += kBlnThreads - 64) {
      s_g[c] = P.g[n0 + c];
      s_beta[c] = P.beta[n0 + c];
    }

  if (warp == 0) {
    // ---------------- TMA producer (as k_gemm) ----------------
    const int sbytes = b.stage_bytes, rank = b.mcast ? (int)(blockIdx.x % b.cs) : 0, cs = b.cs;
    const uint16_t mask = (uint16_t)((1u << cs) - 1u);
    int kb = 0, st = 0, ph = 0;
    for (int s = 0; s < P.nseg; ++s) {
      const GSeg G = P.seg[s];
      const TileGeo geo = tile_geo(P, nreal, G.b_mn);
      const void* am = &b.maps[G.amap];
      const void* bm = &b.maps[G.bmap];
      const int am0 = P.a_m + m0, bn0 = P.b_n + n0;
      const uint32_t tx = kABytes + geo.bbytes;
      if (s == 0) {
        tc::pdl_wait();
        tc::pdl_trigger();
      }
      for (int l = 0; l < G.nkb; ++l, ++kb) {
        if (kb >= S) tc::mbar_wait(&empty_bar[st], ph ^ 1);
        uint8_t* As = smem + st * sbytes;
        uint8_t* Bs = As + kABytes;
        const bool pre = kb < npre;
        const int kc = G.a_k + 64 * l, kcb = G.b_k + 64 * l;
        if (!pre) tc::mbar_expect_tx_e(&full_bar[st], tx);
        if (b.mcast) {
          if ((kb & (cs - 1)) == rank) {
            if (!G.a_mn) {
              tc::tma_load_2d_mc_e(As, am, kc, am0, &full_bar[st], mask);
            } else {
              tc::tma_load_2d_mc_e(As, am, am0, kc, &full_bar[st], mask);
              tc::tma_load_2d_mc_e(As + 8192, am, am0 + 64, kc, &full_bar[st], mask);
            }
          }
        } else if (!G.a_mn) {
          tc::tma_load_2d_e(As, am, kc, am0, &full_bar[st]);
        } else {
          tc::tma_load_2d_e(As, am, am0, kc, &full_bar[st]);
          tc::tma_load_2d_e(As + 8192, am, am0 + 64, kc, &full_bar[st]);
        }
        if (!pre) {
          if (!G.b_mn)
            for (int i = 0; i < geo.nbox_b; ++i)
              tc::tma_load_2d_e(Bs + i * geo.bnb * 128, bm, kcb, bn0 + geo.bnb * i, &full_bar[st]);
          else
            for (int i = 0; i < geo.nbox_b; ++i) tc::tma_load_2d_e(Bs + i * 8192, bm, bn0 + 64 * i, kcb, &full_bar[st]);
        }
        if (++st == S) st = 0, ph ^= 1;
      }
    }
    if (lane == 0) { if (b.dbg) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); b.dbg[blockIdx.x * kDbgSlots + 11] = t; } }
  } else if (warp == 1) {
    // ---------------- MMA issuer (as k_gemm; nreal <= 256: one MMA per K step) ----------------
    const uint32_t smem0 = tc::smem_u32(smem), sbytes = (uint32_t)b.stage_bytes;
    int kb = 0, st = 0, ph = 0;
    for (int s = 0; s < P.nseg; ++s) {
      const GSeg& G = P.seg[s];
      const uint32_t id1 = tc::idesc_bf16_major(128, nreal, G.a_mn, G.b_mn);
      const uint32_t astep = G.a_mn ? 2048u : 32u, bstep = G.b_mn ? 2048u : 32u;
      const uint32_t albo = G.a_mn ? 8192u : 16u, blbo = G.b_mn ? 8192u : 16u;
      for (int l = 0; l < G.nkb; ++l, ++kb) {
        tc::mbar_wait(&full_bar[st], ph);
        tc::fence_after_sync();
        const uint32_t a0 = smem0 + st * sbytes, b0 = a0 + kABytes;
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc::mma_bf16_e(tmem, tc::sdesc_sw128(a0 + astep * k, albo, 1024), tc::sdesc_sw128(b0 + bstep * k, blbo, 1024), id1,
                         (kb | k) != 0);
        tc::mma_commit_e(&empty_bar[st]);
        if (++st == S) st = 0, ph ^= 1;
      }
    }
    tc::mma_commit_e(&done_bar);
  }
  __syncwarp();
  if (BWD && warp < 2) rs_pre = P.rstd[r];
  if (tid == 0) tc::mbar_wait(&done_bar, 0);
  __syncthreads();
  tc::fence_after_sync();
  stamp(3);

  const uint32_t trow = tmem + ((uint32_t)(q * 32) << 16);
  // row totals: the four column quarters of this CTA (smem, in order), then the cluster CTAs
  auto row_total4 = [&](float& t1, float& t2) {
    if (b.cs > 1 && tid == 0) tc::mbar_expect_tx(&stats_bar, b.cs * 128 * 8);
    red[0][hq][rl] = t1;
    red[1][hq][rl] = t2;
    __syncthreads();
    t1 = (red[0][0][rl] + red[0][1][rl]) + (red[0][2][rl] + red[0][3][rl]);
    t2 = (red[1][0][rl] + red[1][1][rl]) + (red[1][2][rl] + red[1][3][rl]);
    if (b.cs > 1) {
      const uint32_t me = (uint32_t)(blockIdx.x % b.cs);
      if (hq == 0)
        for (int rk = 0; rk < b.cs; ++rk)
          tc::st_async_v2(tc::mapa(&cl_red[me][rl], (uint32_t)rk), t1, t2, tc::mapa(&stats_bar, (uint32_t)rk));
      tc::mbar_wait(&stats_bar, 0);
      t1 = t2 = 0.f;
      for (int rk = 0; rk < b.cs; ++rk) {
        t1 += cl_red[rk][rl].x;
        t2 += cl_red[rk][rl].y;
      }
    }
  };
  {
    // x_hat boxes (when not prefetched: now, into the pair's slots past the freed ring start)
    if (!b.xpre_off && hh == 0 && lane == 0) {
      const int nb = (ngrp - pp + 1) / 2;
      if (nb > 0) {
        tc::mbar_expect_tx(&ld_bar[q * 2 + pp], nb * kSlotBytes);
        for (int j = 0; j < nb; ++j)
          tc::tma_load_2d(xs + j * kSlotBytes, &b.maps[P.xmap], n0 + (pp + 2 * j) * 64, row0, &ld_bar[q * 2 + pp]);
      }
    }
    if (pp < ngrp) tc::mbar_wait(&ld_bar[q * 2 + pp], 0);
    stamp(5);
    float* colacc = reinterpret_cast<float*>(smem + kColaccOff);  // [4][3][512]
    // dn = dL/d(g x_hat + beta) through the activation
    auto dnf = [&](float v, float x, float gg, float be) {
      const float n = fmaf(x, gg, be);
      return (EPI == GE_BWD_LN_RELU) ? (n > 0.f ? v : 0.f) : v * sech2_fast(n);
    };
    float s1 = 0.f, s2 = 0.f;
    for (int g = pp; g < ngrp; g += 2) {
      const int c0 = g * 64 + hh * 32;
      const uint8_t* xb = xs + (g >> 1) * kSlotBytes;
      uint32_t cur[8], nxt[8];
      tc::tmem_ld8_async(trow + c0, cur);
      tc::tmem_wait8(cur);
  #pragma unroll 1
      for (int k = 0; k < 4; ++k) {
        if (k < 3) tc::tmem_ld8_async(trow + c0 + 8 * (k + 1), nxt);
        const uint4 u = *reinterpret_cast<const uint4*>(xb + gd::box_off(lane, 4 * hh + k));
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
        const float4 ga = *reinterpret_cast<const float4*>(&s_g[c0 + 8 * k]);
        const float4 gb = *reinterpret_cast<const float4*>(&s_g[c0 + 8 * k + 4]);
        const float4 ba = *reinterpret_cast<const float4*>(&s_beta[c0 + 8 * k]);
        const float4 bb = *reinterpret_cast<const float4*>(&s_beta[c0 + 8 * k + 4]);
        const float gv[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
        const float bv[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
        float pg[8], pb[8];
  #pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float2 f = __bfloat1622float2(h2[j >> 1]);
          const float x = (j & 1) ? f.y : f.x;
          const float dn = dnf(__uint_as_float(cur[j]), x, gv[j], bv[j]);
          const float dxh = dn * gv[j];
          s1 += dxh;
          s2 += dxh * x;
          pg[j] = dn * x;
          pb[j] = dn;
        }
        const float cg = colsum8(pg), cb = colsum8(pb);
        if (lane < 8) {
          colacc[(q * 3 + 1) * 512 + c0 + 8 * k + lane] = cg;
          colacc[(q * 3 + 2) * 512 + c0 + 8 * k + lane] = cb;
        }
        if (k < 3) {
          tc::tmem_wait8(nxt);
  #pragma unroll
          for (int j = 0; j < 8; ++j) cur[j] = nxt[j];
        }
      }
    }
    float m1 = s1, m2 = s2;
    row_total4(m1, m2);
    stamp(6);
    m1 /= (float)P.N;
    m2 /= (float)P.N;
    const float rs = rs_pre;
    for (int g = pp; g < ngrp; g += 2) {
      const int c0 = g * 64 + hh * 32;
      uint8_t* sl = xs + (g >> 1) * kSlotBytes;
      uint32_t cur[8], nxt[8];
      tc::tmem_ld8_async(trow + c0, cur);
      tc::tmem_wait8(cur);
  #pragma unroll 1
      for (int k = 0; k < 4; ++k) {
        if (k < 3) tc::tmem_ld8_async(trow + c0 + 8 * (k + 1), nxt);
        uint4* xp = reinterpret_cast<uint4*>(sl + gd::box_off(lane, 4 * hh + k));
        const uint4 u = *xp;
        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
        const float4 ga = *reinterpret_cast<const float4*>(&s_g[c0 + 8 * k]);
        const float4 gb = *reinterpret_cast<const float4*>(&s_g[c0 + 8 * k + 4]);
        const float4 ba = *reinterpret_cast<const float4*>(&s_beta[c0 + 8 * k]);
        const float4 bb = *reinterpret_cast<const float4*>(&s_beta[c0 + 8 * k + 4]);
        const float gv[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
        const float bv[8] = {ba.x, ba.y, ba.z, ba.w, bb.x, bb.y, bb.z, bb.w};
        float o[8];
  #pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float2 f = __bfloat1622float2(h2[j >> 1]);
          const float x = (j & 1) ? f.y : f.x;
          const float dn = dnf(__uint_as_float(cur[j]), x, gv[j], bv[j]);
          o[j] = rs * (dn * gv[j] - m1 - x * m2);
        }
        *xp = tc::pack_bf16x8(o);
        const float cx = colsum8(o);
        if (lane < 8) colacc[(q * 3 + 0) * 512 + c0 + 8 * k + lane] = cx;
        if (k < 3) {
          tc::tmem_wait8(nxt);
  #pragma unroll
          for (int j = 0; j < 8; ++j) cur[j] = nxt[j];
        }
      }
      // the pair's box g is complete: to the TMA unit (named barrier of the pair's 64 threads)
      tc::fence_async_smem();
      tc::named_bar(1 + q * 2 + pp, 64);
      if (hh == 0 && lane == 0) {
        tc::tma_store_2d(&b.maps[P.omap], sl, n0 + g * 64, row0);
        tc::bulk_commit();
      }
    }
    __syncthreads();
    if (P.part) {
      for (int e = tid; e < 3 * nreal; e += kBlnThreads) {
        const int kk = e / nreal, c = e - kk * nreal;
        float sacc = 0.f;
  #pragma unroll
        for (int qq = 0; qq < 4; ++qq) sacc += colacc[(qq * 3 + kk) * 512 + c];
        P.part[((int64_t)mt * 3 + kk) * P.N + n0 + c] = sacc;
      }
    }
  }
  stamp(7);
  if (lane == 0) tc::bulk_wait_read<0>();
  tc::fence_before_sync();
  __syncthreads();
  stamp(4);
  if (b.dbg && tid == 0) b.dbg[blockIdx.x * kDbgSlots + 15] = (unsigned long long)(EPI | 128) | ((unsigned long long)gridDim.x << 8);
  if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}

// ---------------------------------------------------------------------------------------------
// Split-K variant for narrow row-complete layers (N <= 64 with long K: the projection LayerNorm,
// its backward, the tanh-Gaussian head and its backward).  With one 128-row tile per CTA those
// launches ran on 4-16 SMs, serial over up to 13 K blocks, with a 32-element-per-thread
// epilogue.  Here a cluster of ks CTAs shares one tile: CTA kr accumulates K blocks
// [kr T / ks, (kr + 1) T / ks) in its own TMEM, every warp quarter pushes its 32 accumulator rows
// (fp32, 8 KB) by bulk copy into the shared memory of the CTA that owns those rows (rank
// q ks / 4; completion counted in bytes on the owner's mbarrier), and each CTA sums the ks
// partial tiles of its 128 / ks rows in rank order (deterministic) and runs the epilogue with
// 8 threads per row (8 columns each; row statistics by shuffles).  Column partials of the
// LayerNorm backward are written per 128 / ks-row block: part[(mtile ks + kr)][3][N].
constexpr int kSkRecvBytes = 32768;  // 128 rows x 64 fp32 columns, in ks slots of 128 / ks rows

__device__ __forceinline__ uint32_t sk_off(int row, int chunk) {  // 64-float rows, 16-byte chunks
  return (uint32_t)(row * 256 + ((chunk ^ (row & 7)) << 4));
}

template <int EPI>
__global__ void __launch_bounds__(kThreads, 1) k_gemm_sk(const __grid_constant__ GBatch b) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full_bar[kMaxStages], empty_bar[kMaxStages], done_bar, recv_bar;
  __shared__ uint32_t tmem_slot;
  __shared__ __align__(16) float s_bias[64], s_g[64], s_beta[64];
  __shared__ float s_col[8][3][64];

  const int ks = b.ks;
  const uint32_t kr = tc::cluster_rank();
  const int tile = blockIdx.x / ks;
  int pi = 0;
  while (pi + 1 < b.nprob && tile >= b.p[pi + 1].tile0) ++pi;
  const GProb& P = b.p[pi];
  const int mt = tile - P.tile0;
  const int m0 = mt * 128;
  const int nreal = P.N;
  const int nt = round16(nreal);
  const int R = 128 / ks;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = b.nstages;
  uint8_t* recv = smem + (b.nstages * b.stage_bytes > kSkRecvBytes ? b.nstages * b.stage_bytes : kSkRecvBytes);
  auto stamp = [&](int k) {
    if (b.dbg && tid == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      b.dbg[blockIdx.x * kDbgSlots + k] = t;
    }
  };
  stamp(0);
  int T = 0;
  for (int s = 0; s < P.nseg; ++s) T += P.seg[s].nkb;
  const int kb0 = (int)kr * T / ks, kb1 = ((int)kr + 1) * T / ks;

  if (warp == 0) tc::tmem_alloc(&tmem_slot, 64);
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < S; ++i) {
      tc::mbar_init(&full_bar[i], 1);
      tc::mbar_init(&empty_bar[i], 1);
    }
    tc::mbar_init(&done_bar, 1);
    tc::mbar_init(&recv_bar, 1);
    tc::fence_mbar_init();
  }
  if (warp == 2 && lane < P.nseg) {
    tc::tma_prefetch_desc(&b.maps[P.seg[lane].amap]);
    tc::tma_prefetch_desc(&b.maps[P.seg[lane].bmap]);
  }
  tc::fence_before_sync();
  tc::cluster_sync_init();  // every CTA's recv_bar is initialised before any peer copies into it
  tc::fence_after_sync();
  const uint32_t tmem = tmem_slot;
  stamp(1);
  // walk this CTA's K blocks: (segment, block within the segment) for global block kb
  auto seg_of = [&](int kb, int& l) {
    int s = 0;
    while (kb >= P.seg[s].nkb) kb -= P.seg[s++].nkb;
    l = kb;
    return s;
  };
  int npre = 0;
  if (b.prefetch_b && warp == 0 && lane == 0) {
    for (int kb = kb0; kb < kb1 && kb - kb0 < S; ++kb) {
      int l;
      const GSeg& G = P.seg[seg_of(kb, l)];
      const TileGeo geo = tile_geo(P, nreal, G.b_mn);
      uint8_t* Bs = smem + (kb - kb0) * b.stage_bytes + kABytes;
      tc::mbar_expect_tx(&full_bar[kb - kb0], kABytes + geo.bbytes);
      for (int i = 0; i < geo.nbox_b; ++i) {
        if (!G.b_mn)
          tc::tma_load_2d(Bs + i * geo.bnb * 128, &b.maps[G.bmap], G.b_k + 64 * l, P.b_n + geo.bnb * i, &full_bar[kb - kb0]);
        else
          tc::tma_load_2d(Bs + i * 8192, &b.maps[G.bmap], P.b_n + 64 * i, G.b_k + 64 * l, &full_bar[kb - kb0]);
      }
      ++npre;
    }
  }
  if (warp == 0) npre = __shfl_sync(0xffffffffu, npre, 0);  // the producer loop runs warp-wide
  if (warp != 0) {  // the producer waits right before its first load (see k_gemm)
    tc::pdl_wait();
    tc::pdl_trigger();
  }
  stamp(2);
  // per-row epilogue inputs, loaded while the main loop runs (warps 0 / 1: after their role
  // loops): thread (row tid / 8 + 32 it, column group tid % 8); R / 32 <= 2 rows per thread
  const int cg = tid & 7, c0 = cg * 8;
  const int nit = (R + 31) / 32;  // R = 16 (ks = 8): threads of rows tid / 8 >= R idle
  uint4 xpre[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
  float rspre[2] = {0.f, 0.f};
  float tg_pre[2][2][3];  // tanh-Gaussian: [it][d = cg, cg + 8][mu | l | eps]
  float dlp = 0.f;
  auto load_pre = [&]() {
  for (int it = 0; it < nit; ++it) {
    const int r = m0 + (int)kr * R + (tid >> 3) + 32 * it;
    if (r >= P.M || (tid >> 3) + 32 * it >= R) continue;
    if constexpr (EPI == GE_BWD_LN_TANH || EPI == GE_BWD_LN_RELU) {
      if (c0 < nreal) xpre[it] = *reinterpret_cast<const uint4*>(P.xh + (int64_t)r * P.ldx + c0);
      rspre[it] = P.rstd[r];
    } else if constexpr (EPI == GE_TG_FWD || EPI == GE_TG_BWD) {
      const int A = EPI == GE_TG_FWD ? P.N / 2 : P.N - P.acc_col0;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int d = cg + 8 * u;
        tg_pre[it][u][0] = tg_pre[it][u][1] = tg_pre[it][u][2] = 0.f;
        if (d < A) {
          if (EPI == GE_TG_BWD) {
            tg_pre[it][u][0] = P.tgo[(int64_t)r * 2 * A + d];
            tg_pre[it][u][1] = P.tgo[(int64_t)r * 2 * A + A + d];
          }
          if (P.eps) tg_pre[it][u][2] = P.eps[(int64_t)r * A + d];
        }
      }
    }
  }
  if constexpr (EPI == GE_TG_BWD) dlp = P.dlogp_scale[0];
  };
  if (warp >= 2) load_pre();
  if (warp >= 2) {
    for (int c = tid - 64; c < nt; c += kThreads - 64) {
      const bool ok = c < P.N;
      s_bias[c] = (ok && P.bias) ? P.bias[c] : 0.f;
      s_g[c] = (ok && P.g) ? P.g[c] : 0.f;
      s_beta[c] = (ok && P.beta) ? P.beta[c] : 0.f;
    }
  }
  if (warp == 0) {
    // producer: warp-uniform loop, one elected lane issues (see k_gemm)
    tc::mbar_expect_tx_e(&recv_bar, kSkRecvBytes);
    const int sbytes = b.stage_bytes;
    int st = 0, ph = 0;
    tc::pdl_wait();
    tc::pdl_trigger();
    for (int kb = kb0; kb < kb1; ++kb) {
      const int i = kb - kb0;
      int l;
      const GSeg& G = P.seg[seg_of(kb, l)];
      const TileGeo geo = tile_geo(P, nreal, G.b_mn);
      if (i >= S) tc::mbar_wait(&empty_bar[st], ph ^ 1);
      uint8_t* As = smem + st * sbytes;
      uint8_t* Bs = As + kABytes;
      const bool pre = i < npre;
      if (!pre) tc::mbar_expect_tx_e(&full_bar[st], kABytes + geo.bbytes);
      const int kc = 64 * l;
      if (!G.a_mn) {
        tc::tma_load_2d_e(As, &b.maps[G.amap], G.a_k + kc, P.a_m + m0, &full_bar[st]);
      } else {
        tc::tma_load_2d_e(As, &b.maps[G.amap], P.a_m + m0, G.a_k + kc, &full_bar[st]);
        tc::tma_load_2d_e(As + 8192, &b.maps[G.amap], P.a_m + m0 + 64, G.a_k + kc, &full_bar[st]);
      }
      if (!pre) {
        for (int j = 0; j < geo.nbox_b; ++j) {
          if (!G.b_mn)
            tc::tma_load_2d_e(Bs + j * geo.bnb * 128, &b.maps[G.bmap], G.b_k + kc, P.b_n + geo.bnb * j, &full_bar[st]);
          else
            tc::tma_load_2d_e(Bs + j * 8192, &b.maps[G.bmap], P.b_n + 64 * j, G.b_k + kc, &full_bar[st]);
        }
      }
      if (++st == S) st = 0, ph ^= 1;
    }
  } else if (warp == 1) {
    int st = 0, ph = 0;
    const uint32_t smem0 = tc::smem_u32(smem), sbytes = (uint32_t)b.stage_bytes;
    for (int kb = kb0; kb < kb1; ++kb) {
      const int i = kb - kb0;
      int l;
      const GSeg& G = P.seg[seg_of(kb, l)];
      const uint32_t id = tc::idesc_bf16_major(128, nt, G.a_mn, G.b_mn);
      const uint32_t astep = G.a_mn ? 2048u : 32u, bstep = G.b_mn ? 2048u : 32u;
      const uint32_t albo = G.a_mn ? 8192u : 16u, blbo = G.b_mn ? 8192u : 16u;
      tc::mbar_wait(&full_bar[st], ph);
      tc::fence_after_sync();
      const uint32_t a0 = smem0 + st * sbytes, b0 = a0 + kABytes;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        tc::mma_bf16_e(tmem, tc::sdesc_sw128(a0 + astep * k, albo, 1024), tc::sdesc_sw128(b0 + bstep * k, blbo, 1024), id,
                       (i | k) != 0);
      tc::mma_commit_e(&empty_bar[st]);
      if (++st == S) st = 0, ph ^= 1;
    }
    tc::mma_commit_e(&done_bar);
  }
  __syncwarp();
  if (warp < 2) load_pre();
  if (tid == 0) tc::mbar_wait(&done_bar, 0);
  __syncthreads();
  tc::fence_after_sync();
  stamp(3);

  // ---- push the partial tile: warp quarter q's rows go to the CTA owning them ----
  {
    const int q = warp & 3, hh = warp >> 2;
    uint8_t* stg = smem + q * 8192;  // operand ring is free once the MMAs completed
    if (hh * 32 < nt) {
      float v[32];
      tc::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + hh * 32, v);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<float4*>(stg + sk_off(lane, hh * 8 + j)) = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
    }
    tc::fence_async_smem();
    tc::named_bar(1 + q, 64);
    if (hh == 0 && lane == 0) {
      if (ks <= 4) {
        const uint32_t owner = (uint32_t)(q * ks / 4);
        const int rowoff = q * 32 - (int)owner * R;
        tc::bulk_s2cluster(tc::mapa(recv + ((int)kr * R + rowoff) * 256, owner), stg, 8192, tc::mapa(&recv_bar, owner));
      } else {  // ks = 8: the quarter's 32 rows belong to two owners of 16 rows each
        for (int h2 = 0; h2 < 2; ++h2) {
          const uint32_t owner = (uint32_t)(2 * q + h2);
          tc::bulk_s2cluster(tc::mapa(recv + ((int)kr * R) * 256, owner), stg + h2 * 4096, 4096,
                             tc::mapa(&recv_bar, owner));
        }
      }
    }
  }
  __syncthreads();  // s_bias / s_g / s_beta visible
  tc::mbar_wait(&recv_bar, 0);
  stamp(5);

  // every copy into this CTA has landed; arriving now (waiting only at exit) tells the peers
  // their outgoing copies are complete without a barrier on the critical path
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  // ---- epilogue over this CTA's rows [kr R, kr R + R) of the tile ----
  const int N = P.N;
  auto recv_sum8 = [&](int rr, float (&acc)[8]) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    for (int k = 0; k < ks; ++k) {
      const uint8_t* base = recv + (k * R) * 256;
      const float4 lo = *reinterpret_cast<const float4*>(base + sk_off(rr, 2 * cg));
      const float4 hi = *reinterpret_cast<const float4*>(base + sk_off(rr, 2 * cg + 1));
      acc[0] += lo.x, acc[1] += lo.y, acc[2] += lo.z, acc[3] += lo.w;
      acc[4] += hi.x, acc[5] += hi.y, acc[6] += hi.z, acc[7] += hi.w;
    }
  };
  auto recv_col = [&](int rr, int c) {
    float v = 0.f;
    for (int k = 0; k < ks; ++k)
      v += *reinterpret_cast<const float*>(recv + (k * R) * 256 + sk_off(rr, c >> 2) + (c & 3) * 4);
    return v;
  };
  if constexpr (EPI == GE_LN_TANH || EPI == GE_LN_RELU || EPI == GE_BWD_LN_TANH || EPI == GE_BWD_LN_RELU) {
    float cp[3][8];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
      for (int j = 0; j < 8; ++j) cp[k][j] = 0.f;
    for (int it = 0; it < nit; ++it) {
      const int rr = (tid >> 3) + 32 * it;
      float acc[8];
      recv_sum8(rr < R ? rr : R - 1, acc);
      if (it == 0) stamp(8);
      const int r = m0 + (int)kr * R + rr;
      const bool rv = r < P.M && rr < R;
      if constexpr (EPI == GE_LN_TANH || EPI == GE_LN_RELU) {
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          acc[j] += s_bias[c0 + j];
          if (c0 + j < nreal) s1 += acc[j], s2 += acc[j] * acc[j];
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
          s1 += __shfl_xor_sync(0xffffffffu, s1, o);
          s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        }
        const float mean = s1 / (float)N;
        const float rs = rsqrtf(fmaxf(s2 / (float)N - mean * mean, 0.f) + P.ln_eps);
        float y[8], xh[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          xh[j] = bf16_round((acc[j] - mean) * rs);
          const float n = fmaf(xh[j], s_g[c0 + j], s_beta[c0 + j]);
          y[j] = (EPI == GE_LN_RELU) ? fmaxf(n, 0.f) : tanh_fast(n);
        }
        if (rv && c0 < nreal) {
          const int ncv = min(8, nreal - c0);
          bf16* o = P.out + (int64_t)r * P.ldo + c0;
          if (ncv == 8 && al16(o)) *reinterpret_cast<uint4*>(o) = tc::pack_bf16x8(y);
          else
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j < ncv) o[j] = __float2bfloat16_rn(y[j]);
          if (P.xh) {
            bf16* x = P.xh + (int64_t)r * P.ldx + c0;
            if (ncv == 8 && al16(x)) *reinterpret_cast<uint4*>(x) = tc::pack_bf16x8(xh);
            else
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (j < ncv) x[j] = __float2bfloat16_rn(xh[j]);
          }
          if (cg == 0 && P.rstd) P.rstd[r] = rs;
        }
      } else {
        float x[8];
        {
          const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&xpre[it]);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 f = __bfloat1622float2(h[k]);
            x[2 * k] = f.x, x[2 * k + 1] = f.y;
          }
        }
        float dn[8], s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const bool ok = rv && c0 + j < nreal;
          x[j] = ok ? x[j] : 0.f;
          const float n = fmaf(x[j], s_g[c0 + j], s_beta[c0 + j]);
          dn[j] = ok ? ((EPI == GE_BWD_LN_RELU) ? (n > 0.f ? acc[j] : 0.f) : acc[j] * sech2_fast(n)) : 0.f;
          const float dxh = dn[j] * s_g[c0 + j];
          s1 += dxh;
          s2 += dxh * x[j];
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
          s1 += __shfl_xor_sync(0xffffffffu, s1, o);
          s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        }
        if (it == 0) stamp(9);
        const float m1 = s1 / (float)N, m2 = s2 / (float)N;
        const float rs = rspre[it];
        float dx[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const bool ok = rv && c0 + j < nreal;
          dx[j] = ok ? rs * (dn[j] * s_g[c0 + j] - m1 - x[j] * m2) : 0.f;
          cp[0][j] += dx[j];
          cp[1][j] += dn[j] * x[j];
          cp[2][j] += dn[j];
        }
        if (rv && c0 < nreal) {
          const int ncv = min(8, nreal - c0);
          bf16* o = P.out + (int64_t)r * P.ldo + c0;
          if (ncv == 8 && al16(o)) *reinterpret_cast<uint4*>(o) = tc::pack_bf16x8(dx);
          else
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j < ncv) o[j] = __float2bfloat16_rn(dx[j]);
        }
      }
    }
    stamp(10);
    if constexpr (EPI == GE_BWD_LN_TANH || EPI == GE_BWD_LN_RELU) {
      if (P.part) {
        // column sums over the CTA's rows: lanes 8 apart share a column group; then the 8 warps
#pragma unroll
        for (int k = 0; k < 3; ++k)
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            cp[k][j] += __shfl_xor_sync(0xffffffffu, cp[k][j], 8);
            cp[k][j] += __shfl_xor_sync(0xffffffffu, cp[k][j], 16);
          }
        if (lane < 8)
#pragma unroll
          for (int k = 0; k < 3; ++k)
#pragma unroll
            for (int j = 0; j < 8; ++j) s_col[warp][k][c0 + j] = cp[k][j];
        stamp(11);
        __syncthreads();
        stamp(12);
        for (int e = tid; e < 3 * nreal; e += kThreads) {
          const int k = e / nreal, c = e - k * nreal;
          float s = 0.f;
#pragma unroll
          for (int w = 0; w < 8; ++w) s += s_col[w][k][c];
          P.part[((int64_t)(mt * ks + (int)kr) * 3 + k) * N + c] = s;
        }
      }
    }
  } else if constexpr (EPI == GE_TG_FWD || EPI == GE_TG_BWD) {
    // 8 threads per row, action dimension d = tid % 8 (+ 8)
    for (int it = 0; it < nit; ++it) {
      const int rr = (tid >> 3) + 32 * it;
      const int r = m0 + (int)kr * R + rr;
      const bool rv = r < P.M && rr < R;
      if constexpr (EPI == GE_TG_FWD) {
        const int A = N / 2;
        float lp = 0.f;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int d = cg + 8 * u;
          if (rv && d < A) {
            const float mu = recv_col(rr, d) + s_bias[d], l = recv_col(rr, A + d) + s_bias[A + d];
            if (P.tgo) {
              P.tgo[(int64_t)r * 2 * A + d] = mu;
              P.tgo[(int64_t)r * 2 * A + A + d] = l;
            }
            const float tl = tanhf(l);
            const float log_std = P.lo + 0.5f * (P.hi - P.lo) * (tl + 1.f);
            const float sd = expf(log_std);
            const float e = tg_pre[it][u][2];
            const float uu = fmaf(sd, e, mu);
            const float at = tanhf(uu);
            if (P.act) P.act[(int64_t)r * A + d] = at;
            if (P.act_bf) P.act_bf[(int64_t)r * P.ld_act_bf + d] = __float2bfloat16_rn(at);
            lp += -0.5f * e * e - log_std - 0.5f * kLog2Pi - logf(sech2f(uu) + kSquashEps);
          }
        }
        // butterfly over the 8-lane group (deterministic order)
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) lp += __shfl_xor_sync(0xffffffffu, lp, o);
        if (rv && cg == 0 && P.logp) P.logp[r] = lp;
      } else {
        const int A = N - P.acc_col0;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int d = cg + 8 * u;
          if (rv && d < A) {
            const float mu = tg_pre[it][u][0], l = tg_pre[it][u][1], e = tg_pre[it][u][2];
            const float tl = tanhf(l);
            const float log_std = P.lo + 0.5f * (P.hi - P.lo) * (tl + 1.f);
            const float sd = expf(log_std);
            const float uu = fmaf(sd, e, mu);
            const float a1 = tanhf(uu);
            const float om = sech2f(uu);
            const float du = recv_col(rr, P.acc_col0 + d) * om + dlp * (2.f * a1 * om / (om + kSquashEps));
            const float dls = du * sd * e - dlp;
            P.out[(int64_t)r * P.ldo + d] = __float2bfloat16_rn(du);
            P.out[(int64_t)r * P.ldo + A + d] = __float2bfloat16_rn(dls * 0.5f * (P.hi - P.lo) * sech2f(l));
          }
        }
      }
    }
  }
  stamp(7);
  tc::fence_before_sync();
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // peers' copies from this CTA done
  stamp(4);
  if (b.dbg && tid == 0) b.dbg[blockIdx.x * kDbgSlots + 15] = (unsigned long long)(EPI | 64) | ((unsigned long long)gridDim.x << 8);
  if (warp == 0) tc::tmem_dealloc(tmem, 64);
}

typedef void (*GemmKernel)(GBatch);
GemmKernel kernel_sk_for(int epi) {
  switch (epi) {
    case GE_LN_RELU: return k_gemm_sk<GE_LN_RELU>;
    case GE_LN_TANH: return k_gemm_sk<GE_LN_TANH>;
    case GE_TG_FWD: return k_gemm_sk<GE_TG_FWD>;
    case GE_BWD_LN_RELU: return k_gemm_sk<GE_BWD_LN_RELU>;
    case GE_BWD_LN_TANH: return k_gemm_sk<GE_BWD_LN_TANH>;
    case GE_TG_BWD: return k_gemm_sk<GE_TG_BWD>;
  }
  return nullptr;
}
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

GemmKernel kernel_ln16_for(int epi) {
  switch (epi) {
    case GE_BWD_LN_RELU: return k_gemm_ln16<GE_BWD_LN_RELU>;
    case GE_BWD_LN_TANH: return k_gemm_ln16<GE_BWD_LN_TANH>;
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
  const int n = g_dbg_tiles * kDbgSlots < max_entries ? g_dbg_tiles * kDbgSlots : max_entries;
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

static int plan_fail(int line) {  // a planning / tensor-map failure: -1 (SQUINT_DEBUG_SYNC names the check)
  static const bool dbg = getenv("SQUINT_DEBUG_SYNC") != nullptr;
  if (dbg) fprintf(stderr, "[squint] gemm_launch: plan check at gemm.cu:%d failed\n", line);
  return -1;
}

int gemm_launch(GemmBuilder& gb, cudaStream_t s) {
  GBatch& b = gb.b;
  if (gb.err) return plan_fail(__LINE__);
  if (b.nprob == 0) return 0;
  // plan tiles.  LayerNorm epilogues need whole rows: with N >= 128 the row is split over a
  // cluster of cs CTAs of 64-column multiples (more SMs share the epilogue work).
  const int epi0 = b.p[0].epi;
  const bool ln_launch = epi0 == GE_LN_RELU || epi0 == GE_LN_TANH || epi0 == GE_BWD_LN_RELU || epi0 == GE_BWD_LN_TANH;
  b.cs = 1;
  // split-K clusters for narrow row-complete layers with several K blocks (k_gemm_sk)
  b.ks = 1;
  {
    bool ok = kernel_sk_for(epi0) != nullptr;
    int minkb = 1 << 30;
    for (int i = 0; i < b.nprob && ok; ++i) {
      int k = 0;
      for (int j = 0; j < b.p[i].nseg; ++j) k += b.p[i].seg[j].nkb;
      minkb = k < minkb ? k : minkb;
      ok = ((b.p[i].N + 15) & ~15) <= 64;
    }
    if (ok) b.ks = minkb >= 4 ? 4 : (minkb >= 2 ? 2 : 1);
    // no more split CTAs than two waves: at c3 (B = 4096: 32 row tiles per problem) the 4-way
    // split ran 512 CTAs in 3.5 waves
    int mtiles = 0;
    for (int i = 0; i < b.nprob; ++i) mtiles += (b.p[i].M + 127) / 128;
    // (up to two waves since two-stage split CTAs share an SM: c3 2157 -> 2177 updates/s)
    while (b.ks > 1 && mtiles * b.ks > 2 * 148) b.ks >>= 1;
    // LayerNorm split-K over 8 CTAs (16 rows each) when every CTA still gets >= 1 K block
    int tiles8 = 0;
    for (int i = 0; i < b.nprob; ++i) tiles8 += 8 * ((b.p[i].M + 127) / 128);
    if (ok && minkb >= 8 && tiles8 <= 148 &&
        (epi0 == GE_LN_TANH || epi0 == GE_LN_RELU || epi0 == GE_BWD_LN_TANH || epi0 == GE_BWD_LN_RELU))
      b.ks = 8;  // (one wave on the 148 SMs; c2 4845 -> 4975 updates/s)
  }
  if (b.ks > kGemmMaxSplitK) return plan_fail(__LINE__);
  for (int i = 0; i < b.nprob; ++i)  // column partials: [mtiles * ks][3][N] floats must fit
    if (b.p[i].part && (int64_t)((b.p[i].M + 127) / 128) * b.ks * 3 * b.p[i].N > b.p[i].part_cap) return plan_fail(__LINE__);
  if (ln_launch && b.ks == 1) {
    int cs = 8;
    for (int i = 0; i < b.nprob; ++i) {
      const int n = b.p[i].N;
      // 512-wide rows (c3's critic): 2 CTAs of 256 columns (c3 1538 -> 1683 updates/s against 4 of 128:
      // half the CTAs, each A tile loaded by 2 CTAs instead of 4)
      const int c = n >= 512 && n % 512 == 0 ? 2 : (n >= 256 && n % 256 == 0 ? 4 : (n >= 128 && n % 128 == 0 ? 2 : 1));
      cs = c < cs ? c : cs;
    }
    // LayerNorm backward over 256-column rows: 8-CTA clusters of 32 columns (16 per warp in the
    // epilogue; measured per update 236 / 207 / 186 us with 1 / 2 / 4 CTAs per row)
    // (only for 256-wide rows: at 512 columns, 8 CTAs of 64 measured far slower than 4 of 128 --
    // c3 1227 -> 976 updates/s with the forward and backward both at 8)
    // and only while the 8-CTA tiling still fits one wave on the 148 SMs (c3's B = 4096 would
    // need two)
    if (cs == 4 && (epi0 == GE_BWD_LN_RELU || epi0 == GE_BWD_LN_TANH)) {
      bool ok = true;
      int ctas = 0;
      for (int i = 0; i < b.nprob; ++i) {
        ok = ok && b.p[i].N == 256;
        ctas += 8 * ((b.p[i].M + 127) / 128);
      }
      if (ok && ctas <= 148) cs = 8;
    }
    b.cs = cs;
  }
  int t = 0, bmax = 0;
  for (int i = 0; i < b.nprob; ++i) {
    GProb& p = b.p[i];
    if (p.M < 1 || p.N < 1 || p.nseg < 1) return plan_fail(__LINE__);
    for (int k = 0; k < p.nseg; ++k)  // TMA box starts along a contiguous dim: 16-byte aligned
      if ((p.seg[k].a_mn && (p.a_m & 7)) || (p.seg[k].b_mn && (p.b_n & 7)) || (p.seg[k].a_k & 63) ||
          (p.seg[k].b_k & 63))
        return plan_fail(__LINE__);
    const int n16 = (p.N + 15) & ~15;
    if (row_complete(p.epi)) {
      if (n16 > 512) return plan_fail(__LINE__);
      p.bn = b.cs > 1 ? p.N / b.cs : n16;
      if (b.ks > 1 && n16 > 64) return plan_fail(__LINE__);
    } else if (p.epi == GE_DW) {
      p.bn = n16 >= 256 ? 64 : (n16 > 128 ? 128 : n16);
    } else {
      p.bn = n16 > 128 ? 128 : n16;
      // the masked dh of the encoder at c3 (4096 x 1600, K = 50): 416 tiles of 128 columns ran in
      // 2.8 waves; 256-column tiles halve the waves
      if (p.epi == GE_RELU_MASK && n16 >= 1024 && ((p.M + 127) / 128) * ((p.N + 127) / 128) > 148) p.bn = 256;
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
  // weight gradients (one segment, both operands MN-major): wide TMA boxes of KW K blocks
  b.wide = 1;
  if (epi0 == GE_DW) {
    bool ok = true;
    int nbb = 0, maxk = 0;
    for (int i = 0; i < b.nprob && ok; ++i) {
      const GProb& p = b.p[i];
      ok = p.nseg == 1 && p.seg[0].a_mn && p.seg[0].b_mn;
      nbb = host_bbytes(p, 1) / 8192 > nbb ? host_bbytes(p, 1) / 8192 : nbb;
      maxk = p.seg[0].nkb > maxk ? p.seg[0].nkb : maxk;
    }
    for (int kw = 4; ok && kw >= 2; kw >>= 1) {
      const int sbytes = (2 + nbb) * kw * 8192;
      if (maxk >= kw && 2 * sbytes + 2048 <= 200 * 1024) {
        b.wide = kw;
        b.stage_bytes = sbytes;
        b.prefetch_b = 0;  // the pre-wait B prefetch assumes the one-K-block stage layout
        break;
      }
    }
  }
  int S = (200 * 1024) / b.stage_bytes;
  S = S > kMaxStages ? kMaxStages : S;
  int maxkb = 0;  // no more stages than K blocks
  for (int i = 0; i < b.nprob; ++i) {
    int k = 0;
    for (int j = 0; j < b.p[i].nseg; ++j) k += b.p[i].seg[j].nkb;
    maxkb = k > maxkb ? k : maxkb;
  }
  if (b.ks > 1) maxkb = (maxkb + b.ks - 1) / b.ks;  // K blocks per cluster CTA
  if (b.wide > 1) maxkb = (maxkb + b.wide - 1) / b.wide;  // stages hold b.wide K blocks
  S = S > maxkb ? maxkb : S;
  S = S < 2 ? 2 : S;
  // forward LayerNorm launches of more than one wave (c3: 256 CTAs of 128 x 256 tiles): two stages
  // (96 KB) so that two CTAs fit on an SM (TMEM 2 x 256 columns) and one CTA's epilogue overlaps the
  // other's main loop, where the second wave used to start only after the first had finished
  if ((b.p[0].epi == GE_LN_RELU || b.p[0].epi == GE_LN_TANH) && b.ks == 1 && t > 148) {
    bool fit = true;
    for (int i = 0; i < b.nprob; ++i) fit = fit && b.p[i].bn <= 256;
    if (fit && 2 * b.stage_bytes <= 96 * 1024) S = 2;
  }
  if (b.ks > 1 && t * b.ks > 148) S = 2;  // two split CTAs per SM (two-wave split-K launches)
  if ((size_t)S * b.stage_bytes > 200 * 1024) return plan_fail(__LINE__);
  b.nstages = S;
  // A multicast across a LayerNorm cluster (its CTAs share the rows): only without ring reuse,
  // so no stage is refilled before every CTA's MMAs consumed it
  {
    b.mcast = (b.cs > 1 && b.ks == 1 && maxkb <= S) ? 1 : 0;
  }
  // tensor maps
  b.nmaps = 0;
  for (int i = 0; i < b.nprob; ++i) {
    GProb& p = b.p[i];
    const int bn16 = (p.bn + 15) & ~15;
    for (int k = 0; k < p.nseg; ++k) {
      GSeg& g = p.seg[k];
      if (b.nmaps + 2 > kGemmMaxMaps) return plan_fail(__LINE__);
      if (tmap_get(gb.segA[i][k], g.a_mn ? 64 * b.wide : 128, &b.maps[b.nmaps])) return plan_fail(__LINE__);
      g.amap = b.nmaps++;
      if (tmap_get(gb.segB[i][k], g.b_mn ? 64 * b.wide : (bn16 > 256 ? 256 : bn16), &b.maps[b.nmaps])) return plan_fail(__LINE__);
      g.bmap = b.nmaps++;
    }
  }
  // epilogue tensor maps (64-column x 32-row bf16 boxes)
  for (int i = 0; i < b.nprob; ++i) {
    GProb& p = b.p[i];
    p.omap = p.xmap = p.ymap = -1;
    const bool ln = p.epi == GE_LN_RELU || p.epi == GE_LN_TANH;
    const bool bwd = p.epi == GE_BWD_LN_RELU || p.epi == GE_BWD_LN_TANH;
    if (b.ks > 1) continue;  // the split-K epilogue stores directly
    if (ln || bwd || p.epi == GE_RELU_MASK) {
      if (b.nmaps + 3 > kGemmMaxMaps || !p.out) return plan_fail(__LINE__);
      if (tmap_get(Mat{p.out, p.M, p.N, p.ldo}, 32, &b.maps[b.nmaps])) return plan_fail(__LINE__);
      p.omap = b.nmaps++;
    }
    if ((ln && p.xh) || bwd) {
      if (!p.xh || tmap_get(Mat{p.xh, p.M, p.N, p.ldx}, 32, &b.maps[b.nmaps])) return plan_fail(__LINE__);
      p.xmap = b.nmaps++;
    }
    if (p.epi == GE_RELU_MASK) {
      if (!p.y || tmap_get(Mat{p.y, p.M, p.N, p.ldy}, 32, &b.maps[b.nmaps])) return plan_fail(__LINE__);
      p.ymap = b.nmaps++;
    }
  }
  size_t smem = (size_t)S * b.stage_bytes;
  if (b.ks > 1) {
    if (smem < (size_t)kSkRecvBytes) smem = kSkRecvBytes;
    smem += kSkRecvBytes;
  } else if (smem < (size_t)kEpiBytes) {
    smem = kEpiBytes;
  }
  if (b.p[0].epi == GE_DW) smem += 2048;  // ones tile (bias gradients)
  // LayerNorm backward: x_hat boxes prefetched past the ring when they fit
  b.xpre_off = 0;
  if (b.ks == 1 && (b.p[0].epi == GE_BWD_LN_RELU || b.p[0].epi == GE_BWD_LN_TANH)) {
    int ng = 0;
    for (int i = 0; i < b.nprob; ++i) {
      const int g = (b.p[i].bn + 63) / 64;
      ng = g > ng ? g : ng;
    }
    const size_t xb = (size_t)4 * 4 * 4096;  // 4 pairs x (up to) 4 boxes
    if (ng <= 4 && smem + xb + 1024 + kStaticSmem <= 227 * 1024) {
      b.xpre_off = (int)smem;
      smem += xb;
    }
  }
  smem += 1024;
  const int epi = b.p[0].epi;
  for (int i = 1; i < b.nprob; ++i)
    if (b.p[i].epi != epi) return plan_fail(__LINE__);  // one epilogue kind per launch (template instance)
  // LayerNorm backward over whole slices of 64..256 columns: the 16-warp epilogue kernel
  // (measured for the forward LayerNorm too: no gain, its second pass is bound by the two TMA
  // stores per tile -- c3 ln_relu 124 vs 118 us per update -- so k_gemm keeps it)
  bool bln = b.ks == 1 && (epi == GE_BWD_LN_RELU || epi == GE_BWD_LN_TANH);
  for (int i = 0; i < b.nprob && bln; ++i) {
    const GProb& p = b.p[i];
    bln = p.bn >= 64 && p.bn <= 256 && p.bn % 64 == 0 && p.N % p.bn == 0 && p.M % 128 == 0;
  }
  GemmKernel kern = b.ks > 1 ? kernel_sk_for(epi) : (bln ? kernel_ln16_for(epi) : kernel_for(epi));
  if (!kern) return plan_fail(__LINE__);
  static size_t attr_smem[48] = {0};  // opt-in limit set so far per instance
  const int ai = epi + (b.ks > 1 ? 16 : 0) + (bln ? 32 : 0);
  if (smem > attr_smem[ai]) {
    cudaError_t ae = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // the largest shared-memory carveout, so that two ~110 KB CTAs (two-stage LayerNorm launches)
    // can share an SM
    if (ae == cudaSuccess) ae = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (ae != cudaSuccess) return (int)ae;
    attr_smem[ai] = smem;
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
        cudaMalloc(&g_dbg_dev, 256 * 64 * kDbgSlots * sizeof(unsigned long long));
        cudaMemset(g_dbg_dev, 0, 256 * 64 * kDbgSlots * sizeof(unsigned long long));
      }
      if (all) {
        b.dbg = g_dbg_dev + (size_t)(me % 256) * 64 * kDbgSlots;
        g_dbg_tiles = 256 * 64;
      } else if (me == atoi(dbg_env)) {
        g_dbg_tiles = b.ntiles * b.ks < 4096 ? b.ntiles * b.ks : 4096;
        b.dbg = g_dbg_dev;
      }
    }
  }
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = dim3(b.ntiles * b.ks);
  cfg.blockDim = dim3(bln ? kBlnThreads : kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (g_pdl) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (b.cs > 1 || b.ks > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = b.cs > 1 ? b.cs : b.ks;
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
    static const char* sk_names[9] = {"k_gemm_sk<ln_relu>", "k_gemm_sk<ln_tanh>", "", "k_gemm_sk<tg_fwd>",
                                      "k_gemm_sk<bwd_ln_relu>", "k_gemm_sk<bwd_ln_tanh>", "", "k_gemm_sk<tg_bwd>", ""};
    double flops = 0;
    for (int i = 0; i < b.nprob; ++i)
      for (int k = 0; k < b.p[i].nseg; ++k) flops += 2.0 * b.p[i].M * (double)(b.p[i].N - b.p[i].acc_col0) * b.p[i].seg[k].k;
    static const char* ln16_names[6] = {"", "", "", "", "k_gemm_ln16<bwd_ln_relu>", "k_gemm_ln16<bwd_ln_tanh>"};
    note_launch(s, b.ks > 1 ? sk_names[epi] : (bln ? ln16_names[epi] : names[epi]), flops, 0);
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, b);
  static const bool dbg = getenv("SQUINT_DEBUG_SYNC") != nullptr;
  if (dbg) {
    cudaError_t se = cudaStreamSynchronize(s);
    fprintf(stderr, "[squint] k_gemm epi=%d nprob=%d tiles=%d ks=%d cs=%d wide=%d stages=%d stage_bytes=%d -> %s\n", epi, b.nprob,
            b.ntiles, b.ks, b.cs, b.wide, S, b.stage_bytes, cudaGetErrorString(se));
    for (int i = 0; i < b.nprob; ++i) {
      int K = 0;
      for (int k = 0; k < b.p[i].nseg; ++k) K += b.p[i].seg[k].k;
      fprintf(stderr, "[squint]   problem %d: M %d N %d K %d bn %d tiles %d\n", i, b.p[i].M, b.p[i].N, K, b.p[i].bn,
              b.p[i].tiles_n * ((b.p[i].M + 127) / 128));
    }
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
