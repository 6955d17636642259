// encoder_tc.cu -- the conv encoder (Q7: conv3x3/s2 + ReLU, conv3x3/s1 + ReLU) as implicit-GEMM
// tcgen05 tiles for the bf16 path: forward (a3-a5 / a16) and backward (a10).
//
// Forward, persistent CTAs over groups of G = 5 images (5 * 49 = 245 conv1 rows = 2 UMMA
// tiles, 5 * 25 = 125 conv2 rows = 1 tile):
//   images (replay gather + random shift, Q5; or squint of rendered frames, a1/a16) -> smem
//   conv1: A1[row = (img, oy, ox)][k = (ci, ki, kj)] im2col (K 27 of 32), B = W1 [C][27];
//          epilogue: acc / 255 + b1 (Q6: raw u8 values are exact in bf16), ReLU -> y1 (smem,
//          HWC bf16; also global for the backward)
//   conv2: A2[row = (img, oy, ox)][k = (tap, c)] gathered from y1 one 64-wide K block at a
//          time into a ring of smem stages (the tensor core consumes block kb while the
//          threads build kb + 1), B = W2 permuted to [o][(tap, c)];
//          epilogue: + b2, ReLU -> h (global bf16, HWC flatten pix * C + o).
// Weights are converted from the fp32 master once per CTA into 128B-swizzled K-major tiles.
#include <cuda_runtime.h>

#include "common.cuh"
#include "encoder.cuh"
#include "tc.cuh"

namespace sq {

namespace {

constexpr int kG = 5;        // images per group
constexpr int kThr = 256;
constexpr int kS2 = 4;       // conv2 A ring stages

__device__ __forceinline__ uint32_t sw(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

struct FwdSmem {
  uint32_t w1, w2, a1, y1, a2, xs;  // byte offsets (1024-aligned where tiles)
  uint32_t total;
};
__host__ __device__ inline FwdSmem fwd_smem(int C) {
  FwdSmem s;
  const int nkb2 = (9 * C + 63) / 64;
  uint32_t o = 0;
  auto take = [&](uint32_t b) {
    uint32_t r = o;
    o += (b + 1023) & ~1023u;
    return r;
  };
  s.w1 = take(C * 128);
  s.w2 = take(nkb2 * C * 128);
  s.a1 = take(2 * 16384);
  s.a2 = take(kS2 * 16384);
  s.y1 = take(kG * 49 * C * 2);
  s.xs = take(kG * 3 * 256);
  s.total = o;
  return s;
}

__device__ __forceinline__ uint32_t rhe64(uint32_t s) { return (s + 31u + ((s >> 6) & 1u)) >> 6; }

__global__ void __launch_bounds__(kThr, 1) k_enc_fwd_tc(const __grid_constant__ EncFwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);  // stays a shared pointer
  __shared__ uint64_t bar1, bar2, empty[kS2];
  __shared__ uint32_t tmem_slot;
  const int C = a.C, H = a.H;  // H = 16 stored resolution
  const FwdSmem L = fwd_smem(C);
  const int nkb2 = (9 * C + 63) / 64;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ngroups = (a.B + kG - 1) / kG;
  const int total = ngroups * a.nsrc;

  if (warp == 0) tc::tmem_alloc(&tmem_slot, 256);
  if (tid == 32) {
    tc::mbar_init(&bar1, 1);
    tc::mbar_init(&bar2, 1);
    for (int i = 0; i < kS2; ++i) tc::mbar_init(&empty[i], 1);
    tc::fence_mbar_init();
  }
  // weights -> bf16 swizzled tiles.  W1 [C][27] (k = ci*9 + ki*3 + kj, the master order) padded
  // to 64; W2 [C][(tap, c)] from the master [o][c][ki][kj].
  for (int e = tid; e < C * 8; e += kThr) {
    const int o = e >> 3, ch = e & 7;
    float f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = ch * 8 + j;
      f[j] = k < 27 ? a.w1[o * 27 + k] : 0.f;
    }
    *reinterpret_cast<uint4*>(sm + L.w1 + sw(o, ch)) = tc::pack_bf16x8(f);
  }
  for (int e = tid; e < nkb2 * C * 8; e += kThr) {
    const int kb = e / (C * 8), rem = e - kb * C * 8, o = rem >> 3, ch = rem & 7;
    float f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = kb * 64 + ch * 8 + j, t = k / C, c = k - t * C;
      f[j] = t < 9 ? a.w2[(o * C + c) * 9 + t] : 0.f;
    }
    *reinterpret_cast<uint4*>(sm + L.w2 + kb * C * 128 + sw(o, ch)) = tc::pack_bf16x8(f);
  }
  // conv1 A: K columns 32..63 stay zero for the CTA's lifetime
  for (int e = tid; e < 256 * 4; e += kThr) {
    const int r = e >> 2, ch = 4 + (e & 3);
    *reinterpret_cast<uint4*>(sm + L.a1 + (r >> 7) * 16384 + sw(r & 127, ch)) = make_uint4(0, 0, 0, 0);
  }
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_slot;
  const uint32_t t_c1 = tmem, t_c2 = tmem + 2 * C;  // conv1: 2 tiles x C cols; conv2: C cols
  const uint32_t id_c = tc::idesc_bf16(128, C);
  uint8_t* xs = sm + L.xs;
  bf16_t* y1s = reinterpret_cast<bf16_t*>(sm + L.y1);
  const float inv255 = 1.0f / 255.0f;
  int it2 = 0, gi = 0;

  for (int job = blockIdx.x; job < total; job += gridDim.x, ++gi) {
    const int src = job / ngroups, g = job - src * ngroups;
    const int b0 = g * kG;
    // ---- 1. images (u8) + replay row gathers ------------------------------------------
    if (a.mode == 0) {
      const uint8_t* R = a.src[src];
      for (int e = tid; e < kG * 3 * 256; e += kThr) {
        const int i = e / 768, rem = e - i * 768, cc = rem >> 8, p = rem & 255, y = p >> 4, x = p & 15;
        const int b = b0 + i;
        uint8_t u = 0;
        if (b < a.B) {
          const int64_t row = a.idx[b];
          const int dx = a.shifts[b * 4 + 2 * src], dy = a.shifts[b * 4 + 2 * src + 1];
          const int sy = min(max(y + dy - a.pad, 0), H - 1), sx = min(max(x + dx - a.pad, 0), H - 1);
          u = R[row * 768 + cc * 256 + sy * 16 + sx];
          if (src == 0 && a.img0) a.img0[(int64_t)b * 768 + rem] = u;
        }
        xs[e] = u;
      }
    } else {
      // squint: 8x8 block sums of 128x128 frames, round half to even (Q1), optional ring write
      const uint8_t* Fr = a.src[0];
      for (int e = tid; e < kG * 3 * 16 * 8; e += kThr) {  // (img, ch, oy, 16-byte column chunk)
        const int ck = e & 7, t1 = e >> 3, oy = t1 & 15, t2 = t1 >> 4, cc = t2 % 3, i = t2 / 3;
        const int b = b0 + i;
        uint32_t lo = 0, hi = 0;
        if (b < a.B) {
          const uint8_t* s = Fr + (((int64_t)b * 3 + cc) * 128 + oy * 8) * 128 + ck * 16;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            const uint4 v = __ldcs(reinterpret_cast<const uint4*>(s + r * 128));
            lo = __dp4a(v.x, 0x01010101u, __dp4a(v.y, 0x01010101u, lo));
            hi = __dp4a(v.z, 0x01010101u, __dp4a(v.w, 0x01010101u, hi));
          }
        }
        const uint32_t q0 = rhe64(lo), q1 = rhe64(hi);
        const int p = (i * 3 + cc) * 256 + oy * 16 + 2 * ck;
        xs[p] = (uint8_t)q0;
        xs[p + 1] = (uint8_t)q1;
        if (b < a.B && a.ring)
          *reinterpret_cast<uint16_t*>(a.ring + (a.slots[b] * 3 + cc) * 256 + oy * 16 + 2 * ck) = (uint16_t)(q0 | (q1 << 8));
      }
    }
    for (int jb = 0; jb < a.ngj[src]; ++jb) {
      const GatherJob& gj = a.gj[src][jb];
      for (int e = tid; e < kG * gj.width; e += kThr) {
        const int i = e / gj.width, j = e - i * gj.width, b = b0 + i;
        if (b < a.B) {
          const int64_t row = gj.use_idx ? a.idx[b] : (int64_t)b;
          gj.dst[(int64_t)b * gj.ld + gj.col + j] = __float2bfloat16_rn(gj.src[row * gj.width + j]);
        }
      }
    }
    __syncthreads();
    // ---- 2. conv1 im2col (K columns 0..31) ------------------------------------------------
    for (int e = tid; e < 256 * 4; e += kThr) {
      const int r = e >> 2, ch = e & 3;
      const int i = r / 49, p = r - i * 49, oy = p / 7, ox = p - oy * 7;
      float f[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = ch * 8 + j, ci = k / 9, t = k - ci * 9, ki = t / 3, kj = t - ki * 3;
        f[j] = (r < kG * 49 && k < 27) ? (float)xs[(i * 3 + ci) * 256 + (2 * oy + ki) * 16 + 2 * ox + kj] : 0.f;
      }
      *reinterpret_cast<uint4*>(sm + L.a1 + (r >> 7) * 16384 + sw(r & 127, ch)) = tc::pack_bf16x8(f);
    }
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    if (tid == 0) {
      tc::fence_after_sync();
      const uint32_t a0 = tc::smem_u32(sm + L.a1), w0 = tc::smem_u32(sm + L.w1);
#pragma unroll
      for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int k = 0; k < 2; ++k)
          tc::mma_bf16(t_c1 + t * C, tc::sdesc_k128(a0 + t * 16384 + 32 * k), tc::sdesc_k128(w0 + 32 * k), id_c, k);
      tc::mma_commit(&bar1);
    }
    tc::mbar_wait(&bar1, gi & 1);
    tc::fence_after_sync();
    // ---- 3. conv1 epilogue: warp w -> tile w / 4, TMEM lanes 32 (w % 4) --------------------
    {
      const int t = warp >> 2, q = warp & 3, r = t * 128 + q * 32 + lane;
      const int i = r / 49, p = r - i * 49, b = b0 + i;
      const bool rv = r < kG * 49;
      for (int c0 = 0; c0 < C; c0 += 32) {
        float v[32];
        tc::tmem_ld32(t_c1 + t * C + c0 + ((uint32_t)(q * 32) << 16), v);
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = fmaxf(fmaf(v[j], inv255, a.b1[c0 + j]), 0.f);
        if (rv) {
#pragma unroll
          for (int j8 = 0; j8 < 4; ++j8) {
            float f[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = v[j8 * 8 + j];
            const uint4 u = tc::pack_bf16x8(f);
            *reinterpret_cast<uint4*>(y1s + (i * 49 + p) * C + c0 + j8 * 8) = u;
            if (a.y1b && src == 0 && b < a.B)
              *reinterpret_cast<uint4*>(a.y1b + ((int64_t)b * 49 + p) * C + c0 + j8 * 8) = u;
          }
        }
      }
    }
    tc::fence_before_sync();
    __syncthreads();
    // ---- 4. conv2: ring of gathered K blocks ----------------------------------------------
    for (int kb = 0; kb < nkb2; ++kb, ++it2) {
      const int st = it2 % kS2;
      if (it2 >= kS2) tc::mbar_wait(&empty[st], ((it2 / kS2) - 1) & 1);
      uint8_t* A2 = sm + L.a2 + st * 16384;
      for (int e = tid; e < 128 * 8; e += kThr) {
        const int r = e >> 3, ch = e & 7;
        const int k = kb * 64 + ch * 8, t = k / C, c = k - t * C;
        uint4 u = make_uint4(0, 0, 0, 0);
        if (r < kG * 25 && t < 9) {
          const int i = r / 25, p = r - i * 25, oy = p / 5, ox = p - oy * 5, ki = t / 3, kj = t - ki * 3;
          u = *reinterpret_cast<const uint4*>(y1s + (i * 49 + (oy + ki) * 7 + ox + kj) * C + c);
        }
        *reinterpret_cast<uint4*>(A2 + sw(r, ch)) = u;
      }
      tc::fence_async_smem();
      tc::fence_before_sync();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after_sync();
        const uint32_t a0 = tc::smem_u32(A2), w0 = tc::smem_u32(sm + L.w2 + kb * C * 128);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc::mma_bf16(t_c2, tc::sdesc_k128(a0 + 32 * k), tc::sdesc_k128(w0 + 32 * k), id_c, (kb | k) != 0);
        tc::mma_commit(&empty[st]);
        if (kb == nkb2 - 1) tc::mma_commit(&bar2);
      }
    }
    tc::mbar_wait(&bar2, gi & 1);
    tc::fence_after_sync();
    // ---- 5. conv2 epilogue: warps 0-3 (125 rows) -> h (HWC bf16) ----------------------------
    if (warp < 4) {
      const int r = warp * 32 + lane, i = r / 25, p = r - i * 25, b = b0 + i;
      bf16_t* hout = a.hb[src];
      for (int c0 = 0; c0 < C; c0 += 32) {
        float v[32];
        tc::tmem_ld32(t_c2 + c0 + ((uint32_t)(warp * 32) << 16), v);
        if (r < kG * 25 && b < a.B) {
#pragma unroll
          for (int j8 = 0; j8 < 4; ++j8) {
            float f[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = fmaxf(v[j8 * 8 + j] + a.b2[c0 + j8 * 8 + j], 0.f);
            *reinterpret_cast<uint4*>(hout + (int64_t)b * a.h_ld + p * C + c0 + j8 * 8) = tc::pack_bf16x8(f);
          }
        }
      }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 256);
}


// ---------------------------------------------------------------------------------------------
// Backward (a10), persistent CTAs over groups of G = 5 images, three GEMMs per group:
//   conv2 dX:  dy1[r1 = (img, y, x)][c] = sum_{t, o} D2[img][(y - ki, x - kj)][o] W2[o][c][t]
//              A K-major, built from D2 (zero outside the 5x5 map), B = W2 as [c][(t, o)];
//              epilogue: dA1 = dy1 * (y1 > 0) (ReLU' of conv1) -> smem, MN-major
//   conv2 dW:  dW2[(t, c)][o] += sum_{r2} y1[img][p2 + t][c] D2[r2][o]     (K = the 125 rows)
//              A MN-major (built from y1), B = D2 (MN-major, as loaded); row 9C of A is 1 on
//              valid rows, so that accumulator row is db2 = sum D2
//   conv1 dW:  dW1[(ci, t)][o] += sum_{r1} x[img][ci][2y + ki][2x + kj] dA1[r1][o] (K = 245 rows)
//              A MN-major (im2col of the raw u8 image; 1/255 applied at the end, Q6), B = dA1;
//              row 27 of A is 1 -> db1
// The dW accumulators stay in TMEM across the CTA's groups; at the end each CTA writes its
// partial in the master layout and k_reduce_enc sums the partials in a fixed order.
constexpr int kSB = 3;  // backward A ring stages

struct BwdSmem {
  uint32_t w2t, d2s, y1s, a1s, xs, ring, total;
};
__host__ __device__ inline BwdSmem bwd_smem(int C) {
  BwdSmem s;
  const int nkb2 = (9 * C + 63) / 64;
  uint32_t o = 0;
  auto take = [&](uint32_t b) {
    uint32_t r = o;
    o += (b + 1023) & ~1023u;
    return r;
  };
  s.w2t = take(nkb2 * C * 128);
  s.d2s = take(2 * 8192);
  s.a1s = take(4 * 8192);
  s.ring = take(kSB * 16384);
  s.y1s = take(256 * C * 2);
  s.xs = take(kG * 768);
  s.total = o;
  return s;
}
__host__ __device__ inline int bwd_stride(int C) { return C * C * 9 + C + C * 27 + C; }

__global__ void __launch_bounds__(kThr, 1) k_enc_bwd_tc(const __grid_constant__ EncBwdArgs a) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar_dx, bar_grp, empty[kSB];
  __shared__ uint32_t tmem_slot;
  const int C = a.C;
  const BwdSmem L = bwd_smem(C);
  const int nkb2 = (9 * C + 63) / 64, nt2 = (9 * C + 1 + 127) / 128, cch = C / 8;
  const uint32_t ncols = C == 32 ? 256u : 512u;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ngroups = (a.B + kG - 1) / kG;

  if (warp == 0) tc::tmem_alloc(&tmem_slot, ncols);
  if (tid == 32) {
    tc::mbar_init(&bar_dx, 1);
    tc::mbar_init(&bar_grp, 1);
    for (int i = 0; i < kSB; ++i) tc::mbar_init(&empty[i], 1);
    tc::fence_mbar_init();
  }
  // B of conv2 dX: W2T[c][(t, o)] = W2[o][c][t], K-major 64-wide tiles
  for (int e = tid; e < nkb2 * C * 8; e += kThr) {
    const int kb = e / (C * 8), rem = e - kb * C * 8, c = rem >> 3, ch = rem & 7;
    float f[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = kb * 64 + ch * 8 + j, t = k / C, o = k - t * C;
      f[j] = t < 9 ? a.w2[(o * C + c) * 9 + t] : 0.f;
    }
    *reinterpret_cast<uint4*>(sm + L.w2t + kb * C * 128 + sw(c, ch)) = tc::pack_bf16x8(f);
  }
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_slot;
  const uint32_t t_dx = tmem, t_w2 = tmem + 2 * C, t_w1 = t_w2 + nt2 * C;
  const uint32_t id_k = tc::idesc_bf16(128, C), id_mn = tc::idesc_bf16_major(128, C, 1, 1);
  bf16_t* y1s = reinterpret_cast<bf16_t*>(sm + L.y1s);
  uint8_t* xs = sm + L.xs;
  int it = 0, gi = 0;

  // ring helper: wait for stage reuse; returns the stage buffer
  auto stage_acquire = [&](int& st) -> uint8_t* {
    st = it % kSB;
    if (it >= kSB) tc::mbar_wait(&empty[st], ((it / kSB) - 1) & 1);
    return sm + L.ring + st * 16384;
  };

  for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++gi) {
    const int b0 = g * kG;
    const bool first = gi == 0;
    // ---- load D2 (MN-major SW128, rows r2 = img * 25 + p), y1 rows (HWC), images ----------------
    for (int e = tid; e < 128 * 8; e += kThr) {
      const int r2 = e >> 3, ch = e & 7, i = r2 / 25, p = r2 - i * 25, b = b0 + i;
      uint4 u = make_uint4(0, 0, 0, 0);
      if (r2 < kG * 25 && b < a.B && ch < cch)
        u = *reinterpret_cast<const uint4*>(a.dA2_hwc + (int64_t)b * a.dA2_ld + p * C + ch * 8);
      const int rr = r2 & 63;
      *reinterpret_cast<uint4*>(sm + L.d2s + (r2 >> 6) * 8192 + sw(rr, ch)) = u;
    }
    for (int e = tid; e < kG * 49 * cch; e += kThr) {
      const int r1 = e / cch, ch = e - r1 * cch, i = r1 / 49, p = r1 - i * 49, b = b0 + i;
      uint4 u = make_uint4(0, 0, 0, 0);
      if (b < a.B) u = *reinterpret_cast<const uint4*>(a.y1_hwc + ((int64_t)b * 49 + p) * C + ch * 8);
      *reinterpret_cast<uint4*>(y1s + r1 * C + ch * 8) = u;
    }
    for (int e = tid; e < kG * 48; e += kThr) {  // 16-byte chunks of the 5 images
      const int i = e / 48, b = b0 + i;
      uint4 u = make_uint4(0, 0, 0, 0);
      if (b < a.B) u = *reinterpret_cast<const uint4*>(a.img + (int64_t)b * 768 + (e - i * 48) * 16);
      *reinterpret_cast<uint4*>(xs + e * 16) = u;
    }
    __syncthreads();
    // ---- conv2 dX (2 row tiles x nkb2 K blocks) --------------------------------------------
    for (int mt = 0; mt < 2; ++mt) {
      for (int kb = 0; kb < nkb2; ++kb, ++it) {
        int st;
        uint8_t* A = stage_acquire(st);
        for (int e = tid; e < 128 * 8; e += kThr) {
          const int rr = e >> 3, ch = e & 7, r1 = mt * 128 + rr;
          const int k = kb * 64 + ch * 8, t = k / C, o0 = k - t * C;
          uint4 u = make_uint4(0, 0, 0, 0);
          if (r1 < kG * 49 && t < 9) {
            const int i = r1 / 49, p = r1 - i * 49, y = p / 7, x = p - y * 7, ki = t / 3, kj = t - ki * 3;
            const int yy = y - ki, xx = x - kj;
            if (yy >= 0 && yy < 5 && xx >= 0 && xx < 5) {
              const int r2 = i * 25 + yy * 5 + xx, q = r2 & 63;
              u = *reinterpret_cast<const uint4*>(sm + L.d2s + (r2 >> 6) * 8192 + sw(q, o0 >> 3));
            }
          }
          *reinterpret_cast<uint4*>(A + sw(rr, ch)) = u;
        }
        tc::fence_async_smem();
        tc::fence_before_sync();
        __syncthreads();
        if (tid == 0) {
          tc::fence_after_sync();
          const uint32_t a0 = tc::smem_u32(A), w0 = tc::smem_u32(sm + L.w2t + kb * C * 128);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc::mma_bf16(t_dx + mt * C, tc::sdesc_k128(a0 + 32 * k), tc::sdesc_k128(w0 + 32 * k), id_k,
                         (kb | k) != 0);
          tc::mma_commit(&empty[st]);
          if (mt == 1 && kb == nkb2 - 1) tc::mma_commit(&bar_dx);
        }
      }
    }
    // ---- conv2 dW (+ db2 via the ones row), accumulated across groups -------------------------
    for (int mt = 0; mt < nt2; ++mt) {
      for (int kb = 0; kb < 2; ++kb, ++it) {
        int st;
        uint8_t* A = stage_acquire(st);
        for (int e = tid; e < 2 * 64 * 8; e += kThr) {  // (atom, K row, chunk)
          const int j = e >> 9, rr = (e >> 3) & 63, ch = e & 7, r2 = kb * 64 + rr;
          const int m0 = mt * 128 + j * 64 + ch * 8, t = m0 / C, c0 = m0 - t * C;
          const int i = r2 / 25, p = r2 - i * 25;
          const bool rv = r2 < kG * 25 && b0 + i < a.B;
          uint4 u = make_uint4(0, 0, 0, 0);
          if (rv) {
            if (t < 9) {
              const int oy = p / 5, ox = p - oy * 5, ki = t / 3, kj = t - ki * 3;
              u = *reinterpret_cast<const uint4*>(y1s + (i * 49 + (oy + ki) * 7 + ox + kj) * C + c0);
            } else if (m0 == 9 * C) {
              u.x = 0x3F80u;  // bf16 1.0 in element 0
            }
          }
          *reinterpret_cast<uint4*>(A + j * 8192 + sw(rr, ch)) = u;
        }
        tc::fence_async_smem();
        tc::fence_before_sync();
        __syncthreads();
        if (tid == 0) {
          tc::fence_after_sync();
          const uint32_t a0 = tc::smem_u32(A), b0s = tc::smem_u32(sm + L.d2s + kb * 8192);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc::mma_bf16(t_w2 + mt * C, tc::sdesc_sw128(a0 + 2048 * k, 8192, 1024),
                         tc::sdesc_sw128(b0s + 2048 * k, 8192, 1024), id_mn, !(first && kb == 0 && k == 0));
          tc::mma_commit(&empty[st]);
        }
      }
    }
    // ---- dX epilogue: dA1 = dy1 * (y1 > 0) -> smem (MN-major rows r1) -------------------------
    tc::mbar_wait(&bar_dx, gi & 1);
    tc::fence_after_sync();
    {
      const int t = warp >> 2, q = warp & 3, rr = q * 32 + lane, r1 = t * 128 + rr;
      for (int c0 = 0; c0 < C; c0 += 32) {
        float v[32];
        tc::tmem_ld32(t_dx + t * C + c0 + ((uint32_t)(q * 32) << 16), v);
#pragma unroll
        for (int j8 = 0; j8 < 4; ++j8) {
          float f[8];
          if (r1 < kG * 49) {
            const uint4 yv = *reinterpret_cast<const uint4*>(y1s + r1 * C + c0 + j8 * 8);
            const __nv_bfloat162* yp = reinterpret_cast<const __nv_bfloat162*>(&yv);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const float2 yf = __bfloat1622float2(yp[j]);
              f[2 * j] = yf.x > 0.f ? v[j8 * 8 + 2 * j] : 0.f;
              f[2 * j + 1] = yf.y > 0.f ? v[j8 * 8 + 2 * j + 1] : 0.f;
            }
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = 0.f;
          }
          const int ch = (c0 >> 3) + j8, q1 = r1 & 63;
          *reinterpret_cast<uint4*>(sm + L.a1s + (r1 >> 6) * 8192 + sw(q1, ch)) = tc::pack_bf16x8(f);
        }
      }
      if (C == 32) {  // dA1 MN-major rows hold 64 elements: zero the unused half
        const int q1 = r1 & 63;
#pragma unroll
        for (int ch = 4; ch < 8; ++ch)
          *reinterpret_cast<uint4*>(sm + L.a1s + (r1 >> 6) * 8192 + sw(q1, ch)) = make_uint4(0, 0, 0, 0);
      }
    }
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    // ---- conv1 dW (+ db1), accumulated across groups ---------------------------------------------
    for (int kb = 0; kb < 4; ++kb, ++it) {
      int st;
      uint8_t* A = stage_acquire(st);
      for (int e = tid; e < 2 * 64 * 8; e += kThr) {
        const int j = e >> 9, rr = (e >> 3) & 63, ch = e & 7, r1 = kb * 64 + rr;
        float f[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) f[q] = 0.f;
        const int i = r1 / 49, p = r1 - i * 49, y = p / 7, x = p - y * 7;
        if (j == 0 && ch < 4 && r1 < kG * 49 && b0 + i < a.B) {
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int m = ch * 8 + q, ci = m / 9, t = m - ci * 9, ki = t / 3, kj = t - ki * 3;
            if (m < 27) f[q] = (float)xs[i * 768 + ci * 256 + (2 * y + ki) * 16 + 2 * x + kj];
            else if (m == 27) f[q] = 1.f;
          }
        }
        *reinterpret_cast<uint4*>(A + j * 8192 + sw(rr, ch)) = tc::pack_bf16x8(f);
      }
      tc::fence_async_smem();
      tc::fence_before_sync();
      __syncthreads();
      if (tid == 0) {
        tc::fence_after_sync();
        const uint32_t a0 = tc::smem_u32(A), b0s = tc::smem_u32(sm + L.a1s + kb * 8192);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc::mma_bf16(t_w1, tc::sdesc_sw128(a0 + 2048 * k, 8192, 1024), tc::sdesc_sw128(b0s + 2048 * k, 8192, 1024),
                       id_mn, !(first && kb == 0 && k == 0));
        tc::mma_commit(&empty[st]);
        if (kb == 3) tc::mma_commit(&bar_grp);
      }
    }
    tc::mbar_wait(&bar_grp, gi & 1);  // every MMA of the group done: smem inputs may be reused
    tc::fence_after_sync();
    __syncthreads();
  }
  // ---- per-CTA partials in the master layout -------------------------------------------------------
  float* part = a.part + (int64_t)blockIdx.x * bwd_stride(C);
  if (gi > 0) {
    const int q = warp & 3;
    for (int mt = warp >> 2; mt < nt2 + 1; mt += 2) {
      const bool w1 = mt == nt2;
      const int m = (w1 ? 0 : mt * 128) + q * 32 + lane;
      const uint32_t base = (w1 ? t_w1 : t_w2 + mt * C) + ((uint32_t)(q * 32) << 16);
      for (int c0 = 0; c0 < C; c0 += 32) {
        float v[32];
        tc::tmem_ld32(base + c0, v);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int o = c0 + j;
          if (!w1) {
            if (m < 9 * C) {
              const int t = m / C, c = m - t * C;
              part[(o * C + c) * 9 + t] = v[j];
            } else if (m == 9 * C) {
              part[C * C * 9 + o] = v[j];
            }
          } else {
            if (m < 27) part[C * C * 9 + C + o * 27 + m] = v[j] * (1.0f / 255.0f);
            else if (m == 27) part[C * C * 9 + C + C * 27 + o] = v[j];
          }
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, ncols);
}

// out[i] = sum over CTA partials, fixed order: 4 threads per output each sum a quarter of the
// partials, then the four quarter sums are added in order.
__global__ void __launch_bounds__(256) k_reduce_enc(const float* __restrict__ part, int nchunk, int C,
                                                    float* __restrict__ gw2, float* __restrict__ gb2,
                                                    float* __restrict__ gw1, float* __restrict__ gb1) {
  __shared__ float red[4][64];
  const int stride = bwd_stride(C);
  const int i = blockIdx.x * 64 + (threadIdx.x & 63), sl = threadIdx.x >> 6;
  const int c0 = (nchunk * sl) / 4, c1 = (nchunk * (sl + 1)) / 4;
  float s = 0.f;
  if (i < stride)
    for (int c = c0; c < c1; ++c) s += __ldg(part + (int64_t)c * stride + i);
  red[sl][threadIdx.x & 63] = s;
  __syncthreads();
  if (sl != 0 || i >= stride) return;
  const int t = threadIdx.x;
  s = ((red[0][t] + red[1][t]) + red[2][t]) + red[3][t];
  const int n2 = C * C * 9;
  if (i < n2) gw2[i] = s;
  else if (i < n2 + C) gb2[i - n2] = s;
  else if (i < n2 + C + C * 27) gw1[i - n2 - C] = s;
  else gb1[i - n2 - C - C * 27] = s;
}

}  // namespace

int launch_enc_fwd_tc(const EncFwdArgs& a, cudaStream_t s) {
  if (a.B == 0) return 0;
  if (a.C % 32 || a.C > 64 || a.H != 16 || a.c_in != 3) return (int)cudaErrorInvalidValue;
  if (a.mode == 1 && a.factor != 8) return (int)cudaErrorInvalidValue;
  const FwdSmem L = fwd_smem(a.C);
  const size_t smem = L.total + 1024;
  cudaFuncSetAttribute(k_enc_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int total = ((a.B + kG - 1) / kG) * a.nsrc;
  const int grid = total < 148 ? total : 148;
  {
    const double img = (double)a.B * a.nsrc, C = a.C;
    const double flops = 2.0 * img * (49.0 * C * 27.0 + 25.0 * 9.0 * C * C);
    const double bytes = a.mode == 1 ? img * (3.0 * 128 * 128 + 2.0 * 25 * C) : img * (768.0 + 2.0 * 25 * C);
    note_launch(s, "k_enc_fwd_tc", flops, bytes);
  }
  k_enc_fwd_tc<<<grid, kThr, smem, s>>>(a);
  return (int)cudaGetLastError();
}

size_t enc_bwd_tc_partial_floats(int C, int B) {
  const int ngroups = (B + kG - 1) / kG;
  return (size_t)(ngroups < 148 ? ngroups : 148) * bwd_stride(C);
}

int launch_enc_bwd_tc(const EncBwdArgs& a, cudaStream_t s) {
  if (a.B == 0) return 0;
  if (a.C % 32 || a.C > 64 || a.H != 16 || a.c_in != 3) return (int)cudaErrorInvalidValue;
  const BwdSmem L = bwd_smem(a.C);
  const size_t smem = L.total + 1024;
  cudaFuncSetAttribute(k_enc_bwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int ngroups = (a.B + kG - 1) / kG;
  const int grid = ngroups < 148 ? ngroups : 148;
  {
    const double C = a.C;
    note_launch(s, "k_enc_bwd_tc", 2.0 * a.B * (2.0 * 25.0 * 9.0 * C * C + 49.0 * 27.0 * C), 0);
  }
  k_enc_bwd_tc<<<grid, kThr, smem, s>>>(a);
  const int stride = bwd_stride(a.C);
  note_launch(s, "k_reduce_enc", 0, 0);
  k_reduce_enc<<<(stride + 63) / 64, 256, 0, s>>>(a.part, grid, a.C, a.gw2, a.gb2, a.gw1, a.gb1);
  return (int)cudaGetLastError();
}

}  // namespace sq
