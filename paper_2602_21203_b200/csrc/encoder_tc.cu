// encoder_tc.cu -- the conv encoder (Q7: conv3x3/s2 + ReLU, conv3x3/s1 + ReLU) as implicit-GEMM
// tcgen05 tiles for the bf16 path: forward (a3-a5 / a16) and backward (a10).
//
// Weights: k_conv_tiles converts the fp32 master conv weights once per call/update into the
// exact 128B-swizzled bf16 shared-memory images the kernels use; each CTA then pulls its image
// with one bulk copy (no per-CTA conversion).
//
// Forward, one group of G = 7 images per CTA (7 * 49 = 343 conv1 rows = 3 UMMA tiles,
// 7 * 25 = 175 conv2 rows = 2 tiles; a c2 update's 2 x 512 images are exactly 148 groups):
//   images (replay gather + random shift with replicate padding, Q5, as 16-byte row loads; or
//   the squint of rendered frames, a1/a16) -> smem u8
//   conv1: A1[row = (img, oy, ox)][k = (ci, ki, kj)] im2col (K 27 of 32), B = W1 [C][27];
//          epilogue: acc / 255 + b1 (Q6: raw u8 values are exact in bf16), ReLU -> y1 (smem, HWC
//          bf16; also global for the backward)
//   conv2: A2[row = (img, oy, ox)][k = (tap, c)] gathered from y1, one 64-wide K block (both row
//          tiles) per ring stage: the tensor core consumes block kb while the threads build kb+1;
//          B = W2 as [o][(tap, c)]; epilogue: + b2, ReLU -> h (global bf16, HWC flatten pix*C + o).
//
// Backward, one group of G = 4 images per CTA (196 conv1 rows = 2 tiles, 100 conv2 rows = 1 tile):
//   conv2 dX:  dy1[r1 = (img, y, x)][c] = sum_{t, o} D2[img][(y - ki, x - kj)][o] W2[o][c][t]
//              A K-major, built from D2 (zero outside the 5x5 map), B = W2 as [c][(t, o)];
//              epilogue: dA1 = dy1 * (y1 > 0) (ReLU' of conv1) -> smem, MN-major
//   conv2 dW:  dW2[(t, c)][o] += sum_{r2} y1[img][p2 + t][c] D2[r2][o]     (K = the 100 rows)
//              A MN-major (built from y1), B = D2 (MN-major, as loaded); row 9C of A is 1 on
//              valid rows, so that accumulator row is db2 = sum D2
//   conv1 dW:  dW1[(ci, t)][o] += sum_{r1} x[img][ci][2y + ki][2x + kj] dA1[r1][o] (K = 196 rows)
//              A MN-major (im2col of the raw u8 image; 1/255 applied at the end, Q6), B = dA1;
//              row 27 of A is 1 -> db1
// The dW accumulators stay in TMEM across the CTA's groups; each CTA writes its partial rows
// (row-major, coalesced) and k_reduce_enc sums the partials in a fixed order into the master
// layout (deterministic).
#include <cuda_runtime.h>

#include <cstdlib>

#include "common.cuh"
#include "encoder.cuh"
#include "tc.cuh"

namespace sq {

namespace {

constexpr int kThr = 256;
constexpr int kGF = 7;  // forward images per group
constexpr int kGB = 4;  // backward images per group

__device__ __forceinline__ uint32_t sw(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }
__device__ __forceinline__ uint32_t rhe64(uint32_t s) { return (s + 31u + ((s >> 6) & 1u)) >> 6; }

__host__ __device__ inline int nkb2_of(int C) { return (9 * C + 63) / 64; }
__host__ __device__ inline uint32_t fwd_wbytes(int C) { return (uint32_t)(C * 128 + nkb2_of(C) * C * 128); }
__host__ __device__ inline uint32_t bwd_wbytes(int C) { return (uint32_t)(nkb2_of(C) * C * 128); }
__host__ __device__ inline uint32_t bwd_woff(int C) { return (fwd_wbytes(C) + 1023u) & ~1023u; }

// ---- weight images --------------------------------------------------------------------------
// fwd: W1 tile [o][k = ci*9 + ki*3 + kj] (K 27 padded to 64), W2 tiles [kb][o][k = t*C + c];
// bwd: W2T tiles [kb][c][k = t*C + o].  Element (row, k) of a tile at sw(row, k / 8) + 2 (k % 8).
__global__ void __launch_bounds__(256) k_conv_tiles(const float* __restrict__ w1, const float* __restrict__ w2, int C,
                                                    uint8_t* __restrict__ out) {
  grid_wait();
  grid_trigger();
  const int nkb2 = nkb2_of(C);
  const int n1 = C * 8, n2 = nkb2 * C * 8;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n1 + 2 * n2; e += gridDim.x * blockDim.x) {
    float f[8];
    uint8_t* dst;
    if (e < n1) {
      const int o = e >> 3, ch = e & 7;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = ch * 8 + j;
        f[j] = k < 27 ? w1[o * 27 + k] : 0.f;
      }
      dst = out + sw(o, ch);
    } else if (e < n1 + n2) {
      const int x = e - n1, kb = x / (C * 8), rem = x - kb * C * 8, o = rem >> 3, ch = rem & 7;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = kb * 64 + ch * 8 + j, t = k / C, c = k - t * C;
        f[j] = t < 9 ? w2[(o * C + c) * 9 + t] : 0.f;
      }
      dst = out + C * 128 + kb * C * 128 + sw(o, ch);
    } else {
      const int x = e - n1 - n2, kb = x / (C * 8), rem = x - kb * C * 8, c = rem >> 3, ch = rem & 7;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int k = kb * 64 + ch * 8 + j, t = k / C, o = k - t * C;
        f[j] = t < 9 ? w2[(o * C + c) * 9 + t] : 0.f;
      }
      dst = out + bwd_woff(C) + kb * C * 128 + sw(c, ch);
    }
    *reinterpret_cast<uint4*>(dst) = tc::pack_bf16x8(f);
  }
}

__device__ unsigned long long g_enc_stamps[160][32];  // debug: per-CTA phase timestamps (SQUINT_ENC_DBG)
__device__ __forceinline__ void enc_stamp_any(bool on, int k) {  // caller picks the thread
  if (on && blockIdx.x < 160) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_enc_stamps[blockIdx.x][k] = t;
  }
}
__device__ __forceinline__ void enc_stamp(bool on, int k) {
  if (on && threadIdx.x == 0 && blockIdx.x < 160) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_enc_stamps[blockIdx.x][k] = t;
  }
}
// ---- forward ---------------------------------------------------------------------------------
template <int C>
struct FwdL {
  static constexpr uint32_t w = 0;
  static constexpr uint32_t ring = (C * 128 + ((9 * C + 63) / 64) * C * 128 + 1023) & ~1023u;  // A1 / A2 stages
  static constexpr uint32_t y1 = ring + 65536;
  // conv1 output as the conv2 A operand: rows = (image, 7x7 pixel) flattened, C bf16 per row,
  // K-major with the 64-byte (C = 32) / 128-byte (C = 64) swizzle; 416 rows cover the three
  // 128-row output tiles plus the largest tap shift (2 * 7 + 2)
  static constexpr uint32_t y1_rows = 416;
  static constexpr uint32_t xs = y1 + ((y1_rows * C * 2 + 1023) & ~1023u);
  static constexpr uint32_t total = xs + kGF * 768;
};
// byte offset of (row, 16-byte chunk) in a K-major swizzled tile with C-channel rows (C * 2 bytes):
// the hardware XORs address bits [4, 4 + b) with bits [7, 7 + b) (b = 2 for 64-byte rows, 3 for
// 128-byte rows), so a descriptor may start at any row
template <int C>
__device__ __forceinline__ uint32_t y1_off(int row, int chunk) {
  const uint32_t a = (uint32_t)(row * C * 2 + chunk * 16);
  return C == 32 ? a ^ (((a >> 7) & 3u) << 4) : a ^ (((a >> 7) & 7u) << 4);
}
__device__ __forceinline__ uint64_t sdesc_sw(uint32_t saddr, int rowbytes) {  // K-major, SW64 / SW128
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1u << 16;
  d |= (uint64_t)(((8u * rowbytes) >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1u << 46;
  d |= (uint64_t)(rowbytes == 128 ? 2u : 4u) << 61;
  return d;
}

// byte x of a 16-byte row held as a uint4
__device__ __forceinline__ uint32_t byte_of(const uint4& v, int x) {
  const uint32_t w = x < 8 ? (x < 4 ? v.x : v.y) : (x < 12 ? v.z : v.w);
  return (w >> ((x & 3) * 8)) & 0xFFu;
}

template <int C>
__global__ void __launch_bounds__(kThr, 1) k_enc_fwd_tc(const __grid_constant__ EncFwdArgs a) {
  using L = FwdL<C>;
  constexpr uint32_t kCols = C == 32 ? 256u : 512u;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);  // stays a shared pointer
  __shared__ uint64_t wbar, bar1, bar2;
  __shared__ uint32_t tmem_slot;
  __shared__ int s_koff[32];  // conv1 tap k = ci*9 + ki*3 + kj -> input byte offset ci*256 + ki*16 + kj
  const int H = a.H;  // 16
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, q = warp & 3, hh = warp >> 2;
  const int ngroups = (a.B + kGF - 1) / kGF;
  const int total = ngroups * a.nsrc;
  // forward phases in stamp slots 10..15 (the backward uses 0..9)
  enc_stamp(a.dbg, 10);

  if (warp == 0) tc::tmem_alloc(&tmem_slot, kCols);
  if (tid == 32) {
    tc::mbar_init(&wbar, 1);
    tc::mbar_init(&bar1, 1);
    tc::mbar_init(&bar2, 1);
    tc::fence_mbar_init();
  }
  if (warp == 2) {
    const int k = lane, ci = k / 9, t = k - ci * 9, ki = t / 3, kj = t - ki * 3;
    s_koff[k] = k < 27 ? ci * 256 + ki * 16 + kj : 0;
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  grid_wait();  // weight tiles and inputs come from earlier kernels
  grid_trigger();
  if (tid == 0) {
    tc::mbar_expect_tx(&wbar, fwd_wbytes(C));
    tc::bulk_load_1d(sm + L::w, a.wtiles, fwd_wbytes(C), &wbar);
  }
  const uint32_t tmem = tmem_slot;
  const uint32_t t_c1 = tmem, t_c2 = tmem + 3 * C;  // conv1, conv2: 3 row tiles x C columns each
  const uint32_t id_c = tc::idesc_bf16(128, C);
  uint8_t* xs = sm + L::xs;
  const float inv255 = 1.0f / 255.0f;
  int gi = 0;

  // ---- 1. images (u8) + replay row gathers of group `job` into xs (and global outputs); run
  // for the next group while this group's MMAs and epilogues run (xs is free once the
  // im2col has read it)
  auto stage = [&](int job) {
    const int src = job / ngroups, g = job - src * ngroups;
    const int b0 = g * kGF;
    if (a.mode == 0) {
      // one 16-pixel row per item: shifted crop with replicate padding from the source row
      const uint8_t* R = a.src[src];
      for (int e = tid; e < kGF * 48; e += kThr) {
        const int i = e / 48, rem = e - i * 48, cc = rem >> 4, y = rem & 15;
        const int b = b0 + i;
        uint4 o = make_uint4(0, 0, 0, 0);
        if (b < a.B) {
          const int64_t row = a.idx[b];
          const int dx = a.shifts[b * 4 + 2 * src], dy = a.shifts[b * 4 + 2 * src + 1];
          const int sy = min(max(y + dy - a.pad, 0), H - 1);
          const uint4 v = *reinterpret_cast<const uint4*>(R + row * 768 + cc * 256 + sy * 16);
          uint32_t wv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            uint32_t acc = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) acc |= byte_of(v, min(max(4 * k + j + dx - a.pad, 0), H - 1)) << (8 * j);
            wv[k] = acc;
          }
          o = make_uint4(wv[0], wv[1], wv[2], wv[3]);
          uint8_t* dump = src == 0 ? a.img0 : a.img1;
          if (dump) *reinterpret_cast<uint4*>(dump + (int64_t)b * 768 + cc * 256 + y * 16) = o;
        }
        *reinterpret_cast<uint4*>(xs + i * 768 + cc * 256 + y * 16) = o;
      }
    } else if (a.factor == 1) {
      // frames already at the stored resolution (squinted by squint_insert2): 768-byte copies
      const uint8_t* Fr = a.src[0];
      for (int e = tid; e < kGF * 48; e += kThr) {
        const int i = e / 48, rem = e - i * 48, b = b0 + i;
        uint4 o = make_uint4(0, 0, 0, 0);
        if (b < a.B) {
          o = __ldcs(reinterpret_cast<const uint4*>(Fr + (int64_t)b * 768) + rem);
          if (a.ring) reinterpret_cast<uint4*>(a.ring + a.slots[b] * 768)[rem] = o;
        }
        reinterpret_cast<uint4*>(xs + i * 768)[rem] = o;
      }
    } else {
      // squint: 8x8 block sums of 128x128 frames, round half to even (Q1), optional ring write
      // (img, ch, oy, 16-byte column chunk) items; a thread keeps the loads of kU items (kU x 8 x
      // 16 bytes) in flight before reducing them: the frames stream from HBM once, and the per-SM
      // memory-level parallelism sets the rate
      const uint8_t* Fr = a.src[0];
      constexpr int kItems = kGF * 3 * 16 * 8, kU = 3;
      for (int e0 = tid; e0 < kItems; e0 += kU * kThr) {
        uint4 v[kU][8];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int e = e0 + u * kThr;
          const int ck = e & 7, t1 = e >> 3, oy = t1 & 15, t2 = t1 >> 4, cc = t2 % 3, i = t2 / 3;
          const int b = b0 + i;
          if (e < kItems && b < a.B) {
            const uint8_t* s = Fr + (((int64_t)b * 3 + cc) * 128 + oy * 8) * 128 + ck * 16;
#pragma unroll
            for (int r = 0; r < 8; ++r) v[u][r] = __ldcs(reinterpret_cast<const uint4*>(s + r * 128));
          } else {
#pragma unroll
            for (int r = 0; r < 8; ++r) v[u][r] = make_uint4(0, 0, 0, 0);
          }
        }
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int e = e0 + u * kThr;
          if (e >= kItems) continue;
          const int ck = e & 7, t1 = e >> 3, oy = t1 & 15, t2 = t1 >> 4, cc = t2 % 3, i = t2 / 3;
          const int b = b0 + i;
          uint32_t lo = 0, hi = 0;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            lo = __dp4a(v[u][r].x, 0x01010101u, __dp4a(v[u][r].y, 0x01010101u, lo));
            hi = __dp4a(v[u][r].z, 0x01010101u, __dp4a(v[u][r].w, 0x01010101u, hi));
          }
          const uint32_t q0 = rhe64(lo), q1 = rhe64(hi);
          const int p = (i * 3 + cc) * 256 + oy * 16 + 2 * ck;
          *reinterpret_cast<uint16_t*>(xs + p) = (uint16_t)(q0 | (q1 << 8));
          if (b < a.B && a.ring)
            *reinterpret_cast<uint16_t*>(a.ring + (a.slots[b] * 3 + cc) * 256 + oy * 16 + 2 * ck) = (uint16_t)(q0 | (q1 << 8));
        }
      }
    }
    for (int jb = 0; jb < a.ngj[src]; ++jb) {
      const GatherJob& gj = a.gj[src][jb];
      for (int e = tid; e < kGF * gj.width; e += kThr) {
        const int i = e / gj.width, j = e - i * gj.width, b = b0 + i;
        if (b < a.B) {
          const int64_t row = gj.use_idx ? a.idx[b] : (int64_t)b;
          gj.dst[(int64_t)b * gj.ld + gj.col + j] = __float2bfloat16_rn(gj.src[row * gj.width + j]);
        }
      }
    }
  };
  if (blockIdx.x < total) stage(blockIdx.x);
  for (int job = blockIdx.x; job < total; job += gridDim.x, ++gi) {
    const int src = job / ngroups, g = job - src * ngroups;
    const int b0 = g * kGF;
    (void)src;
    __syncthreads();
    enc_stamp(a.dbg && gi == 0, 11);
    // ---- 2. conv1 im2col: 3 row tiles, K 0..26 from the image (k = ci*9 + ki*3 + kj at byte
    // offset koff[k] from the output pixel's top-left input byte), 27..63 zero -----------------
    for (int e = tid; e < 384 * 8; e += kThr) {
      const int r = e >> 3, ch = e & 7;
      float f[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) f[j] = 0.f;
      if (ch < 4 && r < kGF * 49) {
        const int i = r / 49, p = r - i * 49, oy = p / 7, ox = p - oy * 7;
        const uint8_t* px = xs + i * 768 + 2 * oy * 16 + 2 * ox;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = ch * 8 + j;
          if (k < 27) f[j] = (float)px[s_koff[k]];
        }
      }
      *reinterpret_cast<uint4*>(sm + L::ring + (r >> 7) * 16384 + sw(r & 127, ch)) = tc::pack_bf16x8(f);
    }
    tc::fence_async_smem();
    tc::fence_before_sync();
    __syncthreads();
    if (tid == 0) {
      tc::mbar_wait(&wbar, 0);  // weight image landed (first group; completed phase afterwards)
      tc::fence_after_sync();
      const uint32_t a0 = tc::smem_u32(sm + L::ring), w0 = tc::smem_u32(sm + L::w);
#pragma unroll
      for (int t = 0; t < 3; ++t)
#pragma unroll
        for (int k = 0; k < 2; ++k)
          tc::mma_bf16(t_c1 + t * C, tc::sdesc_k128(a0 + t * 16384 + 32 * k), tc::sdesc_k128(w0 + 32 * k), id_c, k);
      tc::mma_commit(&bar1);
    }
    if (job + (int)gridDim.x < total) stage(job + (int)gridDim.x);  // overlaps the MMAs below
    tc::mbar_wait(&bar1, gi & 1);
    tc::fence_after_sync();
    enc_stamp(a.dbg && gi == 0, 12);
    // ---- 3. conv1 epilogue: warp (q, hh) -> tiles hh, hh + 2 ------------------------------------
    for (int t = hh; t < 3; t += 2) {
      const int r = t * 128 + q * 32 + lane;
      const int i = r / 49, p = r - i * 49, b = b0 + i;
      const bool rv = r < kGF * 49;
#pragma unroll
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
            *reinterpret_cast<uint4*>(sm + L::y1 + y1_off<C>(r, (c0 + j8 * 8) / 8)) = u;
            if (a.y1b && src == 0 && b < a.B)
              *reinterpret_cast<uint4*>(a.y1b + ((int64_t)b * 49 + p) * C + c0 + j8 * 8) = u;
          }
        }
      }
    }
    tc::fence_async_smem();  // y1 (generic stores) -> the tensor core's operand reads
    tc::fence_before_sync();
    __syncthreads();
    enc_stamp(a.dbg && gi == 0, 13);
    // ---- 4. conv2 as nine row-shifted GEMMs: output position o = i*49 + oy*7 + ox of the full 7x7
    // grid reads y1 row o + ki*7 + kj for tap (ki, kj), so tap t's A operand is y1 itself started
    // t's shift rows later (no im2col); positions with oy or ox > 4 are computed and dropped ----
    if (tid == 0) {
      tc::fence_after_sync();
      const uint32_t y0 = tc::smem_u32(sm + L::y1), w0 = tc::smem_u32(sm + L::w + C * 128);
#pragma unroll
      for (int t = 0; t < 3; ++t)
        for (int tap = 0; tap < 9; ++tap) {
          const int shift = (tap / 3) * 7 + tap % 3;
          // W2 K-block layout: k = tap * C + c in blocks of 64 (128-byte swizzled rows)
          const int kb = (tap * C) / 64, koff = (tap * C) % 64;
#pragma unroll
          for (int k = 0; k < C / 16; ++k)
            tc::mma_bf16(t_c2 + t * C, sdesc_sw(y0 + (t * 128 + shift) * C * 2 + 32 * k, C * 2),
                         tc::sdesc_k128(w0 + kb * C * 128 + (koff + 16 * k) * 2), id_c, (tap | k) != 0);
        }
      tc::mma_commit(&bar2);
    }
    tc::mbar_wait(&bar2, gi & 1);
    tc::fence_after_sync();
    enc_stamp(a.dbg && gi == 0, 14);
    // ---- 5. conv2 epilogue: warp (q, hh) -> tiles hh, hh + 2; valid 5x5 positions -> h (HWC) ----
    {
      bf16_t* hout = a.hb[src];
      for (int t = hh; t < 3; t += 2) {
        const int r = t * 128 + q * 32 + lane, i = r / 49, p = r - i * 49, oy = p / 7, ox = p - oy * 7, b = b0 + i;
        const bool ok = i < kGF && oy < 5 && ox < 5 && b < a.B;
#pragma unroll
        for (int c0 = 0; c0 < C; c0 += 32) {
          float v[32];
          tc::tmem_ld32(t_c2 + t * C + c0 + ((uint32_t)(q * 32) << 16), v);
          if (ok) {
#pragma unroll
            for (int j8 = 0; j8 < 4; ++j8) {
              float f[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) f[j] = fmaxf(v[j8 * 8 + j] + a.b2[c0 + j8 * 8 + j], 0.f);
              *reinterpret_cast<uint4*>(hout + (int64_t)b * a.h_ld + (oy * 5 + ox) * C + c0 + j8 * 8) = tc::pack_bf16x8(f);
            }
          }
        }
      }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
  }
  if (tid == 0 && gi == 0) tc::mbar_wait(&wbar, 0);  // never exit with the bulk copy in flight
  tc::fence_before_sync();
  __syncthreads();
  enc_stamp(a.dbg, 15);
  if (warp == 0) tc::tmem_dealloc(tmem, kCols);
}

// ---- forward, warp-specialised and pipelined across a CTA's groups ------------------------------
// (replay gather + shift, mode 0, and pre-squinted frames, mode 1 with factor 1.)  The round-1 kernel
// above runs each group's phases back to back with the whole CTA; here they run in separate roles so
// the tensor core works through one group's conv2 while the CUDA cores stage and im2col the next
// group and run the previous group's epilogues:
//   P  warps 0-7   images of group i -> xs (u8, two buffers; group i+1's global loads in flight
//                  during group i's im2col), conv1 im2col -> A1                (a1_full / a1_empty)
//   E1 warps 8-11  conv1 accumulator T1 -> ReLU(acc / 255 + b1) -> y1 (smem) + y1b (global)
//                                                       (t1_full / t1_empty, y1_full / y1_empty)
//   E2 warps 12-15 conv2 accumulator T2 -> ReLU(acc + b2) -> h (global)      (t2_full / t2_empty)
//   M  warp 16     conv1 MMAs (A1, W1) -> T1; conv2 as nine row-shifted MMAs per tile (y1, W2) -> T2
// Every barrier completes once per group; TMEM holds T1 (3 C columns) and T2 (3 C columns).
constexpr int kPW = 12;               // producer warps
constexpr int kWsWarps = kPW + 9;     // + conv1 / conv2 epilogue teams (4 + 4) + the MMA warp
template <int C>
struct FwdW {
  static constexpr uint32_t w = 0;
  // conv1 A: 384 rows x 32 K (27 used) bf16, 64-byte rows with the 64-byte swizzle
  static constexpr uint32_t a1 = (C * 128 + ((9 * C + 63) / 64) * C * 128 + 1023) & ~1023u;
  static constexpr uint32_t y1sz = (416u * C * 2 + 1023) & ~1023u;
  static constexpr uint32_t y1 = a1 + 384 * 64;                 // 2 buffers (group parity)
  static constexpr uint32_t xs = y1 + 2 * y1sz;                 // 2 buffers of kGF images
  static constexpr uint32_t total = xs + 2 * kGF * 768;
  // fused squint (act, mode 1 with factor 8; C = 32 only): a 2-slot ring of rendered 3x128x128 frames
  static constexpr uint32_t fring = (total + 1023) & ~1023u;
  static constexpr uint32_t total_sq = fring + 2 * 49152;
};

template <int C>
__global__ void __launch_bounds__(kWsWarps * 32, 1) k_enc_fwd_ws(const __grid_constant__ EncFwdArgs a) {
  using L = FwdW<C>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t wbar, a1_full, a1_empty, t1_full, t1_empty, y1_full[2], y1_empty[2], t2_full, t2_empty, fbar[2];
  __shared__ uint32_t tmem_slot;
  __shared__ int s_koff[32];
  __shared__ float s_b1[64], s_b2[64];
  // mode 0: this CTA's replay rows and shifts, group i image ii at [i * kGF + ii] (read once up front so
  // a group's image loads are one memory round trip; groups beyond kMaxLoc read them from global memory)
  constexpr int kMaxLoc = 32;
  __shared__ int64_t s_row[kMaxLoc * kGF];
  __shared__ uint8_t s_dx[kMaxLoc * kGF], s_dy[kMaxLoc * kGF];
  const int H = a.H;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ngroups = (a.B + kGF - 1) / kGF;
  const int total = ngroups * a.nsrc;
  const int nloc = blockIdx.x < total ? (total - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
  enc_stamp(a.dbg, 10);
  if (warp == 0) tc::tmem_alloc(&tmem_slot, 512);
  if (tid == 32) {
    tc::mbar_init(&wbar, 1);
    tc::mbar_init(&a1_full, kPW);
    tc::mbar_init(&a1_empty, 1);
    tc::mbar_init(&t1_full, 1);
    tc::mbar_init(&t1_empty, 4);
    tc::mbar_init(&y1_full[0], 4);
    tc::mbar_init(&y1_full[1], 4);
    tc::mbar_init(&y1_empty[0], 1);
    tc::mbar_init(&y1_empty[1], 1);
    tc::mbar_init(&t2_full, 1);
    tc::mbar_init(&t2_empty, 4);
    tc::mbar_init(&fbar[0], 1);
    tc::mbar_init(&fbar[1], 1);
    tc::fence_mbar_init();
  }
  if (warp == 2) {
    const int k = lane, ci = k / 9, t = k - ci * 9, ki = t / 3, kj = t - ki * 3;
    s_koff[k] = k < 27 ? ci * 256 + ki * 16 + kj : 0;
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  grid_wait();  // weight tiles, inputs and biases come from earlier kernels
  grid_trigger();
  if (tid < C) {
    s_b1[tid] = a.b1[tid];
    s_b2[tid] = a.b2[tid];
  }
  if (a.mode == 0)
    for (int e = tid; e < min(nloc, kMaxLoc) * kGF; e += kWsWarps * 32) {
      const int i = e / kGF, ii = e - i * kGF, job = blockIdx.x + i * gridDim.x;
      const int src = job / ngroups, b = (job - src * ngroups) * kGF + ii;
      if (b < a.B) {
        s_row[e] = a.idx[b];
        s_dx[e] = a.shifts[b * 4 + 2 * src];
        s_dy[e] = a.shifts[b * 4 + 2 * src + 1];
      }
    }
  if (tid == 32) {
    tc::mbar_expect_tx(&wbar, fwd_wbytes(C));
    tc::bulk_load_1d(sm + L::w, a.wtiles, fwd_wbytes(C), &wbar);
  }
  __syncthreads();  // s_b1, s_b2
  const uint32_t tmem = tmem_slot;
  const uint32_t t_c1 = tmem, t_c2 = tmem + 3 * C;
  uint8_t* xs = sm + L::xs;

  if (warp < kPW) {
    // ---- P: stage + conv1 im2col --------------------------------------------------------------------
    // The global loads of group i + 1's images (replay gather + shift, or 768-byte pre-squinted rows)
    // are issued into registers before group i's im2col, so their latency hides behind it; xs alternates
    // between two buffers.
    const int pt = tid;  // 0 .. kPW * 32 - 1
    constexpr int NPT = kPW * 32, NU = (kGF * 48 + NPT - 1) / NPT;

    // fused squint: frame k of this CTA (k = i * kGF + ii) streams into ring slot k % 2 by one bulk copy
    // (49,152 B, completion on fbar[k % 2]); the copy of frame k + 2 is issued once frame k is reduced
    const bool squint = a.mode == 1 && a.factor == 8;
    const int nfr = nloc * kGF;
    auto frame_b = [&](int k) {  // image index of this CTA's frame k, or -1
      const int job = blockIdx.x + (k / kGF) * gridDim.x;
      const int b = (job % ngroups) * kGF + k % kGF;
      return b < a.B ? b : -1;
    };
    auto issue_frame = [&](int k) {
      const int b = k < nfr ? frame_b(k) : -1;
      if (pt == 0 && b >= 0) {
        tc::mbar_expect_tx(&fbar[k & 1], 49152u);
        tc::bulk_load_1d(sm + L::fring + (k & 1) * 49152, a.src[0] + (int64_t)b * 49152, 49152u, &fbar[k & 1]);
      }
    };
    if (squint) {
      issue_frame(0);
      issue_frame(1);
    }
    uint4 rvA[NU], rvB[NU];  // image rows of two groups in flight (group parity)
    int rdxA[NU], rdxB[NU];
    // replay row gathers of s, a, s' (GatherJobs): each thread's items of the flattened (job, image,
    // column) list, loaded with the group's images
    constexpr int NG = 2;  // <= 2 * 256 items: 7 images x (12 + 6 + 12 + 12) columns per source at most
    float gvA[NG], gvB[NG];
    auto gj_item = [&](int src, int e, int& jb, int& ii, int& jj) -> bool {
      for (jb = 0; jb < a.ngj[src]; ++jb) {
        const int n = kGF * a.gj[src][jb].width;
        if (e < n) {
          ii = e / a.gj[src][jb].width;
          jj = e - ii * a.gj[src][jb].width;
          return true;
        }
        e -= n;
      }
      return false;
    };
    auto load_stage = [&](int i, uint4 (&rv)[NU], int (&rdx)[NU], float (&gv)[NG]) {  // group i -> registers
      const int job = blockIdx.x + i * gridDim.x;
      const int src = job / ngroups, g = job - src * ngroups, b0 = g * kGF;
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const int e = pt + u * NPT;
        rv[u] = make_uint4(0, 0, 0, 0);
        rdx[u] = -1;
        if (e < kGF * 48) {
          const int ii = e / 48, rem = e - ii * 48, b = b0 + ii;
          if (b < a.B) {
            if (a.mode == 0) {
              const int cc = rem >> 4, y = rem & 15, si = i * kGF + ii;
              const int64_t row = i < kMaxLoc ? s_row[si] : a.idx[b];
              const int dx = i < kMaxLoc ? s_dx[si] : a.shifts[b * 4 + 2 * src];
              const int dy = i < kMaxLoc ? s_dy[si] : a.shifts[b * 4 + 2 * src + 1];
              const int sy = min(max(y + dy - a.pad, 0), H - 1);
              rv[u] = *reinterpret_cast<const uint4*>(a.src[src] + row * 768 + cc * 256 + sy * 16);
              rdx[u] = dx;
            } else {
              rv[u] = __ldcs(reinterpret_cast<const uint4*>(a.src[0] + (int64_t)b * 768) + rem);
              rdx[u] = a.pad;  // no horizontal shift
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < NG; ++u) {
        int jb, ii, jj;
        gv[u] = 0.f;
        if (gj_item(src, pt + u * NPT, jb, ii, jj) && b0 + ii < a.B) {
          const GatherJob& gj = a.gj[src][jb];
          const int64_t row =
              gj.use_idx ? (i < kMaxLoc && a.mode == 0 ? s_row[i * kGF + ii] : a.idx[b0 + ii]) : (int64_t)(b0 + ii);
          gv[u] = gj.src[row * gj.width + jj];
        }
      }
    };
    auto store_stage = [&](int i, uint8_t* xb, const uint4 (&rv)[NU], const int (&rdx)[NU], const float (&gv)[NG]) {
      const int job = blockIdx.x + i * gridDim.x;
      const int src = job / ngroups, g = job - src * ngroups, b0 = g * kGF;
#pragma unroll
      for (int u = 0; u < NU; ++u) {
        const int e = pt + u * NPT;
        if (e >= kGF * 48) continue;
        const int ii = e / 48, rem = e - ii * 48, b = b0 + ii;
        uint4 o = make_uint4(0, 0, 0, 0);
        if (rdx[u] >= 0) {
          if (a.mode == 0) {
            const int dx = rdx[u];
            uint32_t wv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              uint32_t acc = 0;
#pragma unroll
              for (int j = 0; j < 4; ++j) acc |= byte_of(rv[u], min(max(4 * k + j + dx - a.pad, 0), H - 1)) << (8 * j);
              wv[k] = acc;
            }
            o = make_uint4(wv[0], wv[1], wv[2], wv[3]);
            uint8_t* dump = src == 0 ? a.img0 : a.img1;
            if (dump) *reinterpret_cast<uint4*>(dump + (int64_t)b * 768 + rem * 16) = o;
          } else {
            o = rv[u];
            if (a.ring) reinterpret_cast<uint4*>(a.ring + a.slots[b] * 768)[rem] = o;
          }
        }
        reinterpret_cast<uint4*>(xb + ii * 768)[rem] = o;
      }
#pragma unroll
      for (int u = 0; u < NG; ++u) {
        int jb, ii, jj;
        if (gj_item(src, pt + u * NPT, jb, ii, jj) && b0 + ii < a.B) {
          const GatherJob& gj = a.gj[src][jb];
          gj.dst[(int64_t)(b0 + ii) * gj.ld + gj.col + jj] = __float2bfloat16_rn(gv[u]);
        }
      }
    };
    // two groups ahead: group i + 2's loads are issued while group i is stored and im2col'ed
    if (!squint && nloc > 0) load_stage(0, rvA, rdxA, gvA);
    if (!squint && nloc > 1) load_stage(1, rvB, rdxB, gvB);
    for (int i = 0; i < nloc; ++i) {
      const int job = blockIdx.x + i * gridDim.x;
      const int src = job / ngroups, g = job - src * ngroups, b0 = g * kGF;
      uint8_t* xb = xs + (i & 1) * (kGF * 768);
      if (i == 3 && pt == 0) enc_stamp_any(a.dbg, 16);
      if (squint) {
        // 8x8 block sums of each frame from shared memory, round half to even (Q1) -> xs (+ ring)
        for (int ii = 0; ii < kGF; ++ii) {
          const int k = i * kGF + ii, b = b0 + ii;
          uint8_t* dst = xb + ii * 768;
          if (b < a.B) {
            tc::mbar_wait(&fbar[k & 1], (k >> 1) & 1);
            const uint8_t* F = sm + L::fring + (k & 1) * 49152;
            for (int e = pt; e < 3 * 16 * 8; e += NPT) {  // (channel, output row, 16-byte column chunk)
              const int ck = e & 7, oy = (e >> 3) & 15, cc = e >> 7;
              const uint8_t* srcp = F + (cc * 128 + oy * 8) * 128 + ck * 16;
              uint32_t lo = 0, hi = 0;
#pragma unroll
              for (int r = 0; r < 8; ++r) {
                const uint4 v = *reinterpret_cast<const uint4*>(srcp + r * 128);
                lo = __dp4a(v.x, 0x01010101u, __dp4a(v.y, 0x01010101u, lo));
                hi = __dp4a(v.z, 0x01010101u, __dp4a(v.w, 0x01010101u, hi));
              }
              const uint16_t qv = (uint16_t)(rhe64(lo) | (rhe64(hi) << 8));
              const int off = cc * 256 + oy * 16 + 2 * ck;
              *reinterpret_cast<uint16_t*>(dst + off) = qv;
              if (a.ring) *reinterpret_cast<uint16_t*>(a.ring + a.slots[b] * 768 + off) = qv;
            }
          } else {
            for (int e = pt; e < 48; e += NPT) reinterpret_cast<uint4*>(dst)[e] = make_uint4(0, 0, 0, 0);
          }
          tc::named_bar(1, NPT);  // slot k % 2 read by every P thread
          issue_frame(k + 2);
        }
      } else if (i & 1) {
        store_stage(i, xb, rvB, rdxB, gvB);
      } else {
        store_stage(i, xb, rvA, rdxA, gvA);
      }
      if (i == 3 && pt == 0) enc_stamp_any(a.dbg, 17);
      if (squint)  // (the other modes gather with their images in load_stage / store_stage)
        for (int jb = 0; jb < a.ngj[src]; ++jb) {
          const GatherJob& gj = a.gj[src][jb];
          for (int e = pt; e < kGF * gj.width; e += NPT) {
            const int ii = e / gj.width, jj = e - ii * gj.width, b = b0 + ii;
            if (b < a.B) {
              const int64_t row = gj.use_idx ? a.idx[b] : (int64_t)b;
              gj.dst[(int64_t)b * gj.ld + gj.col + jj] = __float2bfloat16_rn(gj.src[row * gj.width + jj]);
            }
          }
        }
      if (!squint && i + 2 < nloc) {  // in flight during this and the next group's im2col
        if (i & 1)
          load_stage(i + 2, rvB, rdxB, gvB);
        else
          load_stage(i + 2, rvA, rdxA, gvA);
      }
      if (i == 3 && pt == 0) enc_stamp_any(a.dbg, 18);
      tc::named_bar(1, NPT);  // xs[i % 2] complete
      if (i == 3 && pt == 0) enc_stamp_any(a.dbg, 19);
      if (i >= 1) tc::mbar_wait(&a1_empty, (i - 1) & 1);
      if (i == 3 && pt == 0) enc_stamp_any(a.dbg, 20);
      // conv1 im2col: row (img, oy, ox), K 0..26 = (ci, ki, kj) at byte offset koff[k] from the output
      // pixel's top-left input byte; K 27..31 zero (the MMAs read the first 64 bytes of each row)
      // one thread per output row: the 3 x 3 x 3 window as 18 aligned 16-bit loads (columns 2 ox ..
      // 2 ox + 3 of each input row), was 27 byte gathers through an offset table per row
      for (int r = pt; r < 384; r += NPT) {
        float f[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) f[j] = 0.f;
        if (r < kGF * 49) {
          const int ii = r / 49, p = r - ii * 49, oy = p / 7, ox = p - oy * 7;
          const uint8_t* px = xb + ii * 768 + 2 * oy * 16 + 2 * ox;
#pragma unroll
          for (int ci = 0; ci < 3; ++ci)
#pragma unroll
            for (int ki = 0; ki < 3; ++ki) {
              const uint16_t* rp = reinterpret_cast<const uint16_t*>(px + ci * 256 + ki * 16);
              const uint32_t w0 = rp[0], w1 = rp[1];
              const int k = ci * 9 + ki * 3;
              f[k] = (float)(w0 & 0xffu);
              f[k + 1] = (float)(w0 >> 8);
              f[k + 2] = (float)(w1 & 0xffu);
            }
        }
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          float g[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) g[j] = f[ch * 8 + j];
          *reinterpret_cast<uint4*>(sm + L::a1 + y1_off<32>(r, ch)) = tc::pack_bf16x8(g);
        }
      }
      tc::fence_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&a1_full);
      if (i == 0) enc_stamp(a.dbg, 11);
      if (i == 3 && pt == 0) enc_stamp_any(a.dbg, 21);
      if (i == 4 && pt == 0) enc_stamp_any(a.dbg, 30);
    }
  } else if (warp < kPW + 4) {
    // ---- E1: conv1 epilogue -> y1 ---------------------------------------------------------------
    const int q = warp & 3;
    const float inv255 = 1.0f / 255.0f;
    for (int i = 0; i < nloc; ++i) {
      const int job = blockIdx.x + i * gridDim.x;
      const int src = job / ngroups, g = job - src * ngroups, b0 = g * kGF;
      uint8_t* y1b_s = sm + L::y1 + (i & 1) * L::y1sz;  // y1 buffer of this group's parity
      tc::mbar_wait(&t1_full, i & 1);
      if (i >= 2) tc::mbar_wait(&y1_empty[i & 1], ((i - 2) >> 1) & 1);  // conv2 of group i - 2 read it
      tc::fence_after_sync();
      if (i == 3 && warp == kPW && lane == 0) enc_stamp_any(a.dbg, 22);
#pragma unroll 1
      for (int t = 0; t < 3; ++t) {
        const int r = t * 128 + q * 32 + lane;
        const int ii = r / 49, p = r - ii * 49, b = b0 + ii;
        const bool rv = r < kGF * 49;
#pragma unroll
        for (int c0 = 0; c0 < C; c0 += 32) {
          float v[32];
          tc::tmem_ld32(t_c1 + t * C + c0 + ((uint32_t)(q * 32) << 16), v);
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = fmaxf(fmaf(v[j], inv255, s_b1[c0 + j]), 0.f);
          if (rv) {
#pragma unroll
            for (int j8 = 0; j8 < 4; ++j8) {
              float f[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) f[j] = v[j8 * 8 + j];
              const uint4 u = tc::pack_bf16x8(f);
              *reinterpret_cast<uint4*>(y1b_s + y1_off<C>(r, (c0 + j8 * 8) / 8)) = u;
              if (a.y1b && src == 0 && b < a.B)
                *reinterpret_cast<uint4*>(a.y1b + ((int64_t)b * 49 + p) * C + c0 + j8 * 8) = u;
            }
          }
        }
      }
      tc::fence_async_smem();  // y1 (generic stores) -> the tensor core
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive(&y1_full[i & 1]);
        tc::mbar_arrive(&t1_empty);
      }
      if (i == 3 && warp == kPW && lane == 0) enc_stamp_any(a.dbg, 23);
    }
  } else if (warp < kPW + 8) {
    // ---- E2: conv2 epilogue -> h (valid 5x5 positions, HWC) ------------------------------------------
    const int q = warp & 3;
    for (int i = 0; i < nloc; ++i) {
      const int job = blockIdx.x + i * gridDim.x;
      const int src = job / ngroups, g = job - src * ngroups, b0 = g * kGF;
      bf16_t* hout = a.hb[src];
      tc::mbar_wait(&t2_full, i & 1);
      tc::fence_after_sync();
      if (i == 3 && warp == kPW + 4 && lane == 0) enc_stamp_any(a.dbg, 24);
#pragma unroll 1
      for (int t = 0; t < 3; ++t) {
        const int r = t * 128 + q * 32 + lane, ii = r / 49, p = r - ii * 49, oy = p / 7, ox = p - oy * 7, b = b0 + ii;
        const bool ok = ii < kGF && oy < 5 && ox < 5 && b < a.B;
#pragma unroll
        for (int c0 = 0; c0 < C; c0 += 32) {
          float v[32];
          tc::tmem_ld32(t_c2 + t * C + c0 + ((uint32_t)(q * 32) << 16), v);
          if (ok) {
#pragma unroll
            for (int j8 = 0; j8 < 4; ++j8) {
              float f[8];
#pragma unroll
              for (int j = 0; j < 8; ++j) f[j] = fmaxf(v[j8 * 8 + j] + s_b2[c0 + j8 * 8 + j], 0.f);
              *reinterpret_cast<uint4*>(hout + (int64_t)b * a.h_ld + (oy * 5 + ox) * C + c0 + j8 * 8) =
                  tc::pack_bf16x8(f);
            }
          }
        }
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&t2_empty);
      if (i == 3 && warp == kPW + 4 && lane == 0) enc_stamp_any(a.dbg, 25);
    }
  } else {
    // ---- M: the MMAs (whole warp, one elected lane issues) --------------------------------------------
    // conv1 of group i + 1 is issued ahead of conv2 of group i when its operand is already built, so the
    // conv1 epilogue of i + 1 (into the other y1 buffer) overlaps conv2 of i on the tensor core
    const uint32_t id_c = tc::idesc_bf16(128, C);
    const uint32_t a0 = tc::smem_u32(sm + L::a1), w0 = tc::smem_u32(sm + L::w), w2 = w0 + C * 128;
    auto conv1 = [&](int i) {
      tc::mbar_wait(&a1_full, i & 1);
      if (i >= 1) tc::mbar_wait(&t1_empty, (i - 1) & 1);
      tc::fence_after_sync();
#pragma unroll
      for (int t = 0; t < 3; ++t)
#pragma unroll
        for (int k = 0; k < 2; ++k)
          tc::mma_bf16_e(t_c1 + t * C, sdesc_sw(a0 + t * 128 * 64 + 32 * k, 64), tc::sdesc_k128(w0 + 32 * k), id_c, k);
      tc::mma_commit_e(&a1_empty);
      tc::mma_commit_e(&t1_full);
    };
    if (nloc > 0) {
      tc::mbar_wait(&wbar, 0);
      conv1(0);
    }
    for (int i = 0; i < nloc; ++i) {
      tc::mbar_wait(&y1_full[i & 1], (i >> 1) & 1);
      if (i == 3 && lane == 0) enc_stamp_any(a.dbg, 26);
      if (i >= 1) tc::mbar_wait(&t2_empty, (i - 1) & 1);
      if (i == 3 && lane == 0) enc_stamp_any(a.dbg, 27);
      tc::fence_after_sync();
      // (y1_full(i) implies t1_empty(i): E1 arrives both; the producers are rarely behind by more than
      // the tensor core's conv2 time, so waiting for group i + 1's im2col here costs less than letting
      // its conv1 queue behind conv2 of group i)
      if (i + 1 < nloc) conv1(i + 1);
      if (i == 3 && lane == 0) enc_stamp_any(a.dbg, 28);
      // conv2 as nine row-shifted GEMMs over the full 7x7 grid (see k_enc_fwd_tc)
      const uint32_t y0 = tc::smem_u32(sm + L::y1 + (i & 1) * L::y1sz);
      for (int t = 0; t < 3; ++t)
        for (int tap = 0; tap < 9; ++tap) {
          const int shift = (tap / 3) * 7 + tap % 3;
          const int kb = (tap * C) / 64, koff = (tap * C) % 64;
#pragma unroll
          for (int k = 0; k < C / 16; ++k)
            tc::mma_bf16_e(t_c2 + t * C, sdesc_sw(y0 + (t * 128 + shift) * C * 2 + 32 * k, C * 2),
                           tc::sdesc_k128(w2 + kb * C * 128 + (koff + 16 * k) * 2), id_c, (tap | k) != 0);
        }
      tc::mma_commit_e(&y1_empty[i & 1]);
      tc::mma_commit_e(&t2_full);
      if (i == 3 && lane == 0) enc_stamp_any(a.dbg, 29);
    }
  }
  if (tid == 32 && nloc == 0) tc::mbar_wait(&wbar, 0);  // never exit with the bulk copy in flight
  tc::fence_before_sync();
  __syncthreads();
  enc_stamp(a.dbg, 15);
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// ---- backward --------------------------------------------------------------------------------
// element offset of (row r, 8-channel chunk ch) in the backward's y1 rows: the chunk index is XORed
// with row bits so that 32 lanes reading one chunk of 32 consecutive rows (the dX epilogue's ReLU'
// mask) hit distinct bank groups; 8 lanes reading the 8 chunks of one row (the dW2 gathers) still do
template <int C>
__device__ __forceinline__ int y1x(int r, int ch) {
  return r * C + ((C == 64 ? (ch ^ (r & 7)) : (ch ^ ((r >> 1) & 3))) << 3);
}
template <int C>
struct BwdL {
  static constexpr int nst = C == 32 ? 4 : 2;  // ring stages of 16 KB (one K block of an operand tile)
  static constexpr uint32_t w = 0;
  static constexpr uint32_t d2s = (((9 * C + 63) / 64) * C * 128 + 1023) & ~1023u;
  static constexpr uint32_t a1s = d2s + 2 * 8192;
  static constexpr uint32_t ring = a1s + 4 * 8192;
  static constexpr uint32_t d2p = ring + nst * 16384;  // D2 on zero-padded 9x9 grids, K-major rows
  static constexpr uint32_t y1s = d2p + ((288u * C * 2 + 1023) & ~1023u);
  static constexpr uint32_t xs = y1s + ((kGB * 49 * C * 2 + 1023) & ~1023u);
  static constexpr uint32_t total = xs + kGB * 768;
};
__host__ __device__ constexpr int part_rows(int C) { return 9 * C + 1 + 28; }  // dW2 (+ db2), dW1 (+ db1)

// Backward, one group of kGB = 4 images per CTA iteration.  Roles: warps 0-7 build operand tiles and
// run the dX epilogue; warp 8 issues every MMA (warp-uniform, elected lane).
//   conv2 dX as nine row-shifted GEMMs (no operand build): D2 of image i sits on a zero-padded 9x9 grid
//     whose rows are i * 63 + Y * 9 + X (consecutive images share their two zero pad rows), so output
//     (y, x) of the 7 x 9 grid, row o = i * 63 + y * 9 + x, reads D2pad row o + (2 - ki) * 9 + (2 - kj)
//     for tap (ki, kj): tap t's A operand is the padded tile itself started that many rows later;
//     B = W2 as [c][(t, o)]; positions x >= 7 are computed and dropped.  2 row tiles (252 rows).
//   conv2 dW / conv1 dW: operand tiles built into a ring of 16 KB stages (one K block each) while the
//     dX MMAs run; the dW accumulators stay in TMEM across the CTA's groups.
template <int C>
__global__ void __launch_bounds__(kThr + 32, 1) k_enc_bwd_tc(const __grid_constant__ EncBwdArgs a, int dbg) {
  using L = BwdL<C>;
  constexpr int nt2 = (9 * C + 1 + 127) / 128, cch = C / 8, NS = L::nst;
  constexpr uint32_t kCols = C == 32 ? 256u : 512u;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t wbar, bar_dx, bar_grp, d2_full, empty[NS], full[NS];
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, q = warp & 3, hh = warp >> 2;
  const int ngroups = (a.B + kGB - 1) / kGB;
  enc_stamp(dbg, 0);

  if (warp == 0) tc::tmem_alloc(&tmem_slot, kCols);
  if (tid == 32) {
    tc::mbar_init(&wbar, 1);
    tc::mbar_init(&bar_dx, 1);
    tc::mbar_init(&bar_grp, 1);
    tc::mbar_init(&d2_full, kThr / 32);
    for (int i = 0; i < NS; ++i) {
      tc::mbar_init(&empty[i], 1);
      tc::mbar_init(&full[i], kThr / 32);
    }
    tc::fence_mbar_init();
  }
  // The zero pads of the dX operand grids (rows i * 63 + Y * 9 + X outside the 5 x 5 interior, and
  // rows 252 .. 287) are never written per group: zeroed once here
  for (int e = tid; e < 288 * cch; e += kThr + 32) {
    const int R = e / cch, ch = e - R * cch, rem = R % 63, Y = rem / 9, X = rem - Y * 9;
    if (R >= kGB * 63 || Y < 2 || Y >= 7 || X < 2 || X >= 7)
      *reinterpret_cast<uint4*>(sm + L::d2p + y1_off<C>(R, ch)) = make_uint4(0, 0, 0, 0);
  }
  // dA1 rows 196 .. 255 (the K tail of conv1 dW) and, for C = 32, the unused half of every 128-byte
  // row stay zero: written once here, never by the per-group epilogue
  for (int e = tid; e < 256 * 8; e += kThr + 32) {
    const int r1 = e >> 3, ch = e & 7;
    if (r1 >= kGB * 49 || ch >= cch)
      *reinterpret_cast<uint4*>(sm + L::a1s + (r1 >> 6) * 8192 + sw(r1 & 63, ch)) = make_uint4(0, 0, 0, 0);
  }
  tc::fence_async_smem();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  grid_wait();
  grid_trigger();
  if (tid == 0) {
    tc::mbar_expect_tx(&wbar, bwd_wbytes(C));
    tc::bulk_load_1d(sm + L::w, a.wtiles + bwd_woff(C), bwd_wbytes(C), &wbar);
  }
  const uint32_t tmem = tmem_slot;
  const uint32_t t_dx = tmem, t_w2 = tmem + 2 * C, t_w1 = t_w2 + nt2 * C;
  const uint32_t id_k = tc::idesc_bf16(128, C), id_mn = tc::idesc_bf16_major(128, C, 1, 1);
  bf16_t* y1s = reinterpret_cast<bf16_t*>(sm + L::y1s);
  uint8_t* xs = sm + L::xs;
  int it = 0, gi = 0;
  enc_stamp(dbg, 1);

  if (warp == kThr / 32) {
    // ---- MMA warp ------------------------------------------------------------------------------------
    int mit = 0, mgi = 0;
    const uint32_t d2p0 = tc::smem_u32(sm + L::d2p), w0 = tc::smem_u32(sm + L::w);
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++mgi) {
      const bool first = mgi == 0;
      auto take = [&]() {
        const int st = mit % NS;
        tc::mbar_wait(&full[st], (mit / NS) & 1);
        tc::fence_after_sync();
        return tc::smem_u32(sm + L::ring + st * 16384);
      };
      tc::mbar_wait(&d2_full, mgi & 1);
      if (first) tc::mbar_wait(&wbar, 0);
      tc::fence_after_sync();
      for (int t = 0; t < 2; ++t)
        for (int tap = 0; tap < 9; ++tap) {
          const int shift = (2 - tap / 3) * 9 + (2 - tap % 3);
          const int kb = (tap * C) / 64, koff = (tap * C) % 64;
#pragma unroll
          for (int k = 0; k < C / 16; ++k)
            tc::mma_bf16_e(t_dx + t * C, sdesc_sw(d2p0 + (t * 128 + shift) * C * 2 + 32 * k, C * 2),
                           tc::sdesc_k128(w0 + kb * C * 128 + (koff + 16 * k) * 2), id_k, (tap | k) != 0);
        }
      tc::mma_commit_e(&bar_dx);
      for (int mt = 0; mt < nt2; ++mt)
        for (int kb = 0; kb < 2; ++kb, ++mit) {
          const uint32_t a0 = take(), b0s = tc::smem_u32(sm + L::d2s + kb * 8192);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            tc::mma_bf16_e(t_w2 + mt * C, tc::sdesc_sw128(a0 + 2048 * k, 8192, 1024),
                           tc::sdesc_sw128(b0s + 2048 * k, 8192, 1024), id_mn, !(first && kb == 0 && k == 0));
          tc::mma_commit_e(&empty[mit % NS]);
        }
      for (int s4 = 0; s4 < 4; ++s4, ++mit) {
        const uint32_t a0 = take(), b0s = tc::smem_u32(sm + L::a1s + s4 * 8192);
#pragma unroll
        for (int k = 0; k < 4; ++k)
          tc::mma_bf16_e(t_w1, tc::sdesc_sw128(a0 + 2048 * k, 8192, 1024), tc::sdesc_sw128(b0s + 2048 * k, 8192, 1024),
                         id_mn, !(first && s4 == 0 && k == 0));
        tc::mma_commit_e(&empty[mit % NS]);
        if (s4 == 3) tc::mma_commit_e(&bar_grp);
      }
    }
    if (mgi == 0) tc::mbar_wait(&wbar, 0);  // never exit with the bulk copy in flight
  } else {
    // ---- builders ------------------------------------------------------------------------------------
    auto stage_acquire = [&](int& st) -> uint8_t* {
      st = it % NS;
      if (it >= NS) tc::mbar_wait(&empty[st], ((it / NS) - 1) & 1);
      return sm + L::ring + st * 16384;
    };
    auto built = [&](int st) {
      tc::fence_async_smem();
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&full[st]);
    };
    // Global loads of a group (D2 dense MN-major rows r2 = img * 25 + p for dW2, D2 on the padded
    // grids for dX, y1 rows, the u8 images) go to registers; group g + 1's are issued as soon as
    // group g's are stored, so their latency hides behind group g's operand builds.
    constexpr int n_d2 = 128 * 8 / kThr, n_y1 = (kGB * 49 * cch + kThr - 1) / kThr;
    uint4 ud[n_d2], uy[n_y1], ux;
    auto load_group = [&](int g) {
      const int b0 = g * kGB;
      const bool gv = g < ngroups;
#pragma unroll
      for (int k = 0; k < n_d2; ++k) {
        const int e = tid + k * kThr, r2 = e >> 3, ch = e & 7, i = r2 / 25, p = r2 - i * 25, b = b0 + i;
        ud[k] = make_uint4(0, 0, 0, 0);
        if (gv && r2 < kGB * 25 && b < a.B && ch < cch)
          ud[k] = *reinterpret_cast<const uint4*>(a.dA2_hwc + (int64_t)b * a.dA2_ld + p * C + ch * 8);
      }
#pragma unroll
      for (int k = 0; k < n_y1; ++k) {
        const int e = tid + k * kThr, r1 = e / cch, ch = e - r1 * cch, i = r1 / 49, p = r1 - i * 49, b = b0 + i;
        uy[k] = make_uint4(0, 0, 0, 0);
        if (gv && e < kGB * 49 * cch && b < a.B)
          uy[k] = *reinterpret_cast<const uint4*>(a.y1_hwc + ((int64_t)b * 49 + p) * C + ch * 8);
      }
      ux = make_uint4(0, 0, 0, 0);
      if (gv && tid < kGB * 48 && b0 + tid / 48 < a.B)  // 16-byte chunks of the images
        ux = *reinterpret_cast<const uint4*>(a.img + (int64_t)(b0 + tid / 48) * 768 + (tid % 48) * 16);
    };
    // loop-invariant operand-build geometry of this thread (its 16-byte chunk ch of every 8-row
    // item is fixed: e = tid + n * kThr with kThr % 8 == 0)
    const int bch = tid & 7, brr = tid >> 3;  // chunk, first K row (the second is brr + 32)
    // conv1 dW operand: element u of the thread's chunk is K row m = 8 bch + u = (ci, ki, kj) of the
    // im2col; its byte offset in an image (>= 0), or -2 for the ones row (m = 27), -1 for zero
    int xoff[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int m = bch * 8 + u, ci = m / 9, t = m - ci * 9, ki = t / 3, kj = t - ki * 3;
      xoff[u] = (bch < 4 && m < 27) ? ci * 256 + ki * 16 + kj : (m == 27 ? -2 : -1);
    }
    if (blockIdx.x < ngroups) load_group(blockIdx.x);
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x, ++gi) {
      const int b0 = g * kGB;
      {
#pragma unroll
        for (int k = 0; k < n_d2; ++k) {
          const int e = tid + k * kThr, r2 = e >> 3, ch = e & 7;
          *reinterpret_cast<uint4*>(sm + L::d2s + (r2 >> 6) * 8192 + sw(r2 & 63, ch)) = ud[k];
          // the same D2 value at its place (i, y + 2, x + 2) on the zero-padded grids of the dX MMAs
          // (the pad rows were zeroed once at entry; invalid images store zeros here)
          if (r2 < kGB * 25 && ch < cch) {
            const int i = r2 / 25, p = r2 - i * 25, y = p / 5, x = p - y * 5;
            *reinterpret_cast<uint4*>(sm + L::d2p + y1_off<C>(i * 63 + (y + 2) * 9 + x + 2, ch)) = ud[k];
          }
        }
#pragma unroll
        for (int k = 0; k < n_y1; ++k) {
          const int e = tid + k * kThr, r1 = e / cch, ch = e - r1 * cch;
          if (e < kGB * 49 * cch) *reinterpret_cast<uint4*>(y1s + y1x<C>(r1, ch)) = uy[k];
        }
        if (tid < kGB * 48) *reinterpret_cast<uint4*>(xs + tid * 16) = ux;
      }
      // d2p (and d2s) -> the tensor core; also orders this group after the previous group's dX
      // epilogue (TMEM reads) for the MMA warp
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::named_bar(1, kThr);
      if (lane == 0) tc::mbar_arrive(&d2_full);
      load_group(g + gridDim.x);  // in flight during this group's builds
      enc_stamp(dbg && gi == 0, 2);
      // ---- conv2 dW (+ db2 via the ones row), accumulated across groups: one row tile x one K block
      //      per stage, built while the dX MMAs run.  Item (j, h) of a stage: A row m = 128 mt + 64 j +
      //      8 bch .. +7 (tap t, channels c0 ..), K row r2 = 64 kb + brr + 32 h (image i, output p) ->
      //      y1 row i * 49 + (oy + ki) * 7 + ox + kj ------------------------------------------------------
      int rbase[2][2];  // [kb][h]: y1 row of output r2 at tap (0, 0), or -1 past the group
#pragma unroll
      for (int kb = 0; kb < 2; ++kb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r2 = kb * 64 + brr + 32 * h, i = r2 / 25, p = r2 - i * 25, oy = p / 5, ox = p - oy * 5;
          rbase[kb][h] = (r2 < kGB * 25 && b0 + i < a.B) ? i * 49 + oy * 7 + ox : -1;
        }
      for (int mt = 0; mt < nt2; ++mt) {
        int toff[2], tcc[2];  // [j]: tap offset in y1 rows (-1: ones row, -2: zero), channel chunk
#pragma unroll
        for (int jj = 0; jj < 2; ++jj) {
          const int m0 = mt * 128 + jj * 64 + bch * 8, t = m0 / C, c0 = m0 - t * C;
          toff[jj] = t < 9 ? (t / 3) * 7 + t % 3 : (m0 == 9 * C ? -1 : -2);
          tcc[jj] = c0 >> 3;
        }
#pragma unroll
        for (int kb = 0; kb < 2; ++kb, ++it) {
          int st;
          uint8_t* A = stage_acquire(st);
          uint4 u[4];
#pragma unroll
          for (int n = 0; n < 4; ++n) {  // n = 2 j + h
            const int jj = n >> 1, h = n & 1, rb = rbase[kb][h];
            u[n] = make_uint4(0, 0, 0, 0);
            if (rb >= 0) {
              if (toff[jj] >= 0)
                u[n] = *reinterpret_cast<const uint4*>(y1s + y1x<C>(rb + toff[jj], tcc[jj]));
              else if (toff[jj] == -1)
                u[n].x = 0x3F80u;  // bf16 1.0 in element 0
            }
          }
#pragma unroll
          for (int n = 0; n < 4; ++n)
            *reinterpret_cast<uint4*>(A + (n >> 1) * 8192 + sw(brr + 32 * (n & 1), bch)) = u[n];
          built(st);
        }
      }
      enc_stamp(dbg && gi == 0, 4);
      // ---- dX epilogue: dA1 = dy1 * (y1 > 0) -> smem (MN-major rows r1); warp (q, hh) -> tile hh -----
      tc::mbar_wait(&bar_dx, gi & 1);
      tc::fence_after_sync();
      enc_stamp(dbg && gi == 0, 5);
      {
        const int o = hh * 128 + q * 32 + lane, i = o / 63, rem = o - i * 63, y = rem / 9, x = rem - y * 9;
        const bool ov = i < kGB && x < 7;
        const int r1 = i * 49 + y * 7 + x;
#pragma unroll
        for (int c0 = 0; c0 < C; c0 += 32) {
          float v[32];
          tc::tmem_ld32(t_dx + hh * C + c0 + ((uint32_t)(q * 32) << 16), v);
          if (ov) {
#pragma unroll
            for (int j8 = 0; j8 < 4; ++j8) {
              float f[8];
              const uint4 yv = *reinterpret_cast<const uint4*>(y1s + y1x<C>(r1, (c0 >> 3) + j8));
              const __nv_bfloat162* yp = reinterpret_cast<const __nv_bfloat162*>(&yv);
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                const float2 yf = __bfloat1622float2(yp[jj]);
                f[2 * jj] = yf.x > 0.f ? v[j8 * 8 + 2 * jj] : 0.f;
                f[2 * jj + 1] = yf.y > 0.f ? v[j8 * 8 + 2 * jj + 1] : 0.f;
              }
              const int ch = (c0 >> 3) + j8;
              *reinterpret_cast<uint4*>(sm + L::a1s + (r1 >> 6) * 8192 + sw(r1 & 63, ch)) = tc::pack_bf16x8(f);
            }
          }
        }
      }
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::named_bar(1, kThr);
      enc_stamp(dbg && gi == 0, 6);
      // ---- conv1 dW (+ db1), accumulated across groups: 4 steps of one K block (64 rows r1) ---------
      for (int s4 = 0; s4 < 4; ++s4, ++it) {
        int st;
        uint8_t* A = stage_acquire(st);
        // items (j, h): A row m = 64 j + 8 bch + u (j = 1 and m >= 28 are zero), K row r1 = 64 s4 +
        // brr + 32 h (image i, output (y, x)) -> byte (ci, 2 y + ki, 2 x + kj) of image i
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int rr = brr + 32 * h, r1 = s4 * 64 + rr, i = r1 / 49, p = r1 - i * 49, y = p / 7, x = p - y * 7;
          const bool rv = bch < 4 && r1 < kGB * 49 && b0 + i < a.B;
          const uint8_t* xb = xs + i * 768 + 2 * y * 16 + 2 * x;
          float f[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) f[u] = !rv ? 0.f : (xoff[u] >= 0 ? (float)xb[xoff[u]] : (xoff[u] == -2 ? 1.f : 0.f));
          *reinterpret_cast<uint4*>(A + sw(rr, bch)) = tc::pack_bf16x8(f);
          *reinterpret_cast<uint4*>(A + 8192 + sw(rr, bch)) = make_uint4(0, 0, 0, 0);
        }
        built(st);
      }
      enc_stamp(dbg && gi == 0, 7);
      tc::mbar_wait(&bar_grp, gi & 1);  // every MMA of the group done: smem inputs may be reused
      tc::fence_after_sync();
      tc::named_bar(1, kThr);
      enc_stamp(dbg && gi == 0, 8);
    }
    // ---- per-CTA partials, row-major [row][o]: rows 0..9C = dW2 (t, c) (+ db2), then dW1 (ci, t) (+ db1)
    float* part = a.part + (int64_t)blockIdx.x * part_rows(C) * C;
    if (gi > 0) {
      for (int mt = hh; mt < nt2 + 1; mt += 2) {
        const bool w1 = mt == nt2;
        const int m = q * 32 + lane + (w1 ? 0 : mt * 128);
        const uint32_t base = (w1 ? t_w1 : t_w2 + mt * C) + ((uint32_t)(q * 32) << 16);
        const int prow = w1 ? (m < 28 ? 9 * C + 1 + m : -1) : (m <= 9 * C ? m : -1);
#pragma unroll
        for (int c0 = 0; c0 < C; c0 += 32) {
          float v[32];
          tc::tmem_ld32(base + c0, v);
          if (prow >= 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              reinterpret_cast<float4*>(part + (int64_t)prow * C + c0)[j] =
                  make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  enc_stamp(dbg, 9);
  if (warp == 0) tc::tmem_dealloc(tmem, kCols);
}

// gradients = sum of the CTA partials in a fixed order (4 threads per element, each a quarter of
// the CTAs, then the quarters in order), permuted into the master layouts.
__global__ void __launch_bounds__(256) k_reduce_enc(const float* __restrict__ part, int nchunk, int C,
                                                    float* __restrict__ gw2, float* __restrict__ gb2,
                                                    float* __restrict__ gw1, float* __restrict__ gb1) {
  grid_wait();
  grid_trigger();
  __shared__ float red[4][64];
  const int stride = part_rows(C) * C;
  const int i = blockIdx.x * 64 + (threadIdx.x & 63), sl = threadIdx.x >> 6;
  const int c0 = (nchunk * sl) / 4, c1 = (nchunk * (sl + 1)) / 4;
  float s = 0.f;
  if (i < stride)
    for (int c = c0; c < c1; ++c) s += __ldg(part + (int64_t)c * stride + i);
  red[sl][threadIdx.x & 63] = s;
  __syncthreads();
  if (sl != 0 || i >= stride) return;
  const int tt = threadIdx.x;
  s = ((red[0][tt] + red[1][tt]) + red[2][tt]) + red[3][tt];
  const int row = i / C, o = i - row * C;
  if (row < 9 * C) {
    const int t = row / C, c = row - t * C;
    gw2[(o * C + c) * 9 + t] = s;
  } else if (row == 9 * C) {
    gb2[o] = s;
  } else {
    const int m = row - (9 * C + 1);
    if (m < 27) gw1[o * 27 + m] = s * (1.0f / 255.0f);
    else gb1[o] = s;
  }
}

template <int C>
int launch_fwd_c(const EncFwdArgs& a, cudaStream_t s) {
  if (a.mode == 0 || a.factor == 1 || (a.factor == 8 && C == 32)) {  // the pipelined kernel
    const size_t smem = (a.mode == 1 && a.factor == 8 ? FwdW<C>::total_sq : FwdW<C>::total) + 1024;
    cudaFuncSetAttribute(k_enc_fwd_ws<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int total = ((a.B + kGF - 1) / kGF) * a.nsrc;
    const int cap = a.max_ctas > 0 && a.max_ctas < 148 ? a.max_ctas : 148;
    const int grid = total < cap ? total : cap;
    launch_pdl(k_enc_fwd_ws<C>, grid, dim3(kWsWarps * 32), smem, s, a);
    return (int)cudaGetLastError();
  }
  const size_t smem = FwdL<C>::total + 1024;
  cudaFuncSetAttribute(k_enc_fwd_tc<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int total = ((a.B + kGF - 1) / kGF) * a.nsrc;
  const int cap = a.max_ctas > 0 && a.max_ctas < 148 ? a.max_ctas : 148;
  const int grid = total < cap ? total : cap;
  launch_pdl(k_enc_fwd_tc<C>, grid, dim3(kThr), smem, s, a);
  return (int)cudaGetLastError();
}
template <int C>
int launch_bwd_c(const EncBwdArgs& a, int grid, int dbg, cudaStream_t s) {
  const size_t smem = BwdL<C>::total + 1024;
  cudaFuncSetAttribute(k_enc_bwd_tc<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  launch_pdl(k_enc_bwd_tc<C>, grid, dim3(kThr + 32), smem, s, a, dbg);
  return (int)cudaGetLastError();
}

}  // namespace

size_t conv_tiles_bytes(int C) { return bwd_woff(C) + bwd_wbytes(C); }

int launch_conv_tiles(const float* w1, const float* w2, int C, uint8_t* tiles, cudaStream_t s) {
  note_launch(s, "k_conv_tiles", 0, 0);
  launch_pdl(k_conv_tiles, dim3(64), dim3(256), 0, s, w1, w2, C, tiles);
  return (int)cudaGetLastError();
}

int launch_enc_fwd_tc(const EncFwdArgs& a, cudaStream_t s) {
  if (a.B == 0) return 0;
  if ((a.C != 32 && a.C != 64) || a.H != 16 || a.c_in != 3 || !a.wtiles) return (int)cudaErrorInvalidValue;
  if (a.mode == 1 && a.factor != 8 && a.factor != 1) return (int)cudaErrorInvalidValue;
  {
    const double img = (double)a.B * a.nsrc, C = a.C;
    const double flops = 2.0 * img * (49.0 * C * 27.0 + 25.0 * 9.0 * C * C);
    const double bytes = (a.mode == 1 && a.factor == 8) ? img * (3.0 * 128 * 128 + 2.0 * 25 * C) : img * (768.0 + 2.0 * 25 * C);
    const bool ws = a.mode == 0 || a.factor == 1 || (a.factor == 8 && a.C == 32);  // launch_fwd_c's choice
    note_launch(s, ws ? "k_enc_fwd_ws" : "k_enc_fwd_tc", flops, bytes);
  }
  static const bool dbg = getenv("SQUINT_ENC_DBG") != nullptr;
  EncFwdArgs b = a;
  b.dbg = dbg ? 1 : 0;
  return b.C == 32 ? launch_fwd_c<32>(b, s) : launch_fwd_c<64>(b, s);
}

size_t enc_bwd_tc_partial_floats(int C, int B) {
  const int ngroups = (B + kGB - 1) / kGB;
  return (size_t)(ngroups < 148 ? ngroups : 148) * part_rows(C) * C;
}

int launch_enc_bwd_tc(const EncBwdArgs& a, cudaStream_t s) {
  if (a.B == 0) return 0;
  if ((a.C != 32 && a.C != 64) || a.H != 16 || a.c_in != 3 || !a.wtiles) return (int)cudaErrorInvalidValue;
  const int ngroups = (a.B + kGB - 1) / kGB;
  const int cap = a.max_ctas > 0 && a.max_ctas < 148 ? a.max_ctas : 148;
  const int grid = ngroups < cap ? ngroups : cap;
  static const bool dbg = getenv("SQUINT_ENC_DBG") != nullptr;
  {
    const double C = a.C;
    note_launch(s, "k_enc_bwd_tc", 2.0 * a.B * (2.0 * 25.0 * 9.0 * C * C + 49.0 * 27.0 * C), 0);
  }
  int e = a.C == 32 ? launch_bwd_c<32>(a, grid, dbg ? 1 : 0, s) : launch_bwd_c<64>(a, grid, dbg ? 1 : 0, s);
  if (e) return e;
  const int stride = part_rows(a.C) * a.C;
  note_launch(s, "k_reduce_enc", 0, 0);
  launch_pdl(k_reduce_enc, dim3((stride + 63) / 64), dim3(256), 0, s, a.part, grid, a.C, a.gw2, a.gb2, a.gw1, a.gb1);
  return (int)cudaGetLastError();
}

}  // namespace sq

extern "C" __attribute__((visibility("default"))) int squint_debug_enc_stamps(unsigned long long* host) {
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(host, sq::g_enc_stamps, sizeof(unsigned long long) * 160 * 32);
}
