// encoder.cu -- image kernels of the update and of rollout inference (fp32 SIMT).
//
//  a1  squint: integer 8x8 block sums of u8 frames (16-byte vector loads, byte sums with
//      dp4a), round-half-to-even divide (Q1), scatter into the replay ring.
//  a3-a5  replay gather + random shift (replicate pad, Q5) + conv 3x3/s2 + ReLU + conv 3x3/s1
//      + ReLU (Q7), for obs and next_obs in one launch (both encoded with psi).
//  a10 encoder backward: conv2 dX (masked by ReLU'), conv2/conv1 weight gradients as
//      fixed-order per-chunk partials + a fixed-order reduction (bitwise reproducible).
#include <cuda_runtime.h>

#include "common.cuh"
#include "encoder.cuh"

namespace sq {

namespace {

SQ_DEV float bfr(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }
SQ_DEV float bfr_if(bool on, float x) { return on ? bfr(x) : x; }

SQ_DEV uint32_t rhe_div(uint32_t s, uint32_t n) {
  uint32_t q = s / n, r = s - q * n;
  if (2 * r > n || (2 * r == n && (q & 1u))) ++q;
  return q;
}

// Byte sums of a 16-byte vector: bytes 0-7 and 8-15.
SQ_DEV void sum16(const uint4 v, uint32_t& lo, uint32_t& hi) {
  lo = __dp4a(v.x, 0x01010101u, __dp4a(v.y, 0x01010101u, lo));
  hi = __dp4a(v.z, 0x01010101u, __dp4a(v.w, 0x01010101u, hi));
}

// ---- a1 standalone insert ---------------------------------------------------------
// factor 8, frame width a multiple of 16: one thread = 2 output pixels (one 16-byte
// column chunk over 8 rows).
__global__ void __launch_bounds__(256) k_insert_f8(const uint8_t* __restrict__ frames, int64_t n, int c, int h,
                                                   int w, const int64_t* __restrict__ slots,
                                                   uint8_t* __restrict__ ring, const int64_t* __restrict__ slots2,
                                                   uint8_t* __restrict__ ring2) {
  grid_wait();
  grid_trigger();
  const int ho = h / 8, wo = w / 8, chunks = w / 16;
  const int64_t items = n * c * ho * chunks;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int ch = (int)(it % chunks);
    int64_t t = it / chunks;
    const int oy = (int)(t % ho);
    t /= ho;
    const int cc = (int)(t % c);
    const int64_t f = t / c;
    const uint8_t* src = frames + ((f * c + cc) * (int64_t)h + oy * 8) * w + ch * 16;
    uint4 v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = __ldcs(reinterpret_cast<const uint4*>(src + (int64_t)r * w));
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int r = 0; r < 8; ++r) sum16(v[r], lo, hi);
    const uint32_t q0 = (lo + 31u + ((lo >> 6) & 1u)) >> 6;  // RHE(lo / 64)
    const uint32_t q1 = (hi + 31u + ((hi >> 6) & 1u)) >> 6;
    const uint16_t q = (uint16_t)(q0 | (q1 << 8));
    const int64_t off = (int64_t)cc * (ho * wo) + oy * wo + ch * 2;
    *reinterpret_cast<uint16_t*>(ring + slots[f] * c * (int64_t)(ho * wo) + off) = q;
    if (ring2) *reinterpret_cast<uint16_t*>(ring2 + slots2[f] * c * (int64_t)(ho * wo) + off) = q;
  }
}

// generic factor: one thread per output pixel
__global__ void k_insert_generic(const uint8_t* __restrict__ frames, int64_t n, int c, int h, int w, int f,
                                 const int64_t* __restrict__ slots, uint8_t* __restrict__ ring,
                                 const int64_t* __restrict__ slots2, uint8_t* __restrict__ ring2) {
  const int ho = h / f, wo = w / f;
  const int64_t items = n * c * ho * wo;
  for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < items;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int ox = (int)(it % wo);
    int64_t t = it / wo;
    const int oy = (int)(t % ho);
    t /= ho;
    const int cc = (int)(t % c);
    const int64_t fr = t / c;
    const uint8_t* src = frames + ((fr * c + cc) * (int64_t)h + oy * f) * w + ox * f;
    uint32_t s = 0;
    for (int a = 0; a < f; ++a)
      for (int b = 0; b < f; ++b) s += src[(int64_t)a * w + b];
    const uint8_t q = (uint8_t)rhe_div(s, (uint32_t)(f * f));
    ring[(slots[fr] * c + cc) * (int64_t)(ho * wo) + oy * wo + ox] = q;
    if (ring2) ring2[(slots2[fr] * c + cc) * (int64_t)(ho * wo) + oy * wo + ox] = q;
  }
}

// ---- a3-a5 / a16 encoder forward ----------------------------------------------------
__global__ void __launch_bounds__(256) k_enc_fwd(const __grid_constant__ EncFwdArgs a, int ipb) {
  extern __shared__ float sm[];
  const int C = a.C, ci = a.c_in, H = a.H, H1 = (H - 3) / 2 + 1, P1 = H1 * H1, H2 = H1 - 2, P2 = H2 * H2;
  const int HH = H * H;
  float* w1t = sm;                        // [9*ci][C+1]
  float* w2t = w1t + 9 * ci * (C + 1);    // [9*C][C+1]
  float* xs = w2t + 9 * C * (C + 1);      // [ipb][ci][HH]
  float* y1s = xs + ipb * ci * HH;        // [ipb][C][P1]
  const int tid = threadIdx.x;
  const int src_i = blockIdx.y;
  const int b0 = blockIdx.x * ipb;

  for (int e = tid; e < C * 9 * ci; e += 256) {  // global [o][c][kk] -> [c*9+kk][o]
    const int o = e / (9 * ci), r = e % (9 * ci);
    w1t[r * (C + 1) + o] = bfr_if(a.emul & 8, a.w1[e]);
  }
  for (int e = tid; e < C * 9 * C; e += 256) {
    const int o = e / (9 * C), r = e % (9 * C);
    w2t[r * (C + 1) + o] = bfr_if(a.emul & 8, a.w2[e]);
  }
  for (int jb = 0; jb < a.ngj[src_i]; ++jb) {
    const GatherJob& g = a.gj[src_i][jb];
    for (int e = tid; e < ipb * g.width; e += 256) {
      const int i = e / g.width, j = e - i * g.width, b = b0 + i;
      if (b < a.B) {
        const int64_t row = g.use_idx ? a.idx[b] : (int64_t)b;
        g.dst[(int64_t)b * g.ld + g.col + j] = __float2bfloat16_rn(g.src[row * g.width + j]);
      }
    }
  }
  const float inv255 = 1.0f / 255.0f;
  if (a.mode == 0) {
    const uint8_t* src = a.src[src_i];
    for (int e = tid; e < ipb * ci * HH; e += 256) {
      const int i = e / (ci * HH), r = e % (ci * HH), cc = r / HH, p = r % HH, y = p / H, x = p % H;
      const int b = b0 + i;
      float v = 0.f;
      if (b < a.B) {
        const int64_t row = a.idx[b];
        const int dx = a.shifts[b * 4 + 2 * src_i], dy = a.shifts[b * 4 + 2 * src_i + 1];
        const int sy = min(max(y + dy - a.pad, 0), H - 1), sx = min(max(x + dx - a.pad, 0), H - 1);
        const uint8_t u = src[row * (ci * HH) + cc * HH + sy * H + sx];
        if (src_i == 0 && a.img0) a.img0[(int64_t)b * ci * HH + r] = u;
        v = (float)u * inv255;
      }
      xs[e] = v;
    }
  } else {
    // squint: factor-f block sums of raw frames, RHE; optional ring write.
    const int f = a.factor, W = H * f;
    const uint8_t* frames = a.src[0];
    if (f == 8 && (W % 16) == 0) {
      const int chunks = W / 16;  // 2 output pixels per chunk
      for (int e = tid; e < ipb * ci * H * chunks; e += 256) {
        const int ch = e % chunks, t1 = e / chunks, oy = t1 % H, t2 = t1 / H, cc = t2 % ci, i = t2 / ci;
        const int b = b0 + i;
        uint32_t lo = 0, hi = 0;
        if (b < a.B) {
          const uint8_t* src = frames + (((int64_t)b * ci + cc) * W + oy * 8) * W + ch * 16;
          uint4 v[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) v[r] = __ldcs(reinterpret_cast<const uint4*>(src + (int64_t)r * W));
#pragma unroll
          for (int r = 0; r < 8; ++r) sum16(v[r], lo, hi);
        }
        const uint32_t q0 = (lo + 31u + ((lo >> 6) & 1u)) >> 6, q1 = (hi + 31u + ((hi >> 6) & 1u)) >> 6;
        xs[(i * ci + cc) * HH + oy * H + 2 * ch] = (float)q0 * inv255;
        xs[(i * ci + cc) * HH + oy * H + 2 * ch + 1] = (float)q1 * inv255;
        if (b < a.B && a.ring)
          *reinterpret_cast<uint16_t*>(a.ring + (a.slots[b] * ci + cc) * (int64_t)HH + oy * H + 2 * ch) =
              (uint16_t)(q0 | (q1 << 8));
      }
    } else {
      for (int e = tid; e < ipb * ci * HH; e += 256) {
        const int i = e / (ci * HH), r = e % (ci * HH), cc = r / HH, p = r % HH, oy = p / H, ox = p % H;
        const int b = b0 + i;
        uint32_t q = 0;
        if (b < a.B) {
          const uint8_t* src = frames + (((int64_t)b * ci + cc) * W + oy * f) * W + ox * f;
          uint32_t s = 0;
          for (int u = 0; u < f; ++u)
            for (int v = 0; v < f; ++v) s += src[(int64_t)u * W + v];
          q = rhe_div(s, (uint32_t)(f * f));
          if (a.ring) a.ring[(a.slots[b] * ci + cc) * (int64_t)HH + p] = (uint8_t)q;
        }
        xs[e] = (float)q * inv255;
      }
    }
  }
  __syncthreads();

  // conv1: 3x3 stride 2 valid + ReLU.  thread: o = tid % C, positions strided by 256 / C.
  const int o = tid % C, grp = tid / C, ngrp = 256 / C;
  for (int p = grp; p < ipb * P1; p += ngrp) {
    const int i = p / P1, pix = p % P1, y = pix / H1, x = pix % H1;
    float acc = a.b1[o];
    for (int cc = 0; cc < ci; ++cc) {
      const float* xi = xs + (i * ci + cc) * HH + (2 * y) * H + 2 * x;
#pragma unroll
      for (int ki = 0; ki < 3; ++ki)
#pragma unroll
        for (int kj = 0; kj < 3; ++kj) acc = fmaf(w1t[(cc * 9 + ki * 3 + kj) * (C + 1) + o], xi[ki * H + kj], acc);
    }
    const float v = bfr_if(a.emul & 8, fmaxf(acc, 0.f));
    y1s[(i * C + o) * P1 + pix] = v;
    const int b = b0 + i;
    if (src_i == 0 && a.y1 && b < a.B) a.y1[((int64_t)b * C + o) * P1 + pix] = v;
  }
  __syncthreads();
  // conv2: 3x3 stride 1 valid + ReLU -> h[b][o*P2 + pix] (CHW flatten)
  float* hout = a.h[src_i];
  for (int p = grp; p < ipb * P2; p += ngrp) {
    const int i = p / P2, pix = p % P2, y = pix / H2, x = pix % H2;
    const int b = b0 + i;
    float acc = a.b2[o];
    for (int cc = 0; cc < C; ++cc) {
      const float* yi = y1s + (i * C + cc) * P1 + y * H1 + x;
#pragma unroll
      for (int ki = 0; ki < 3; ++ki)
#pragma unroll
        for (int kj = 0; kj < 3; ++kj) acc = fmaf(w2t[(cc * 9 + ki * 3 + kj) * (C + 1) + o], yi[ki * H1 + kj], acc);
    }
    if (b < a.B) {
      if (a.hb[src_i])
        a.hb[src_i][(int64_t)b * a.h_ld + pix * C + o] = __float2bfloat16_rn(fmaxf(acc, 0.f));
      else
        hout[(int64_t)b * C * P2 + o * P2 + pix] = fmaxf(acc, 0.f);
    }
  }
}

// ---- a10 encoder backward -----------------------------------------------------------
// dA1[b][c][pix] = ReLU'(y1) * sum_{o,ki,kj} dA2[b][o][y-ki][x-kj] W2[o][c][ki][kj]
__global__ void __launch_bounds__(256) k_enc_bwd_dx(const __grid_constant__ EncBwdArgs a, int ipb) {
  extern __shared__ float sm[];
  const int C = a.C, H = a.H, H1 = (H - 3) / 2 + 1, P1 = H1 * H1, H2 = H1 - 2, P2 = H2 * H2;
  float* w2s = sm;               // [o][c][9]
  float* ds = w2s + C * C * 9;   // [ipb][C][P2]
  const int tid = threadIdx.x, b0 = blockIdx.x * ipb;
  for (int e = tid; e < C * C * 9; e += 256) w2s[e] = bfr_if(a.emul & 8, a.w2[e]);
  for (int e = tid; e < ipb * C * P2; e += 256) {
    const int i = e / (C * P2), b = b0 + i, r = e % (C * P2);
    float v = 0.f;
    if (b < a.B) {
      if (a.dA2_hwc) {
        const int o = r / P2, pix = r - o * P2;
        v = __bfloat162float(a.dA2_hwc[(int64_t)b * C * P2 + pix * C + o]);
      } else {
        v = a.dA2[(int64_t)b * C * P2 + r];
      }
    }
    ds[e] = bfr_if(a.emul & 8, v);
  }
  __syncthreads();
  const int c = tid % C, grp = tid / C, ngrp = 256 / C;
  for (int p = grp; p < ipb * P1; p += ngrp) {
    const int i = p / P1, pix = p % P1, y = pix / H1, x = pix % H1, b = b0 + i;
    if (b >= a.B) continue;
    float acc = 0.f;
    for (int o = 0; o < C; ++o) {
      const float* wo = w2s + (o * C + c) * 9;
      const float* d = ds + (i * C + o) * P2;
#pragma unroll
      for (int ki = 0; ki < 3; ++ki) {
        const int yy = y - ki;
        if (yy < 0 || yy >= H2) continue;
#pragma unroll
        for (int kj = 0; kj < 3; ++kj) {
          const int xx = x - kj;
          if (xx < 0 || xx >= H2) continue;
          acc = fmaf(d[yy * H2 + xx], wo[ki * 3 + kj], acc);
        }
      }
    }
    const int64_t gi = ((int64_t)b * C + c) * P1 + pix;
    const float yv = a.y1_hwc ? __bfloat162float(a.y1_hwc[((int64_t)b * P1 + pix) * C + c]) : a.y1[gi];
    a.dA1[gi] = yv > 0.f ? bfr_if(a.emul & 8, acc) : 0.f;
  }
}

// Partial weight gradient of a 3x3 conv over a chunk of images:
//   dW[o][c][ki][kj] = sum_b sum_pix D[b][o][pix] X[b][c][s*y+ki][s*x+kj],  db[o] = sum D.
// grid = (nchunk, O / OB); each thread owns up to 40 weights (fixed summation order).
template <bool kU8>
__global__ void __launch_bounds__(256) k_conv_dw(const float* __restrict__ D, const __nv_bfloat16* __restrict__ Dh,
                                                 const void* __restrict__ Xv, const __nv_bfloat16* __restrict__ Xh, int B,
                                                 int O, int Cin, int Hin, int Hout, int stride, int OB,
                                                 int nchunk, float* __restrict__ part, int emul_d) {
  extern __shared__ float sm[];
  const int Pout = Hout * Hout, HH = Hin * Hin;
  float* Ds = sm;               // [OB][Pout]
  float* Xs = Ds + OB * Pout;   // [Cin][HH]
  const int tid = threadIdx.x;
  const int chunk = blockIdx.x, o0 = blockIdx.y * OB;
  const int per = (B + nchunk - 1) / nchunk, bb0 = chunk * per, bb1 = min(B, bb0 + per);
  const int nw = OB * Cin * 9;
  constexpr int R = 40;
  float acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = 0.f;
  float sb = 0.f;
  for (int b = bb0; b < bb1; ++b) {
    for (int e = tid; e < OB * Pout; e += 256) {
      if (Dh) {
        const int ol = e / Pout, pix = e - ol * Pout;
        Ds[e] = __bfloat162float(Dh[(int64_t)b * O * Pout + pix * O + o0 + ol]);
      } else {
        Ds[e] = bfr_if(emul_d, D[((int64_t)b * O + o0) * Pout + e]);
      }
    }
    for (int e = tid; e < Cin * HH; e += 256) {
      if (kU8)
        Xs[e] = (float)(reinterpret_cast<const uint8_t*>(Xv)[(int64_t)b * Cin * HH + e]) * (1.0f / 255.0f);
      else if (Xh) {
        const int c = e / HH, p = e - c * HH;
        Xs[e] = __bfloat162float(Xh[((int64_t)b * HH + p) * Cin + c]);
      } else
        Xs[e] = reinterpret_cast<const float*>(Xv)[(int64_t)b * Cin * HH + e];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int w = tid + 256 * r;
      if (w >= nw) break;
      const int ol = w / (Cin * 9), c = (w / 9) % Cin, kk = w % 9, ki = kk / 3, kj = kk % 3;
      const float* d = Ds + ol * Pout;
      const float* x = Xs + c * HH + ki * Hin + kj;
      float s = 0.f;
      for (int y = 0; y < Hout; ++y)
        for (int xx = 0; xx < Hout; ++xx) s = fmaf(d[y * Hout + xx], x[stride * y * Hin + stride * xx], s);
      acc[r] += s;
    }
    if (tid < OB) {
      float s = 0.f;
      for (int p = 0; p < Pout; ++p) s += Ds[tid * Pout + p];
      sb += s;
    }
    __syncthreads();
  }
  const int stride_part = O * Cin * 9 + O;
  float* pp = part + (int64_t)chunk * stride_part;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int w = tid + 256 * r;
    if (w >= nw) break;
    pp[o0 * Cin * 9 + w] = acc[r];
  }
  if (tid < OB) pp[O * Cin * 9 + o0 + tid] = sb;
}

// out_w[i] = sum_chunk part[chunk][i] (i < nw), out_b[i] likewise for biases.
__global__ void k_reduce_part(const float* __restrict__ part, int nchunk, int nw, int nb, float* __restrict__ out_w,
                              float* __restrict__ out_b) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int stride = nw + nb;
  if (i >= stride) return;
  float s = 0.f;
  for (int c = 0; c < nchunk; ++c) s += part[(int64_t)c * stride + i];
  if (i < nw)
    out_w[i] = s;
  else
    out_b[i - nw] = s;
}

int fwd_ipb(int C) { return C <= 32 ? 4 : 2; }
size_t fwd_smem(int C, int ci, int H, int ipb) {
  const int H1 = (H - 3) / 2 + 1;
  return sizeof(float) * (size_t)(9 * ci * (C + 1) + 9 * C * (C + 1) + ipb * ci * H * H + ipb * C * H1 * H1);
}
int bwd_ipb(int C) { return C <= 32 ? 8 : 4; }
int ob_of(int O, int Cin) {  // output-channel block so a thread owns <= 40 weights
  int ob = O;
  while (ob > 1 && (ob * Cin * 9 + 255) / 256 > 40) ob /= 2;
  return ob;
}

}  // namespace

int enc_bwd_nchunk(int B) { return B < 128 ? B : 128; }
size_t enc_bwd_partial_floats(int C, int c_in, int nchunk) {
  return (size_t)nchunk * (C * C * 9 + C) + (size_t)nchunk * (C * c_in * 9 + C);
}

int launch_enc_fwd(const EncFwdArgs& a, cudaStream_t s) {
  if (a.B == 0) return 0;
  const int ipb = fwd_ipb(a.C);
  const size_t smem = fwd_smem(a.C, a.c_in, a.H, ipb);
  cudaFuncSetAttribute(k_enc_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((a.B + ipb - 1) / ipb, a.nsrc);
  note_launch(s, "k_enc_fwd", 0, 0); k_enc_fwd<<<grid, 256, smem, s>>>(a, ipb);
  return (int)cudaGetLastError();
}

int launch_enc_bwd(const EncBwdArgs& a, cudaStream_t s) {
  const int C = a.C, H1 = (a.H - 3) / 2 + 1, P1 = H1 * H1, H2 = H1 - 2, P2 = H2 * H2;
  {
    const int ipb = bwd_ipb(C);
    const size_t smem = sizeof(float) * (size_t)(C * C * 9 + ipb * C * P2);
    cudaFuncSetAttribute(k_enc_bwd_dx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    note_launch(s, "k_enc_bwd_dx", 0, 0); k_enc_bwd_dx<<<(a.B + ipb - 1) / ipb, 256, smem, s>>>(a, ipb);
  }
  float* part2 = a.part;
  float* part1 = a.part + (size_t)a.nchunk * (C * C * 9 + C);
  {
    const int ob = ob_of(C, C);
    const size_t smem = sizeof(float) * (size_t)(ob * P2 + C * P1);
    cudaFuncSetAttribute(k_conv_dw<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    note_launch(s, "k_conv_dw", 0, 0); k_conv_dw<false><<<dim3(a.nchunk, C / ob), 256, smem, s>>>(a.dA2, a.dA2_hwc, a.y1, a.y1_hwc, a.B, C, C, H1, H2, 1, ob, a.nchunk,
                                                                 part2, a.emul & 8);
  }
  {
    const int ob = ob_of(C, a.c_in);
    const size_t smem = sizeof(float) * (size_t)(ob * P1 + a.c_in * a.H * a.H);
    cudaFuncSetAttribute(k_conv_dw<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    note_launch(s, "k_conv_dw", 0, 0); k_conv_dw<true><<<dim3(a.nchunk, C / ob), 256, smem, s>>>(a.dA1, nullptr, a.img, nullptr, a.B, C, a.c_in, a.H, H1, 2, ob,
                                                               a.nchunk, part1, 0);
  }
  {
    const int n2 = C * C * 9 + C, n1 = C * a.c_in * 9 + C;
    note_launch(s, "k_reduce_part", 0, 0); k_reduce_part<<<(n2 + 255) / 256, 256, 0, s>>>(part2, a.nchunk, C * C * 9, C, a.gw2, a.gb2);
    note_launch(s, "k_reduce_part", 0, 0); k_reduce_part<<<(n1 + 255) / 256, 256, 0, s>>>(part1, a.nchunk, C * a.c_in * 9, C, a.gw1, a.gb1);
  }
  return (int)cudaGetLastError();
}

// ---- f4 insert variants: HWC frames and colour jitter fused before the squint ----------------
// One CTA per frame: the frame is staged once in shared memory (one HBM read), the jitter's
// frame statistic (mean grey level after the brightness step) is reduced from it, and each thread
// then squints whole output pixels (all channels at once: saturation mixes the channels).
// Jitter (reading R-jit): per frame (b, c, s) > 0, in this order,
//   x1 = u8(b x);  m = sum(grey(x1)) / (h w);  x2 = u8(c x1 + (1 - c) m);  x3 = u8(s x2 + (1 - s) grey(x2))
// with u8(v) = truncate(clamp(v, 0, 255)) and grey(x) = u8((0.2989 R + 0.587 G) + 0.114 B), every
// float32 operation rounded on its own (no contraction) so the integer decisions match the oracle.
// ALU form: bytes become exact floats by one PRMT into the 2^23 mantissa (no I2F), and u8() is a
// clamp plus one round-down add of 2^23 (the integer lands in the low mantissa bits: no F2I).
namespace {
constexpr float kGreyR = 0.2989f, kGreyG = 0.587f, kGreyB = 0.114f, kMagic = 8388608.f;
constexpr uint32_t kMagicBits = 0x4B000000u;
// byte k of w as an exact float
__device__ __forceinline__ float bytef(uint32_t w, int k) {
  return __fsub_rn(__uint_as_float(__byte_perm(w, kMagicBits, 0x7540u | (uint32_t)k)), kMagic);
}
// 2^23 + u8(v): the value is (result - 2^23), the integer is (bits - kMagicBits)
__device__ __forceinline__ float u8m(float v) { return __fadd_rd(fminf(fmaxf(v, 0.f), 255.f), kMagic); }
__device__ __forceinline__ float grey_m(float r, float g, float b) {
  return __fadd_rd(__fadd_rn(__fadd_rn(__fmul_rn(kGreyR, r), __fmul_rn(kGreyG, g)), __fmul_rn(kGreyB, b)), kMagic);
}
__device__ __forceinline__ uint32_t mbits(float m) { return __float_as_uint(m) - kMagicBits; }
__device__ __forceinline__ float mval(float m) { return __fsub_rn(m, kMagic); }
}  // namespace

template <bool HWC, bool JIT>
__global__ void __launch_bounds__(256) k_insert_ex(const uint8_t* __restrict__ frames, int c, int h, int w, int f,
                                                   const float* __restrict__ jitter,
                                                   const int64_t* __restrict__ slots, uint8_t* __restrict__ ring,
                                                   const int64_t* __restrict__ slots2, uint8_t* __restrict__ ring2) {
  extern __shared__ __align__(16) uint8_t sfr[];
  __shared__ uint32_t wsum[8];
  grid_wait();
  grid_trigger();
  const int fr = blockIdx.x, tid = threadIdx.x;
  const int hw = h * w;
  const int64_t fb = (int64_t)c * hw;
  const uint8_t* src = frames + fr * fb;
  if ((fb & 15) == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    for (int64_t i = tid; i < fb / 16; i += 256)
      reinterpret_cast<uint4*>(sfr)[i] = __ldcs(reinterpret_cast<const uint4*>(src) + i);
  } else {
    for (int64_t i = tid; i < fb; i += 256) sfr[i] = src[i];
  }
  __syncthreads();
  // byte offset of (channel ch, pixel p) in the staged frame
  auto off = [&](int ch, int p) -> int { return HWC ? p * 3 + ch : ch * hw + p; };
  float bf = 1.f, cf = 1.f, sf = 1.f, cm = 0.f;
  if constexpr (JIT) {
    // pass 1: x1 = u8(b x) written back in place; sum of grey(x1)
    bf = jitter[fr * 3 + 0], cf = jitter[fr * 3 + 1], sf = jitter[fr * 3 + 2];
    uint32_t gs = 0;
    if ((hw & 3) == 0) {
      uint32_t* s32 = reinterpret_cast<uint32_t*>(sfr);
      for (int g = tid; g < hw / 4; g += 256) {
        uint32_t wd[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) wd[k] = HWC ? s32[g * 3 + k] : s32[(k * hw) / 4 + g];
        uint32_t o[3] = {0u, 0u, 0u};
        float x1[4][3];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const int bi = HWC ? 3 * i + ch : 4 * ch + i;  // byte index within wd
            const float m = u8m(__fmul_rn(bf, bytef(wd[bi >> 2], bi & 3)));
            o[bi >> 2] |= mbits(m) << (8 * (bi & 3));
            x1[i][ch] = mval(m);
          }
#pragma unroll
        for (int i = 0; i < 4; ++i) gs += mbits(grey_m(x1[i][0], x1[i][1], x1[i][2]));
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          if (HWC) s32[g * 3 + k] = o[k];
          else s32[(k * hw) / 4 + g] = o[k];
        }
      }
    } else {
      for (int p = tid; p < hw; p += 256) {
        float x1[3];
#pragma unroll
        for (int ch = 0; ch < 3; ++ch) {
          const float m = u8m(__fmul_rn(bf, (float)sfr[off(ch, p)]));
          sfr[off(ch, p)] = (uint8_t)mbits(m);
          x1[ch] = mval(m);
        }
        gs += mbits(grey_m(x1[0], x1[1], x1[2]));
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) gs += __shfl_xor_sync(0xffffffffu, gs, o);
    if ((tid & 31) == 0) wsum[tid >> 5] = gs;
    __syncthreads();
    uint32_t t = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += wsum[i];
    // the integer sum is exact in fp32 up to 2^24; (1 - c) m is one rounded product
    cm = __fmul_rn(__fsub_rn(1.f, cf), __fdiv_rn((float)t, (float)hw));
  }
  const float oms = __fsub_rn(1.f, sf);
  // one pixel (channel values x[0..2], x1 when jittered) into the channel sums
  auto add_px = [&](const float* x, uint32_t* acc) {
    float x2[3];
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) x2[ch] = mval(u8m(__fadd_rn(__fmul_rn(cf, x[ch]), cm)));
    const float sg = __fmul_rn(oms, mval(grey_m(x2[0], x2[1], x2[2])));
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) acc[ch] += mbits(u8m(__fadd_rn(__fmul_rn(sf, x2[ch]), sg)));
  };
  const int ho = h / f, wo = w / f, npo = ho * wo;
  const bool vec8 = f == 8 && (!JIT || c == 3) && (HWC ? c == 3 : true);
  for (int o = tid; o < npo; o += 256) {
    const int oy = o / wo, ox = o - oy * wo;
    uint32_t acc[4] = {0u, 0u, 0u, 0u};
    if (vec8 && (JIT || HWC)) {
      // 8 rows x 8 pixels x 3 channels: 24 bytes per row in 8-byte loads
      for (int a = 0; a < 8; ++a) {
        const int p0 = (oy * 8 + a) * w + ox * 8;
        uint32_t wd[6];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const uint2 v = HWC ? reinterpret_cast<const uint2*>(sfr + p0 * 3)[k]
                              : *reinterpret_cast<const uint2*>(sfr + k * hw + p0);
          wd[2 * k] = v.x, wd[2 * k + 1] = v.y;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float x[3];
#pragma unroll
          for (int ch = 0; ch < 3; ++ch) {
            const int bi = HWC ? 3 * i + ch : 8 * ch + i;
            x[ch] = JIT ? bytef(wd[bi >> 2], bi & 3) : 0.f;
            if (!JIT) acc[ch] += (wd[bi >> 2] >> (8 * (bi & 3))) & 0xFFu;
          }
          if (JIT) add_px(x, acc);
        }
      }
    } else {
      for (int a = 0; a < f; ++a)
        for (int bb = 0; bb < f; ++bb) {
          const int p = (oy * f + a) * w + ox * f + bb;
          if constexpr (JIT) {
            float x[3];
#pragma unroll
            for (int ch = 0; ch < 3; ++ch) x[ch] = (float)sfr[off(ch, p)];
            add_px(x, acc);
          } else {
#pragma unroll
            for (int ch = 0; ch < 4; ++ch)
              if (ch < c) acc[ch] += sfr[HWC ? p * c + ch : ch * hw + p];
          }
        }
    }
#pragma unroll
    for (int ch = 0; ch < 4; ++ch)
      if (ch < c) {
        const uint8_t q = (uint8_t)rhe_div(acc[ch], (uint32_t)(f * f));
        ring[(slots[fr] * c + ch) * (int64_t)npo + o] = q;
        if (ring2) ring2[(slots2[fr] * c + ch) * (int64_t)npo + o] = q;
      }
  }
}

int launch_insert_ex(const uint8_t* frames, int64_t n, int c, int h, int w, int factor, int hwc, const float* jitter,
                     const int64_t* slots, uint8_t* ring, cudaStream_t s, const int64_t* slots2, uint8_t* ring2) {
  if (n == 0) return 0;
  const size_t smem = (size_t)c * h * w;
  if (c > 4 || (jitter && c != 3) || smem > 200 * 1024 || n > 0x7fffffff) return (int)cudaErrorInvalidValue;
  auto kern = hwc ? (jitter ? k_insert_ex<true, true> : k_insert_ex<true, false>)
                  : (jitter ? k_insert_ex<false, true> : k_insert_ex<false, false>);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  note_launch(s, "k_insert_ex", 0, (double)n * c * h * w + (ring2 ? 2.0 : 1.0) * n * c * (h / factor) * (w / factor));
  launch_pdl(kern, dim3((unsigned)n), dim3(256), smem, s, frames, c, h, w, factor, jitter, slots, ring, slots2, ring2);
  return (int)cudaGetLastError();
}

int launch_insert(const uint8_t* frames, int64_t n, int c, int h, int w, int factor, const int64_t* slots,
                  uint8_t* ring, cudaStream_t s, const int64_t* slots2, uint8_t* ring2) {
  if (n == 0) return 0;
  if (factor == 8 && (w % 16) == 0) {
    const int64_t items = n * c * (h / 8) * (w / 16);
    int64_t blocks = (items + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    note_launch(s, "k_insert_f8", 0, (double)n * c * h * w + (ring2 ? 2.0 : 1.0) * n * c * (h / 8) * (w / 8)); launch_pdl(k_insert_f8, dim3((unsigned)blocks), dim3(256), 0, s, frames, n, c, h, w, slots, ring, slots2, ring2);
  } else {
    const int64_t items = n * c * (h / factor) * (w / factor);
    int64_t blocks = (items + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    note_launch(s, "k_insert_generic", 0, (double)n * c * h * w + (ring2 ? 2.0 : 1.0) * n * c * (h / factor) * (w / factor)); k_insert_generic<<<(unsigned)blocks, 256, 0, s>>>(frames, n, c, h, w, factor, slots, ring, slots2, ring2);
  }
  return (int)cudaGetLastError();
}

}  // namespace sq
