// encoder.cuh -- launch interfaces for the image kernels: squint insert (a1), replay
// gather + random shift + conv encoder forward (a3-a5), encoder backward (a10), and the
// fused squint + encoder of rollout inference (a16).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace sq {

typedef __nv_bfloat16 bf16_t;

// Row gather into a bf16 matrix: dst[b * ld + col + j] = src[row(b) * width + j], j < width,
// row(b) = idx[b] (replay gather, a3) or b (use_idx = 0).
struct GatherJob {
  const float* src;
  int width;
  __nv_bfloat16* dst;
  int ld, col, use_idx;
};

struct EncFwdArgs {
  // source mode 0: replay gather + shift (update); mode 1: raw frames + squint (act)
  int mode;
  const uint8_t* src[2];   // mode 0: ring obs / next_obs [cap, c, H, W]; mode 1: frames [n, c, fH, fW]
  const int64_t* idx;      // mode 0: [B]
  const uint8_t* shifts;   // mode 0: [B, 4]
  int factor;              // mode 1: squint factor (frame = H * factor)
  uint8_t* ring;           // mode 1, optional: write squinted frames to ring[slots[i]]
  const int64_t* slots;
  int B;                   // images per source
  int nsrc;                // mode 0: 2 (obs, next_obs); mode 1: 1
  const float* w1; const float* b1; const float* w2; const float* b2;
  float* h[2];             // [B, F] outputs per source
  float* y1;               // [B, C, P1] conv1 activations of source 0 (NULL: not stored)
  uint8_t* img0;           // [B, c, H, W] shifted images of source 0 (NULL: not stored)
  int C, c_in, H, pad;
  uint8_t* img1;           // tensor-core path: [B, c, H, W] shifted images of source 1 (debug dump,
                           // squint_set_option 5; NULL: not stored)
  // bf16 path: h written as bf16 in HWC flatten order hb[src][b * h_ld + pix * C + o]
  // (instead of fp32 CHW h), plus row gathers of the small replay fields per source.
  __nv_bfloat16* hb[2];
  int h_ld;
  __nv_bfloat16* y1b;      // tensor-core path: conv1 activations of source 0, bf16 HWC [B][49][C]
  GatherJob gj[2][4];
  int ngj[2];
  const uint8_t* wtiles;   // tensor-core path: conv weights as swizzled bf16 smem images (k_conv_tiles)
  int dbg;                 // phase timestamps (SQUINT_ENC_DBG; set by the launcher)
  int max_ctas;            // tensor-core path: grid cap (0: one CTA per job, at most one per SM)
  int emul;                // fp32 path, numerics measurement (squint_set_option 4 bit 3): conv weights
                           // and the conv1 activations rounded to bf16 as the tensor-core path stores them
};

struct EncBwdArgs {
  int B, C, c_in, H;
  const float* dA2;        // [B, F]  dL/d(conv2 pre-activation), CHW (fp32 path) ...
  const __nv_bfloat16* dA2_hwc;  // ... or bf16 HWC [B, P2 * C] (bf16 path; used when non-NULL)
  int dA2_ld;                    // row pitch of dA2_hwc (elements)
  const float* y1;         // [B, C, P1] fp32 CHW ...
  const __nv_bfloat16* y1_hwc;  // ... or bf16 HWC [B][P1][C] (used when non-NULL)
  const uint8_t* img;      // [B, c, H, W]
  const float* w2;         // conv2 weights [C, C, 3, 3]
  float* dA1;              // [B, C, P1] workspace
  float* part;             // partial weight grads [nchunk][C*C*9 + C + C*c*9 + C]
  int nchunk;
  float* gw1; float* gb1; float* gw2; float* gb2;  // final grads (CRITIC layout)
  const uint8_t* wtiles;   // tensor-core path: conv weights as swizzled bf16 smem images (k_conv_tiles)
  int max_ctas;            // tensor-core path: grid cap (0: one CTA per SM); fewer when the kernel
                           // runs beside other work on a graph branch
  int emul;                // fp32 path (squint_set_option 4 bit 3): W2, dA2 and dA1 rounded to bf16
};

int launch_enc_fwd(const EncFwdArgs& a, cudaStream_t s);
// tcgen05 implicit-GEMM encoder forward (encoder_tc.cu): bf16 outputs hb / y1b; C in {32, 64},
// 16x16x3 stored images, squint factor 8 in mode 1.
int launch_enc_fwd_tc(const EncFwdArgs& a, cudaStream_t s);
int launch_enc_bwd(const EncBwdArgs& a, cudaStream_t s);
// tcgen05 implicit-GEMM encoder backward (encoder_tc.cu): reads dA2_hwc, y1_hwc, img, w2; writes
// the conv weight/bias gradients through per-CTA partials (a.part, enc_bwd_tc_partial_floats)
// and a fixed-order reduction (deterministic).
int launch_enc_bwd_tc(const EncBwdArgs& a, cudaStream_t s);
size_t enc_bwd_tc_partial_floats(int C, int B);
// Conv weights (fp32 master, Q7 layouts) -> the bf16 128B-swizzled smem images the tensor-core
// encoder kernels bulk-copy: forward [W1 tile | W2 tiles], backward [W2^T tiles].
size_t conv_tiles_bytes(int C);
int launch_conv_tiles(const float* w1, const float* w2, int C, uint8_t* tiles, cudaStream_t s);
size_t enc_bwd_partial_floats(int C, int c_in, int nchunk);
int enc_bwd_nchunk(int B);

// f4 variants: HWC frames (hwc = 1) and/or colour jitter (jitter [n,3] = brightness, contrast,
// saturation per frame; c == 3) fused before the squint; one CTA per frame (c*h*w <= 200 KB)
int launch_insert_ex(const uint8_t* frames, int64_t n, int c, int h, int w, int factor, int hwc, const float* jitter,
                     const int64_t* slots, uint8_t* ring, cudaStream_t s, const int64_t* slots2 = nullptr,
                     uint8_t* ring2 = nullptr);
// ring2 / slots2 (optional): a second destination written with the same squinted frames
int launch_insert(const uint8_t* frames, int64_t n, int c, int h, int w, int factor, const int64_t* slots,
                  uint8_t* ring, cudaStream_t s, const int64_t* slots2 = nullptr, uint8_t* ring2 = nullptr);

}  // namespace sq
