// gemm.cuh -- grouped bf16 GEMM on tcgen05 tensor cores fed by TMA (gemm.cu).
//
// One launch runs up to kGemmMaxProb independent problems (both critic heads, target and
// online passes, ...).  Problem p computes, for its M x N output,
//     acc[m][n] = sum_s sum_k A_s(m, k) B_s(n, k)        (s = K segment, up to 3)
// with every operand a bf16 row-major matrix read by TMA in 64-wide boxes with the 128-byte
// swizzle.  An operand is either
//     K-major  (matrix rows = M or N, columns = K)  -- forward X W^T, dX's D, or
//     MN-major (matrix rows = K, columns = M or N)   -- W of dX = D W and both dW operands,
// so the weight and activation matrices are used as stored; no transposed copies exist.
// The fp32 accumulator lives in TMEM; the epilogue applies the layer's pointwise math
// (LayerNorm P:159/Q9 with ReLU or tanh, the tanh-Gaussian head Q13-Q14, their backward,
// the weight-gradient store with bias / LN-affine gradients) and writes bf16 activations
// for the next GEMM and fp32 results where a reduction kernel or the optimizer reads them.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "tmap.hpp"

namespace sq {

typedef __nv_bfloat16 bf16;

enum GEpi : int {
  GE_LN_RELU = 0,      // y = relu(LN(acc + b)) -> out (bf16); xh (bf16), rstd (fp32) cached
  GE_LN_TANH = 1,      // y = tanh(LN(acc + b))
  GE_BIAS_F32 = 2,     // outf = acc + b (fp32; logits)
  GE_TG_FWD = 3,       // o = acc + b = [mu | l] -> a = tanh(mu + sigma eps), log pi
  GE_BWD_LN_RELU = 4,  // acc = dL/dy of y = relu(g xh + beta): out = dL/d(pre-LN), part = col sums
  GE_BWD_LN_TANH = 5,  // same with tanh
  GE_RELU_MASK = 6,    // out = acc * (y > 0)
  GE_TG_BWD = 7,       // acc = dL/da (A cols) -> out = dL/d[mu | l] (2A cols)
  GE_DW = 8,           // outf[n][k] = acc (weight gradient); tile-column 0 adds bias/LN grads
};

struct GSeg {
  int amap, bmap;  // indices into GBatch::maps
  int a_mn, b_mn;  // 1: operand is MN-major (matrix rows run along K)
  int a_k, b_k;    // K coordinate of the segment start inside the A / B matrix
  int nkb;         // 64-wide K blocks in the segment
  int k;           // real K of the segment (algorithmic FLOP count)
};

struct GProb {
  int M, N;        // output rows (tile rows, <= A rows) / real output columns
  int a_m, b_n;    // M / N coordinate offsets inside the A / B matrices (MN-major: multiple of 8)
  int acc_col0;    // GE_TG_BWD: accumulator column of output column 0 (b_n alignment slack)
  int nseg;
  GSeg seg[3];
  int bn;          // output columns per tile (<= 512; row-complete epilogues: >= N)
  int tiles_n, tile0;
  int epi;
  const float* bias;
  const float* g;
  const float* beta;
  bf16* out;       // bf16 result, element (m, n) at out[m * ldo + n]
  int ldo;
  float* outf;     // fp32 result (GE_BIAS_F32, GE_DW)
  int ldf;
  bf16* xh;        // LN cache x_hat (bf16, ld = ldx); bwd: read
  int ldx;
  float* rstd;     // LN 1/sigma per row; bwd: read
  const bf16* y;   // GE_RELU_MASK: mask source (ld = ldy)
  int ldy;
  float* part;     // bwd LN: column partial sums [mtile][3][N] = (sum dx, sum dn xh, sum dn)
  int64_t part_cap;  // floats available at `part` (gemm_launch rejects a plan that would overrun it)
  // tanh-Gaussian (A = action dim)
  const float* eps;     // [M][A]
  float* act;           // [M][A] fp32 action (may be NULL)
  bf16* act_bf;         // bf16 action written into a column slot of a critic input (may be NULL)
  int ld_act_bf;
  float* logp;          // [M]
  float* tgo;           // fwd: [M][2A] cache of [mu | l] (may be NULL); bwd: read
  const float* dlogp_scale;  // bwd: device scalar, dL/dlog pi
  float lo, hi, ln_eps;
  // GE_DW extras (rows of the dW tile are output features n < M)
  float* db;
  float* dg;
  float* dbeta;
  const float* part_in;      // bwd-LN partials of this layer [part_tiles][3][M]
  int part_tiles;
  int bias_ones;             // else db[n] = sum_m D[m][n]: an extra N = 16 MMA of the D tile against
                             // a shared-memory tile of ones (tile column 0 only)
  int omap, xmap, ymap;      // epilogue tensor maps (set by gemm_launch): out, xh, y (64 x 32 boxes)
};

constexpr int kGemmMaxProb = 16;  // (a K-split weight-gradient launch: up to 4 copies of 4 problems)
// largest split-K cluster gemm_launch plans (k_gemm_sk): LayerNorm column partials of a split-K
// launch take kGemmMaxSplitK * mtiles * 3 * N floats
constexpr int kGemmMaxSplitK = 8;
constexpr int kGemmMaxMaps = 64;

struct GBatch {
  CUtensorMap maps[kGemmMaxMaps];
  GProb p[kGemmMaxProb];
  int nprob, ntiles, nmaps;
  int stage_bytes, nstages;
  int cs;  // cluster size: LayerNorm rows split over cs CTAs (statistics exchanged through DSMEM)
  int ks;  // split-K cluster size (k_gemm_sk; set by gemm_launch): bwd-LN column partials are
           // then written per 128 / ks rows, [mtiles * ks][3][N]
  int mcast;       // cluster CTAs share the A tile: each K block is loaded once and multicast
  int wide;        // GE_DW: K blocks per TMA box / stage (1: one box per 64-row K block)
  int xpre_off;    // LayerNorm backward: smem offset of the prefetched x_hat boxes (0: loaded after the main loop)
  int prefetch_b;  // 1: B operands may be loaded before griddepcontrol.wait (not written by the
                   // immediately preceding kernel); set through GemmBuilder::prefetch_b
  unsigned long long* dbg;  // optional per-CTA phase timestamps (globaltimer ns) [tile][16]
};

// Host-side builder: operands are registered as Mats; maps are created per use.
struct GemmBuilder {
  GBatch b;
  Mat segA[kGemmMaxProb][3], segB[kGemmMaxProb][3];  // operands, mapped at launch
  int err = 0;
  GemmBuilder(int prefetch_b = 0) {
    b.nprob = 0;
    b.nmaps = 0;
    b.ntiles = 0;
    b.prefetch_b = prefetch_b;
    b.ks = 1;
    b.cs = 1;
    b.wide = 1;
  }
  GProb& add(int M, int N, int epi);
  // K segment: A(m, k) from `A` (K-major if !a_mn) and B(n, k) from `Bm`.
  void seg(GProb& p, const Mat& A, int a_mn, int a_k, const Mat& Bm, int b_mn, int b_k, int K);
};

// Plans tiles/smem, creates tensor maps, launches.  Returns cudaError_t (or -1 on a
// planning/map error).
int gemm_launch(GemmBuilder& gb, cudaStream_t s);

// Enable programmatic dependent launch for subsequent gemm launches (default on).
void gemm_set_pdl(int on);
// Debug: when env SQUINT_GEMM_DBG=k is set, the k-th gemm launch (0-based, per process)
// records per-CTA phase timestamps, read back with gemm_debug_times.
int gemm_debug_times(unsigned long long* host, int max_entries);

}  // namespace sq
