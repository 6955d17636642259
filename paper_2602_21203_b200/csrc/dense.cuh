// dense.cuh -- grouped dense-layer problems for the update's MLP phases.
//
// One launch runs up to kMaxProb independent problems (e.g. both critic heads, or the
// four projections of one update).  A problem is  out = epilogue(A @ B^T)  with
//   A [M, K] = concat of up to 3 row-major segments along K (a segment may gather its
//             rows through an int64 index list -- the replay gather of a3 is fused here),
//   B (n, k) = up to 2 segments stacked along K, each K-major (W[n][k], forward) or
//             N-major (W[k][n], the dX = dY W of backward),
// and the epilogues of the paper's layers: LayerNorm + ReLU / tanh, the
// tanh-Gaussian head (Q13-Q14) and their backward.
#pragma once
#include <stdint.h>

namespace sq {

enum Epi : int {
  EPI_STORE = 0,       // out = acc
  EPI_BIAS = 1,        // out = acc + bias
  EPI_LN_RELU = 2,     // out = relu(LN(acc + bias)); writes xh, rstd      (row-complete)
  EPI_LN_TANH = 3,     // out = tanh(LN(acc + bias)); writes xh, rstd      (row-complete)
  EPI_TG_FWD = 4,      // o = acc + bias = [mu | l]; a = tanh(mu + sigma eps), log pi   (row-complete)
  EPI_BWD_LN_RELU = 5, // acc = dL/dy, y = relu(n): out = dL/d(pre-LN), out2 = dL/dn (row-complete)
  EPI_BWD_LN_TANH = 6, // same with y = tanh(n)                                         (row-complete)
  EPI_RELU_MASK = 7,   // out = acc * (y > 0)
  EPI_TG_BWD = 8,      // acc = dL/da (A cols): out = dL/d[mu | l] (2A cols)             (row-complete)
};

inline bool epi_row_complete(int e) {
  return e == EPI_LN_RELU || e == EPI_LN_TANH || e == EPI_TG_FWD || e == EPI_BWD_LN_RELU ||
         e == EPI_BWD_LN_TANH || e == EPI_TG_BWD;
}

struct ASeg {
  const float* ptr;
  const int64_t* rows;  // NULL: row m; else row rows[m] (replay gather)
  int ld, width;
};
struct BSeg {
  const float* ptr;
  int ld, width;  // width along K
  int kmajor;     // 1: B(n,k) = ptr[n*ld + k]; 0: B(n,k) = ptr[k*ld + n]
};

struct DenseProb {
  int M, N, K;
  int nA, nB;
  ASeg A[3];
  BSeg B[2];
  int epi;
  const float* bias;
  const float* g;     // LN gain (fwd: applied; bwd: d xh = dn * g)
  const float* beta;  // LN bias
  float* out;         // [M, ldo]
  int ldo;
  float* out2;        // bwd LN: dL/dn [M, N]
  float* xh;          // LN cache [M, N]
  float* rstd;        // LN cache [M]
  const float* y;     // bwd: layer output [M, N] (act'); RELU_MASK: mask source [M, N]
  // tanh-Gaussian
  const float* eps;   // [M, A] (may be NULL => eps = 0)
  float* act;         // [M, A]
  float* logp;        // [M]
  const float* tg_o;  // bwd: cached [mu | l] [M, 2A]
  const float* dlogp_scale;  // bwd: device scalar s, dL/dlogpi = s (e.g. alpha+ / B)
  float dlogp_mult;
  float lo, hi, ln_eps;
  int tiles_n;        // tiles along N
  int tile0;          // first tile index of this problem in the launch
};

constexpr int kMaxProb = 8;
struct DenseBatch {
  int nprob;
  int ntiles;
  int emul;  // numerics experiment (SQUINT_EMUL): bit0 rounds activation operands to bf16, bit1 weights
  DenseProb p[kMaxProb];
};

// Weight-gradient problems: dW[n][k] = sum_m D[m][n] X[m][k]; db[n] = sum_m D[m][n];
// dg[n] = sum_m DN[m][n] xh[m][n]; dbeta[n] = sum_m DN[m][n].  Deterministic (no atomics).
struct DwProb {
  int M, N, K;
  const float* D;  // [M, N] grad w.r.t. the linear output
  int nA;
  ASeg A[3];       // layer input X [M, K]
  float* dW;       // [N, K]
  float* db;       // [N] or NULL
  const float* DN; // [M, N] grad w.r.t. LN output, or NULL (no LN)
  const float* xh; // [M, N]
  float* dg;
  float* dbeta;
  int tiles_k, tile0;
};
constexpr int kMaxDw = 8;
struct DwBatch {
  int nprob;
  int ntiles;
  int emul;
  DwProb p[kMaxDw];
};

// Launchers (dense_f32.cu).  Return cudaError_t as int.
int launch_dense_f32(const DenseBatch& b, int tn, cudaStream_t s);
int launch_dw_f32(const DwBatch& b, cudaStream_t s);
// Plan tiles for a batch (sets tiles_n / tile0 / ntiles); returns the TN template arg.
int plan_dense(DenseBatch& b);
void plan_dw(DwBatch& b);

constexpr int kDenseBM = 16;
constexpr int kDwBN = 32, kDwBK = 64;

}  // namespace sq
