// dense_tc.cuh -- problem description of the tcgen05 grouped dense kernel (dense_tc.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "dense.cuh"

namespace sq {

// One operand segment along K.  Element (r, k), r < rows of the operand, k < width:
//   kcontig: ptr[(gather ? gather[r] : r) * ld + k]      (row-major source, K contiguous)
//   else:    ptr[(gather ? gather[k] : k) * ld + r]      (source is [K][rows]: transposed read)
struct TcSeg {
  const float* ptr;
  const int64_t* gather;
  int ld, width, kcontig;
};
struct TcOp {
  int rows, nseg;
  TcSeg s[3];
};
struct TcProb {
  int M, N, K;
  TcOp A, B;  // out[m][n] = epilogue(sum_k A(m, k) B(n, k))
  int epi;
  const float* bias;
  const float* g;
  const float* beta;
  float* out;
  int ldo, out_col0;
  float* out2;
  float* xh;
  float* rstd;
  const float* y;
  const float* eps;
  float* act;
  float* logp;
  const float* tg_o;
  const float* dlogp_scale;
  float dlogp_mult, lo, hi, ln_eps;
  int bn, tiles_n, tile0;
};
constexpr int kMaxTc = 12;
struct TcBatch {
  int nprob, ntiles;
  TcProb p[kMaxTc];
};

void plan_tc(TcBatch& b);
int launch_tc(const TcBatch& b, cudaStream_t s);
int launch_dense_bf16(const DenseBatch& d, cudaStream_t s);
int launch_dw_bf16(const DwBatch& d, cudaStream_t s);

}  // namespace sq
