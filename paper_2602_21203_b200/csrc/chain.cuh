// chain.cuh -- fused MLP chains on tcgen05 (chain.cu): a whole head / actor pass (2-3 layers)
// in one launch.
//
// A 4-CTA cluster owns one 128-row tile of one problem.  In every LayerNorm layer CTA j computes
// output columns [64 j, 64 j + 64) of the 256-wide hidden layer (row statistics exchanged
// through distributed shared memory, as in gemm.cu) and bulk-copies its bf16 64-column result
// into every cluster CTA's shared memory as K block j of the next layer's A operand; the next
// layer's weight slice is TMA-prefetched during the current layer.  The chain's first A comes
// from global memory by TMA; each layer's activation (and x_hat cache) is also stored to global
// memory by TMA for the weight-gradient GEMMs.  Last layers: logits (bias, fp32; 32 columns per
// CTA) or the tanh-Gaussian head (one CTA).  Backward chains use the same machinery with
// dX = dY W (W MN-major) and the LayerNorm-backward epilogue.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "gemm.cuh"
#include "tmap.hpp"

namespace sq {

struct CLayer {
  int epi;         // GE_LN_RELU, GE_LN_TANH, GE_BWD_LN_RELU, GE_BWD_LN_TANH, GE_BIAS_F32, GE_TG_FWD
  int N;           // real output columns of the whole row
  int K;           // real K
  int nkb;         // 64-wide K blocks
  int b_mn;        // weight operand MN-major (dX = dY W) or K-major (X W^T)
  int bmap;        // weight tensor map (K-major box {64, slice}; MN-major box {64, 64})
  int slice;       // output columns per CTA (64 hidden, 32 logits, 16 tanh-Gaussian)
  const float* bias;
  const float* g;
  const float* beta;
  int omap, xmap;  // bf16 output / x_hat tensor maps (64 x 32 boxes), -1: none
  int emap;        // LayerNorm layers feeding a next layer: the global copy of the output the
                   // cluster CTAs exchange through (omap, or a workspace scratch); -1: DSMEM copies
  float* rstd;     // fwd LN: written; bwd LN: read
  float* part;     // bwd LN: column partials [mtile][3][N] (may be NULL)
  float* outf;     // GE_BIAS_F32 output (fp32, ld = ldf)
  int ldf;
  // tanh-Gaussian head (GE_TG_FWD)
  const float* eps;
  float* act;
  bf16* act_bf;
  int ld_act_bf;
  float* logp;
  float* tgo;
  float lo, hi, ln_eps;
};

constexpr int kChainMaxLayers = 3;
struct CProb {
  int M;
  int c0;          // first cluster of this problem in the launch (set by chain_launch)
  int amap;        // first layer's A (K-major, box {64, 128})
  int nlayers;
  CLayer L[kChainMaxLayers];
};

constexpr int kChainMaxProb = 4;
constexpr int kChainMaxMaps = 48;
struct CBatch {
  CUtensorMap maps[kChainMaxMaps];
  CProb p[kChainMaxProb];
  int nprob, nclusters;
  int prefetch_b;  // weights may be loaded before griddepcontrol.wait
  unsigned long long* dbg;  // optional per-CTA phase timestamps [cta][16] (SQUINT_CHAIN_DBG)
};

// Host builder.  Matrices as in gemm.cuh (bf16 row-major, logical size, 16-byte pitch).
struct ChainBuilder {
  CBatch b;
  Mat amat[kChainMaxProb];
  Mat wmat[kChainMaxProb][kChainMaxLayers], omat[kChainMaxProb][kChainMaxLayers], xmat[kChainMaxProb][kChainMaxLayers];
  int err = 0;
  // global scratch for the next-layer exchange of layers without a stored output (chain_launch
  // maps M x 256 bf16 per such layer while it lasts; the rest exchange through DSMEM)
  char* xscr = nullptr;
  size_t xcap = 0;
  explicit ChainBuilder(int prefetch_b = 1) {
    b.nprob = 0;
    b.nclusters = 0;
    b.prefetch_b = prefetch_b;
  }
  CProb& add(int M, const Mat& A);
  // Layer l of problem p: weight W (K-major [N][K] for forward, MN-major [K][N] for dX), output
  // O (bf16 [M][N], may have ptr == NULL), x_hat X (bf16 [M][N], fwd store / bwd load, may be NULL).
  CLayer& layer(CProb& p, int epi, const Mat& W, int b_mn, int N, int K, const Mat& O, const Mat& X);
};

// Returns 0 on success, a cudaError_t, or -1 on a planning error (unsupported shape).
int chain_launch(ChainBuilder& cb, cudaStream_t s);
// The chain handles hidden width 256 (4 x 64-column slices) with K <= 256 per layer.
bool chain_supported(int hidden);
int chain_debug_times(unsigned long long* host, int max_entries);
unsigned long long* chain_dbg_for_launch(int nctas);  // SQUINT_CHAIN_DBG stamps buffer or NULL

}  // namespace sq
