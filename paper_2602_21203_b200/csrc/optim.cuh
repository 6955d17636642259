// optim.cuh -- temperature step, fused Adam, Polyak, per-update metrics (a11, a13, a14).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace sq {

// Scalar slots in the workspace (float[kScal]).
enum Scal : int {
  S_ALPHA1 = 0,        // alpha after its Adam step
  S_ALPHA1_SCALE = 1,  // alpha1 * loss scale (dL_pi / dlog pi)
  S_MEAN_LOGP = 2,
  S_LALPHA = 3,
  S_LQ = 4,
  S_C1_CRITIC = 5, S_C2_CRITIC = 6, S_C1_ACTOR = 7, S_C2_ACTOR = 8,
  kScal = 32
};
// Row sums that the data-parallel path all-reduces together with the critic gradient.
enum Extra : int { X_SUM_LOGP = 0, X_SUM_LQ = 1, kExtra = 32 };

struct ScalarsArgs {
  int B;                 // local rows
  float inv_btotal;      // 1 / global batch
  const float* logp;     // [B] current-state log pi (pre-step phi)
  const float* row_loss; // [B] per-row L_Q terms (already scaled)
  float* extras;         // [kExtra] row sums (written when compute_sums, else read)
  int compute_sums;
  float* log_alpha; float* m_alpha; float* v_alpha;
  int64_t* step;         // [3]
  float lr_alpha, beta1, beta2, adam_eps, target_entropy;
  float loss_scale;      // 1 / global batch
  float* scal;           // [kScal]
  int steps_done;        // 1: step[0], step[1] and their bias corrections were taken earlier
};

int launch_row_sums(const float* logp, const float* row_loss, int B, float* extras, cudaStream_t s);
int launch_scalars(const ScalarsArgs& a, cudaStream_t s);

// p -= lr * (m c1) / (sqrt(v c2) + eps) with m, v updated from g (Q26).  c1 = 1/(1-b1^t),
// c2 = 1/(1-b2^t) read from scal.  n % 4 == 0, 16-byte aligned.  If sumsq_part != NULL,
// writes sum(g^2) per block (kAdamBlocks entries, fixed order).
constexpr int kAdamBlocks = 296;
constexpr int kEncAdamBlocks = 16;  // the encoder's slice of the critic Adam (bf16 path, own stream)
int launch_adam(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2, float eps,
                const float* c1, const float* c2, float* sumsq_part, cudaStream_t s);
// target = (1 - tau) target + tau online; any n, any alignment.
int launch_polyak(float* target, const float* online, int64_t n, float tau, cudaStream_t s);

// bf16 shadow copies of the linear weights (bf16 tensor-core path).  Entry e maps the fp32
// tensor at flat offset src (rows x cols, row-major) of a group buffer onto the bf16 matrix
// dst[row * ld + col'] with col' = col, or, for perm_c > 0 (projection weights, whose input is
// the conv feature map flattened CHW, Q7), col = ch * perm_p + pix -> col' = pix * perm_c + ch
// (the HWC order the encoder writes).
struct ShadowEnt {
  int64_t src, dst;
  int rows, cols, ld, perm_c, perm_p;
};
constexpr int kMaxShadow = 8;
struct ShadowTable {
  int n;
  __nv_bfloat16* base;
  ShadowEnt e[kMaxShadow];
};
// Full refresh of one group's shadow from its fp32 master.
int launch_shadow(const float* master, const ShadowTable& t, cudaStream_t s);
// the three group shadows in one launch (a NULL table is skipped)
int launch_shadow3(const float* const master[3], const ShadowTable* const t[3], cudaStream_t s);
// Adam (as launch_adam) that also writes the updated weights' bf16 shadow (t may be NULL).
// `base` = flat group index of p[0] (shadow lookups), `nblocks` = grid (= partial sums written).
// grad_perm: gradients of permuted shadow entries (the projection weight) are stored in the
// shadow's column order (pixel-major, row pitch = cols) and gathered through the permutation.
int launch_adam_shadow(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                       float eps, const float* c1, const float* c2, float* sumsq_part, const ShadowTable* t,
                       cudaStream_t s, int64_t base = 0, int nblocks = kAdamBlocks, int grad_perm = 0);
// Polyak over a 16-byte aligned buffer (n % 4 == 0) that also refreshes the target shadow.
// dst (device) <- src (device-mapped pinned host memory), read by the SMs over PCIe
int launch_stage_pinned(void* dst, const void* src, size_t bytes, cudaStream_t s);
int launch_polyak_shadow(float* target, const float* online, int64_t n, float tau, const ShadowTable* t,
                         cudaStream_t s);

// dst_j[i] = sum_{r < nsplit} src_j[r n_j + i] in r order (the K-split partials of weight-gradient
// launches; fixed order: bitwise reproducible)
constexpr int kMaxSplitJobs = 16;
struct SplitSumJobs {
  int njobs, nsplit;
  float* dst[kMaxSplitJobs];
  const float* src[kMaxSplitJobs];
  int n[kMaxSplitJobs];
};
int launch_split_sum(const SplitSumJobs& j, cudaStream_t s);

struct MetricsArgs {
  int B;
  float inv_btotal;
  const float* row_lpi;  // [B] (scaled)
  const float* row_q;    // [B]
  const float* sumsq_part;  // [kAdamBlocks]
  const float* scal;
  const float* extras;
  float* out;            // [8]
  int npart;             // number of Adam partial sums of squares (0 -> kAdamBlocks)
  int reduce_local;      // 1: sum row_lpi/row_q here; 0: read pre-reduced sums from extras2
  const float* extras2;  // [2] = (sum row_lpi, sum row_q) when reduce_local == 0
};
int launch_metrics(const MetricsArgs& a, cudaStream_t s);
int launch_lpi_sums(const float* row_lpi, const float* row_q, int B, float* out2, cudaStream_t s);

// ---- f1: peer-memory all-reduce fused with a sharded Adam (data-parallel bf16 update) ----------
// Pointers are every rank's copy of a buffer as mapped in this process (CUDA IPC; own rank = local).
constexpr int kDpMaxRanks = 8;
struct DpSync {
  unsigned* flag[kDpMaxRanks];  // rank q's arrival counters [kDpMaxRanks] (+ its epoch)
  unsigned* own;                // this rank's counters; own[kDpMaxRanks] = its epoch
  int G, rank;
  const float* tail[kDpMaxRanks];  // every rank's row-sum tail (ntail floats), or unused
  float* tail_out;                 // [ntail] local: sum over ranks
  int ntail;
  // optional (ra != NULL): first this rank's row sums, tail_mine[0] = sum ra[0..B), [1] = sum rb
  const float* ra;
  const float* rb;
  int B;
  float* tail_mine;
};
// [row sums into this rank's tail,] cross-rank barrier (all ranks' earlier stream work done and
// visible), then the tail sum
int launch_dp_sync(const DpSync& a, cudaStream_t s);
struct DpAdam {
  const float* g[kDpMaxRanks];  // every rank's flat gradient of the group
  float* p[kDpMaxRanks];        // every rank's fp32 parameters of the group
  float* part[kDpMaxRanks];     // every rank's sum(g^2) partials [G * kAdamBlocks]
  __nv_bfloat16* sh[kDpMaxRanks];  // every rank's copy of the group's shadow buffer (t->base)
  int G, rank;
  int64_t lo4, hi4;             // this rank's slice, float4 units
};
// Adam (as launch_adam_shadow without the shadow) on this rank's slice of the all-reduced gradient;
// t: the group's shadow table (grad_perm gather; the stepped weights' bf16 entries are stored into
// every rank's shadow buffer sh[q]).  Needs a launch_dp_sync after it before any rank reads its
// parameters or shadows.
int launch_dp_adam(const DpAdam& d, float* m, float* v, float lr, float b1, float b2, float eps, const float* c1,
                   const float* c2, const ShadowTable* t, int grad_perm, cudaStream_t s);

}  // namespace sq
