// heads.cuh -- row kernels of the distributional critic (a9, a10, a12).
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

namespace sq {

struct TargetCEArgs {
  int B, N;
  float v_min, v_max, gamma, scale;
  const float* tlogits;    // [2][B][N] target heads (theta_bar) on (z', s', a')
  const float* logits;     // [2][B][N] online heads on (z, s, a)
  const int64_t* idx;      // [B] replay rows
  const float* reward;     // ring [cap]
  const uint8_t* done;     // ring [cap]
  const float* logp_next;  // [B]
  const float* log_alpha;  // [1] (alpha_0 = exp, read before the alpha step)
  float* m;                // [B][N]
  float* dlogits;          // [2][B][N] fp32 (fp32 path) ...
  __nv_bfloat16* dlogits_bf;  // ... or bf16 [2][B][ld_dl] (bf16 path; used when non-NULL)
  int ld_dl;
  float* row_loss;         // [B]
  // optional (step != NULL): block 0 takes the critic and actor Adam steps, step[0..1] += 1, and
  // writes their bias corrections into scal (so the optimizers need not wait for the alpha step)
  int64_t* step;
  float* scal;
  float beta1, beta2;
  unsigned long long* dbg;  // optional per-warp globaltimer stamps [B][4] (SQUINT_TCE_DBG)
  int cdq;                  // 1: project the head with the smaller expected value (f3)
  int mse;                  // 1: scalar critic (N == 1): m = y [B], dL/dQ_i = 2 s (Q_i - y) (f3)
};

struct ActorQArgs {
  int B, N;
  float v_min, v_max, scale;
  const float* logits;     // [2][B][N] critic theta+ on (z+, s, a~)
  const float* logp;       // [B]
  const float* alpha1;     // [1] alpha after its step
  float* dlogits;          // [2][B][N] fp32 ...
  __nv_bfloat16* dlogits_bf;  // ... or bf16 [2][B][ld_dl] when non-NULL
  int ld_dl;
  float* row_q;            // [B]
  float* row_lpi;          // [B]
  int mse;                 // 1: scalar critic, Q_i = logits (N == 1), dL_pi/dQ_i = -s/2 (f3)
};

int launch_target_ce(const TargetCEArgs& a, cudaStream_t s);
int launch_actor_q(const ActorQArgs& a, cudaStream_t s);

}  // namespace sq
