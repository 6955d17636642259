/*
 * squint.h -- C ABI of libsquint, the B200 (sm_100a) hot path of Squint's visual SAC
 * (arXiv 2602.21203).  Citations: P:n = PAPER.md line n, S:n = SPEC.md line n,
 * Qn = reading n of SURVEY.md §8(c) (restated in DESIGN.md §3).
 *
 * Conventions for every entry point:
 *  - Pointers are DEVICE pointers unless the comment says "host".
 *  - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy default
 *    stream).  No call synchronises, allocates or frees device memory: the caller
 *    (PyTorch in the Python binding) owns all memory, including `workspace`.
 *  - Calls on one stream serialise.  The library keeps no global state
 *    except a thread-local error string and an optional per-thread graph cache.
 *  - Errors are returned as squint_status; squint_last_error() gives the message.
 *    Host-checkable conditions are checked before any launch (nothing is launched when
 *    a check fails).  Device-side preconditions (index ranges, distinct slots) are
 *    documented and are NOT checked (checking would need a synchronisation).
 *  - Floating-point tensors are row-major fp32; images are u8 CHW planar (Q2).
 */
#ifndef SQUINT_H
#define SQUINT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SQUINT_API __attribute__((visibility("default")))
#else
#define SQUINT_API
#endif

typedef struct CUstream_st* squint_stream_t; /* == cudaStream_t */

typedef enum {
  SQUINT_OK = 0,
  SQUINT_EINVAL = 1,       /* invalid argument value */
  SQUINT_ESHAPE = 2,       /* inconsistent shapes */
  SQUINT_ECUDA = 3,        /* a CUDA launch / runtime call failed */
  SQUINT_ENCCL = 4,        /* an NCCL call failed */
  SQUINT_EUNSUPPORTED = 5  /* shape/precision combination not built */
} squint_status;

enum { SQUINT_FP32 = 0, /* fp32 SIMT path (parity mode)                        */
       SQUINT_BF16 = 1  /* bf16 operands, fp32 accumulate, fp32 master weights */ };

/* Parameter groups.  CRITIC = encoder psi + critic projection + twin heads (the encoder
 * is trained only by the critic loss); ACTOR = actor projection + MLP
 * (P:157); ALPHA = log alpha; TARGET = EMA copy of the critic tensors except psi (Q28). */
enum { SQUINT_GROUP_CRITIC = 0, SQUINT_GROUP_ACTOR = 1, SQUINT_GROUP_ALPHA = 2,
       SQUINT_GROUP_TARGET = 3 };

typedef struct {
  char name[48];   /* e.g. "critic.q1.l2.w" */
  int group;       /* SQUINT_GROUP_* */
  int64_t offset;  /* in floats, into the group's flat buffer (128-byte aligned) */
  int64_t numel;
  int ndim;
  int shape[4];    /* row-major; linear W is [out, in], conv W is [out, in, 3, 3] */
} squint_tensor_desc;

/* Problem shape, host struct.  Architecture per Q7-Q12:
 * conv3x3/s2 -> ReLU -> conv3x3/s1 -> ReLU -> flatten (25*conv_ch) -> two projections
 * Linear->latent->LN->tanh; actor MLP [z,s]->H->LN->ReLU->H->LN->ReLU->2A; twin critic
 * heads [z,s,a]->H->LN->ReLU->H->LN->ReLU->n_atoms. */
typedef struct {
  int img_c, img_h, img_w;      /* 3, 16, 16 stored resolution          */
  int pad;                      /* random-shift pad, 2 (Q5)                      */
  int conv_ch;                  /* 32 | 64                                       */
  int latent;                   /* 50                                            */
  int proprio_dim, action_dim;  /* 12, 6                                         */
  int critic_hidden, actor_hidden; /* 256 | 512, 256                             */
  int n_atoms;                  /* 51 | 101                              */
  float v_min, v_max;           /* atom support, v_min < v_max           */
  int batch;                    /* per-rank batch B                              */
  int precision;                /* SQUINT_FP32 | SQUINT_BF16                     */
  int critic_kind;              /* SQUINT_CRITIC_C51 (the paper's distributional
                                   critic) | SQUINT_CRITIC_MSE: scalar heads
                                   (width 1) trained on the squared TD error of
                                   Eqs. 1-2 / Algorithm 1 (f3); n_atoms, v_min,
                                   v_max are then unused                          */
} squint_dims;
enum { SQUINT_CRITIC_C51 = 0, SQUINT_CRITIC_MSE = 1 };

typedef struct {
  float gamma;          /* discount, 0 <= gamma <= 1                     */
  float tau;            /* Polyak rate, 0 <= tau <= 1 (rho = 1 - tau) */
  float lr_critic, lr_actor, lr_alpha;
  float beta1, beta2, adam_eps;   /* Adam (Q26)                          */
  float target_entropy; /* H_t, -A (Q15)                                  */
  float ln_eps;         /* 1e-5 (Q9)                                      */
  float log_std_min, log_std_max; /* -5, 2 (Q13)                          */
  int target_mode;      /* SQUINT_TARGET_AVG (the paper's, Algorithm 1
                           line 13) | SQUINT_TARGET_CDQ: per sample the target
                           head with the smaller expected value (f3) */
} squint_hparams;
enum { SQUINT_TARGET_AVG = 0, SQUINT_TARGET_CDQ = 1 };

/* Replay ring, structure of arrays, caller-owned. */
typedef struct {
  const uint8_t* obs;           /* [capacity, C, H, W] u8 */
  const uint8_t* next_obs;      /* [capacity, C, H, W] u8 */
  const float* proprio;         /* [capacity, P] */
  const float* next_proprio;    /* [capacity, P] */
  const float* action;          /* [capacity, A] in [-1, 1] */
  const float* reward;          /* [capacity] */
  const uint8_t* done;          /* [capacity], 1 = terminal (Q22) */
  int64_t capacity, size;       /* sampled indices must be < size (not checked) */
} squint_replay;

/* Learner state: flat fp32 buffers laid out by squint_param_layout (caller-owned). */
typedef struct {
  float* critic;         /* group CRITIC params (master fp32)          */
  float* critic_target;  /* group TARGET params                         */
  float* actor;          /* group ACTOR params                          */
  float* log_alpha;      /* [1]                                         */
  float* m_critic; float* v_critic;   /* Adam moments, same layout */
  float* m_actor;  float* v_actor;
  float* m_alpha;  float* v_alpha;    /* [1] each */
  int64_t* step;         /* [3] Adam step counters: critic, actor, alpha */
} squint_state;

/* ---- host-side layout queries (no GPU needed) ------------------------------------ */
SQUINT_API const char* squint_last_error(void);
SQUINT_API const char* squint_version(void);

/* Fills `out[0..max_out)` (host, may be NULL) with every tensor of every group, sets
 * *n_tensors, and group_sizes[4] (floats, padded) for CRITIC, ACTOR, ALPHA, TARGET.
 * Errors: EINVAL on invalid dims (batch <= 0 ...). */
SQUINT_API squint_status squint_param_layout(const squint_dims* dims, squint_tensor_desc* out, int max_out,
                                  int* n_tensors, int64_t group_sizes[4]);

/* Device workspace bytes needed by squint_update for `dims` (utd does not change it). */
SQUINT_API squint_status squint_workspace_bytes(const squint_dims* dims, int utd, size_t* bytes);

/* Offset/bytes of a named workspace region (debug/test access to intermediates):
 * 0 = critic gradient (CRITIC layout), 1 = actor gradient (ACTOR layout) -- in SQUINT_BF16
 *     precision the projection weights' gradients (critic.proj.w, actor.proj.w, [latent][25C])
 *     are stored pixel-major, column pix * C + c (the bf16 encoder's HWC flatten order; the
 *     optimizer gathers them), every other tensor as in squint_param_layout,
 * 2 = target distribution m [B, n_atoms], 3 = h [B, 25C], 4 = log pi (current) [B],
 * 5 = log pi' (next) [B], 6 = actions a~ [B, A], 7 = scalars [16],
 * 8 = the last update's gathered, shifted obs images u8 [B, C, H, W] (a3-a4; the conv1 weight
 *     gradient's input), 9 = (SQUINT_BF16, with squint_set_option(5, 1)) the same for next_obs,
 * 10 = (SQUINT_BF16) the obs images' conv1 activations, bf16 [B, 7 * 7, conv_ch] (pixel-major). */
SQUINT_API squint_status squint_workspace_region(const squint_dims* dims, int region, size_t* offset, size_t* bytes);

/* Workspace bytes needed by squint_act for n frames. */
SQUINT_API squint_status squint_act_workspace_bytes(const squint_dims* dims, int64_t n, size_t* bytes);

/* ---- multi-GPU (data parallel) ------------------------------------ */
/* Writes a 128-byte NCCL unique id to `id_out` (host).  Call on rank 0, broadcast the
 * bytes with torch.distributed, then every rank calls squint_comm_init. */
SQUINT_API squint_status squint_comm_unique_id(void* id_out);
SQUINT_API squint_status squint_comm_init(void** comm, const void* id /* host, 128 B */, int rank, int nranks);
SQUINT_API squint_status squint_comm_destroy(void* comm);
/* Gradient exchange of the SQUINT_BF16 update (the per-update gradient
 * steps of Algorithm 1, with the critic, alpha and actor ordering of Q19):
 *   mode 0 (default): ncclAllReduce(sum) of each flat gradient group + its row-sum tail, then
 *          Adam replicated on every rank;
 *   mode 1: peer memory over NVLink.  Every rank's gradient, parameter and partial-sum buffers are
 *          mapped into each process (cudaIpcMemHandle records exchanged with ncclAllGather on
 *          first use of a buffer -- so that first call must not be inside a stream capture);
 *          per group one kernel sums this rank's 1/G slice of the gradients from all peers in rank
 *          order, steps Adam on it (m, v: the slice only is touched) and stores the stepped
 *          fp32 slice into every rank's parameters; a one-block cross-rank barrier (system-scope
 *          release/acquire counters, own epoch in device memory, graph-replay safe) follows,
 *          then each rank refreshes its bf16 shadows.  The row-sum tails (alpha step, metrics)
 *          are summed in the barrier before the critic step.  G <= 8.
 *          The fp32 update (SQUINT_FP32) keeps mode 0.
 * Call on every rank with the same mode before the next squint_update.  The state's parameter
 * tensors (critic, actor) and the workspace must be device allocations (cudaMalloc-backed).
 * Errors: EINVAL (NULL comm, mode not 0/1), EUNSUPPORTED (G > 8, allocation failure). */
SQUINT_API squint_status squint_comm_set_mode(void* comm, int mode);

/* ---- a1: resolution squint + insert (Q1, Q4) ------------
 * frames u8 [n, c, h, w]; ring u8 [capacity, c, h/factor, w/factor];
 * ring[slots[f]][ch][i][j] = round_half_even(sum_{a,b<factor} frames[f][ch][factor*i+a][factor*j+b] / factor^2).
 * Preconditions (device, unchecked): 0 <= slots[f] < capacity, slots distinct.
 * Errors: ESHAPE if h or w is not divisible by factor; EINVAL if n < 0,
 * factor < 1, capacity < 1, or (w % 16) != 0 when factor == 8 (vector path).
 * n == 0 is a no-op. */
SQUINT_API squint_status squint_insert(const uint8_t* frames, int64_t n, int c, int h, int w, int factor,
                            const int64_t* slots, uint8_t* ring, int64_t capacity,
                            squint_stream_t stream);

/* a1 twice from one read of the frames: the squinted frames go to
 * ring[slots[f]] and to ring2[slots2[f]] (both [capacity, c, h/factor, w/factor]).  In the
 * Algorithm-1 loop the new observation o_{t+1} is the finished transition's next_obs (ring =
 * next_obs, slots = this step's slots) and the next transition's obs (ring2 = obs, slots2 = the
 * next step's slots); squint_act at the next step can then read the squinted rows (factor 1)
 * instead of squinting the full frames again.  Same preconditions and errors as squint_insert;
 * ring2 and slots2 are both NULL (then exactly squint_insert) or both non-NULL (EINVAL
 * otherwise); capacity bounds both slot arrays (the smaller ring's row count). */
SQUINT_API squint_status squint_insert2(const uint8_t* frames, int64_t n, int c, int h, int w, int factor,
                                        const int64_t* slots, uint8_t* ring, const int64_t* slots2, uint8_t* ring2,
                                        int64_t capacity, squint_stream_t stream);

/* a1 with the renderer-side variants of SURVEY §8(f) f4, fused before the squint.
 *   layout  SQUINT_LAYOUT_CHW: frames u8 [n, c, h, w] (as squint_insert);
 *           SQUINT_LAYOUT_HWC: frames u8 [n, h, w, c] (what renderers emit); the ring
 *           rows are CHW [c, h/factor, w/factor] either way.
 *   jitter  NULL, or f32 [n, 3] = (brightness, contrast, saturation) factors per frame, > 0,
 *           drawn by the caller (per episode or per step); needs c == 3.  Applied to
 *           the full-resolution frame before squinting, in this order (DESIGN.md reading
 *           R-jit; P:267 names "lighting and color jitter", S:55-63 the three factors):
 *             x1 = u8(b x);  m = sum_p grey(x1) / (h w);  x2 = u8(c x1 + (1 - c) m);
 *             x3 = u8(s x2 + (1 - s) grey(x2));  squint(x3)
 *           u8(v) = truncate(clamp(v, 0, 255)), grey(x) = u8((0.2989 R + 0.587 G) + 0.114 B),
 *           every f32 product and sum rounded separately.  (1, 1, 1) is a bitwise no-op.
 *   factor  1 is the direct-render path (Fig. 2: frames rendered at the stored resolution).
 * ring2 / slots2 as in squint_insert2.  CHW without jitter is exactly squint_insert2; the
 * other cases stage each frame in shared memory (one CTA per frame) and need c <= 4 and
 * c*h*w <= 200 KB (SQUINT_EUNSUPPORTED otherwise).  Errors: EINVAL (layout, NULL, jitter with
 * c != 3, ring2 without slots2), ESHAPE (divisibility). */
#define SQUINT_LAYOUT_CHW 0
#define SQUINT_LAYOUT_HWC 1
SQUINT_API squint_status squint_insert_ex(const uint8_t* frames, int64_t n, int c, int h, int w, int factor,
                                          int layout, const float* jitter, const int64_t* slots, uint8_t* ring,
                                          const int64_t* slots2, uint8_t* ring2, int64_t capacity,
                                          squint_stream_t stream);

/* ---- a16: batched rollout inference (Algorithm 1 L4-5) -------------------
 * frames u8 [n, img_c, frame_h, frame_w] with frame_h = img_h * f, frame_w = img_w * f
 * (f >= 1; f = 1 means already squinted); proprio [n, P]; eps [n, A] N(0,1) noise or
 * NULL for the mean action tanh(mu) (log pi then evaluated at eps = 0).
 * Outputs action_out [n, A], logp_out [n] (may be NULL).  If `ring`/`slots` are non-NULL
 * the squinted frames are also written to ring[slots[i]] (fused insert, Q4).
 * actor_params / critic_params are the ACTOR / CRITIC flat buffers (the encoder psi is
 * read from the head of CRITIC).  workspace >= squint_act_workspace_bytes.
 * n == 0 is a no-op. */
SQUINT_API squint_status squint_act(const squint_dims* dims, const squint_hparams* hp, const float* actor_params,
                         const float* critic_params, const uint8_t* frames, int64_t n, int frame_h,
                         int frame_w, const float* proprio, const float* eps, float* action_out,
                         float* logp_out, uint8_t* ring, const int64_t* slots, int64_t ring_capacity,
                         void* workspace, squint_stream_t stream);
/* squint_act with weights_read (a cudaEvent_t, may be NULL = squint_act): the act first copies the
 * weights it reads (the whole ACTOR buffer and the CRITIC encoder head) into the tail of its
 * workspace (squint_act_workspace_bytes includes the room), records weights_read on `stream`, and
 * computes from the copies.  A caller that runs the act beside optimizer steps (Algorithm 1 L4-5
 * acting with the pre-update policy while L8-24 update) waits on weights_read before its first
 * step writes ACTOR or CRITIC.  Results are bitwise those of squint_act. */
typedef void* squint_event_t;
SQUINT_API squint_status squint_act_ex(const squint_dims* dims, const squint_hparams* hp, const float* actor_params,
                                       const float* critic_params, const uint8_t* frames, int64_t n, int frame_h,
                                       int frame_w, const float* proprio, const float* eps, float* action_out,
                                       float* logp_out, uint8_t* ring, const int64_t* slots, int64_t ring_capacity,
                                       void* workspace, squint_stream_t stream, squint_event_t weights_read);

/* ---- a2-a15: `utd` sequential SAC updates (Algorithm 1 L8-24; Q17-Q30) -------------
 * idx [utd, B] int64 in [0, replay->size) (device, unchecked);
 * shifts [utd, B, 4] u8 = (dx, dy) for obs then (dx', dy') for next_obs, each in
 * [0, 2*pad] (Q5); eps [utd, 2, B, A] fp32 N(0,1): [:,0] next-state sample (target),
 * [:,1] current-state sample (alpha and actor losses) (Q18, Q32).
 * state is read and updated in place.  metrics [utd, 8] (device) receives, per update,
 * {L_Q, L_pi, L_alpha, alpha+, mean Q, entropy (-mean log pi), |grad critic|_2, nonfinite}.
 * A non-finite loss sets metrics[j][7] = 1 and the update continues.
 * comm: NULL for one GPU, else a handle from squint_comm_init; then B is the per-rank
 * batch, losses are scaled by 1/(B*nranks) and gradients/metric sums are SUM
 * all-reduced over ranks (Q33).
 * SQUINT_BF16 with comm == NULL, outside a stream capture: the call's ~30 launches per update
 * are captured once per distinct argument set (all pointers, dims, hparams, utd; not replay->size,
 * which only bounds the host-side index check) into a
 * CUDA graph kept in a small per-thread cache (8 entries) and replayed on `stream`; calls with
 * changed arguments capture anew.  SQUINT_NO_GRAPH=1 (debugging) launches directly.  Inside a caller's
 * capture the launches join that capture.
 * Errors: EINVAL (utd < 1, batch < 1, gamma/tau outside [0,1], size < 1, bad support),
 * ESHAPE (dims inconsistent), EUNSUPPORTED (shape/precision not built). */
SQUINT_API squint_status squint_update(const squint_dims* dims, const squint_hparams* hp, const squint_replay* replay,
                            const int64_t* idx, const uint8_t* shifts, const float* eps, int utd,
                            const squint_state* state, float* metrics, void* workspace, size_t workspace_bytes,
                            void* comm, squint_stream_t stream);

/* ---- a14: standalone Polyak: target[i] = (1 - tau) target[i] + tau online[i].
 * Errors: EINVAL if n < 0 or tau outside [0, 1]. */
SQUINT_API squint_status squint_soft_update(float* target, const float* online, int64_t n, float tau,
                                 squint_stream_t stream);

/* ---- runtime: stage a step's small inputs from pinned host memory by a kernel ----------
 * dst (device) <- src (page-locked host memory, cudaHostAlloc / cudaHostRegister), `bytes`
 * bytes, read over PCIe by the SMs (16-byte loads when both pointers are 16-byte aligned)
 * rather than by a copy engine: in an environment loop the per-step indices / noise / proprio
 * (~100 KB) then do not queue behind the next 50 MB frame upload on the DMA engine.
 * Asynchronous on `stream`; src must stay valid until the kernel has run.
 * Errors: EINVAL (NULL with bytes > 0, src not page-locked host memory). */
SQUINT_API squint_status squint_stage_pinned(void* dst, const void* src, size_t bytes, squint_stream_t stream);

/* Self-test of the bf16 tensor-core GEMM engine (gemm.cu), used by the GPU tests:
 * out[m][n] = sum_{k<K} A(m, k) B(n, k), fp32 [M][N] row-major (device), where A and B are
 * bf16 row-major device matrices (rows x cols, ld elements per row) read K-major
 * (A(m, k) = A[m][k]) or, with *_mn = 1, MN-major (A(m, k) = A[k][m]); likewise B.
 * Entries outside a matrix read as 0.  Asynchronous on `stream`. */
SQUINT_API squint_status squint_selftest_gemm(const void* A, int a_rows, int a_cols, int a_ld, int a_mn,
                                              const void* B, int b_rows, int b_cols, int b_ld, int b_mn,
                                              int M, int N, int K, float* out, squint_stream_t stream);

/* ---- instrumentation (bench.py) --------------------------------------------------------
 * Number of kernels libsquint has launched in this process (host counter). */
SQUINT_API long squint_launch_count(void);
/* When `events` (host array of n_phases * reps * 2 cudaEvent_t) is non-NULL, phase k of
 * update j (rep j; act/insert use rep 0) records events[(k*reps+j)*2] before and
 * events[(k*reps+j)*2+1] after its kernels on the launch stream.  NULL disables.
 * Phase names: squint_phase_name(k) (16 phases). */
SQUINT_API squint_status squint_set_phase_events(void** events, int n_phases, int reps);
SQUINT_API const char* squint_phase_name(int k);
/* Instrumentation: launch timeline.  While enabled, libsquint records events[i] (host array of
 * cudaEvent_t, created with timing) on the launch stream immediately before its i-th kernel
 * launch (i < n), so consecutive events bracket one launch including any gap after it.
 * Returns the number of events recorded since the previous call; NULL/0 disables. */
SQUINT_API int squint_set_launch_events(void** events, int n);
/* Host options (per process): key 1 = run the bf16 update's encoder-backward branch on an
 * auxiliary stream (1, default) or inline on the caller's stream (0; a launch timeline then
 * brackets consecutive launches of one stream); key 2 = pipeline each update's critic-side
 * forward (encoder, critic/target projections, online heads) onto the previous update's branch
 * (0, default; needs key 1); key 3 = validate the device-side preconditions before each call
 * (0, default): sampled indices in [0, replay.size), insert / act slots in [0, capacity) and
 * pairwise distinct -- a check kernel plus a stream synchronisation per call, returning
 * SQUINT_EINVAL with a message instead of undefined behaviour (skipped inside a stream
 * capture); key 4 = numerics measurement on the SQUINT_FP32 path only (0, default): round to bf16
 * what the SQUINT_BF16 path holds in bf16, before the fp32 arithmetic -- bit 0 the dense layers' GEMM
 * activations / dY, bit 1 their weights, bit 2 the LayerNorm x_hat cache, bit 3 the encoder's conv
 * weights, conv1 activations and conv gradients -- to measure how much of the bf16 path's deviation
 * from the oracle bf16 storage alone explains (reading R-tol-bf16); key 5 = (SQUINT_BF16, 0 default) the
 * encoder also stores the gathered, shifted next_obs images into workspace region 9 (test access to
 * the a3-a4 integer work).  Errors: EINVAL for an unknown key or value. */
SQUINT_API squint_status squint_set_option(int key, int value);
/* Records the next timeline event on `stream` without a launch (closes the last interval). */
SQUINT_API squint_status squint_record_launch_event(squint_stream_t stream);
/* Kernel name (static string) and algorithmic work of timeline launch i: FLOPs and bytes by the
 * problem definition (2*M*N*K summed over a grouped GEMM's problems; bytes an HBM/L2-bound
 * kernel must move), 0 when not tracked.  Host-only. */
SQUINT_API squint_status squint_launch_info(int i, const char** name, double* flops, double* bytes);

#ifdef __cplusplus
}
#endif
#endif /* SQUINT_H */
