// update_bf16.cu -- launch sequence of the bf16 tensor-core path (SQUINT_BF16) for
// squint_update (Algorithm 1 L9-24) and squint_act (L4-5).
//
// Data flow.  Every GEMM operand is a bf16 row-major matrix read by TMA (gemm.cu):
//  * linear weights: bf16 "shadow" copies of the fp32 master parameters, refreshed from the
//    master at the start of each call (k_shadow) and rewritten by every Adam / Polyak step
//    (a13, a14), so the tensor cores never read a stale weight;
//  * activations: each layer's epilogue writes its bf16 output straight into the next
//    GEMM's operand matrix.  Layer inputs that are concatenations (critic [z, s, a], Q11;
//    actor [z, s], Q12) are single matrices whose column blocks are filled by their
//    producers: the projection epilogue (z), the encoder kernel's replay row gathers (s, a;
//    a3), the tanh-Gaussian epilogue (a~, a~').
// The conv feature map h is stored HWC (pix * C + ch); the projection weights' shadow is
// column-permuted to match, and their gradient is written back in the master's CHW order.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <optional>
#include <string>

#include "../../include/squint.h"
#include "comm.hpp"
#include "common.cuh"
#include "encoder.cuh"
#include "chain.cuh"
#include "gemm.cuh"
#include "heads.cuh"
#include "layout.hpp"
#include "optim.cuh"
#include "update_bf16.hpp"

namespace sq {

namespace {

// row pitch of the bf16 workspace matrices and weight shadows: 128 bytes (64 elements), so every
// TMA box row starts on a 128-byte line (unaligned pitches cost ~30-40 % of the TMA rate)
inline int ldp(int x) { return (x + 63) & ~63; }
inline int mtiles(int m) { return (m + 127) / 128; }

struct FB {  // fp32 buffer inside the workspace
  size_t off;
  int64_t n;  // floats
};

struct BM {  // bf16 matrix inside the workspace
  size_t off;
  int rows, cols, ld;
};

struct ShadowPlan {
  ShadowTable t;  // base filled at call time
  size_t off;     // bytes into the workspace
  size_t elems;
};

struct BfLay {
  BM Xh, Xhn, Xq, Xt, Xq1, Xan, Xac;
  BM Xh_alt, Xq1_alt, Xac_alt;  // odd updates (the pipelined forward of update j+1 runs beside j)
  BM H1an, H2an, H1ac, H2ac;
  BM tqH1[2], tqH2[2], qH1[2], qH2[2], q1H1[2], q1H2[2];
  BM XH1ac, XH2ac, XHpq, XHpp, XHpq1, qXH1[2], qXH2[2], q1XH1[2], q1XH2[2];  // bf16 LN caches x_hat
  BM dlog, dlog1;  // [2B][N] (head i = rows i*B ...)
  BM dA2c[2], dA1c[2], dA2a[2], dA1a[2], dAp, dh, dO, adA2, adA1, adAp;
  size_t R1ac, R2ac, Rpq, Rpp, Rpq1, qR1[2], qR2[2], q1R1[2], q1R2[2];
  size_t tlogits, logits, logits1, m, tgo_ac, a_cur, logp_cur, logp_next, row_loss, row_q, row_lpi;
  FB part_q2[2], part_q1[2], part_pq, part_a2, part_a1, part_pp;  // LayerNorm column partials
  size_t grad_critic, grad_actor, adam_part, scal, lpi_sums, dp_tail;
  size_t y1b, img0, img1, dA1enc, enc_part, wtiles;
  FB dwsplit;  // fp32 partials of K-split weight-gradient launches (dw_launch)
  size_t xchg, xchg_bytes;  // chain next-layer exchange scratch (ChainBuilder::xscr)
  // bf16 shadows: critic, target, actor, and a second critic set -- update j reads the critic set of
  // parity j (theta) and its Adam writes the other one (theta+), so a kernel still reading theta on the
  // forked branch (the dh GEMM) never races the main stream's Adam (with_parity swaps sh[0] / sh[3])
  ShadowPlan sh[4];
  size_t total;
};

const char* kHeads[2] = {"critic.q1", "critic.q2"};
constexpr int kDwMaxSplit = 4;

ShadowPlan shadow_plan(WsPlan& P, const squint_dims& d, const Layout& L, int grp) {
  ShadowPlan s;
  memset(&s, 0, sizeof(s));
  const int C = d.conv_ch, P2 = conv2_out(d) * conv2_out(d);
  size_t e = 0;
  auto add = [&](const std::string& name, int perm) {
    for (const auto& t : L.t) {
      if (t.group != grp || t.name != name) continue;
      ShadowEnt& x = s.t.e[s.t.n++];
      x.src = t.off;
      x.rows = t.shape[0];
      x.cols = t.shape[1];
      x.ld = ldp(x.cols);
      x.dst = (int64_t)e;
      x.perm_c = perm ? C : 0;
      x.perm_p = perm ? P2 : 0;
      e += (((size_t)x.rows * x.ld) + 63) & ~size_t(63);
    }
  };
  if (grp == SQUINT_GROUP_ACTOR) {
    add("actor.proj.w", 1);
    add("actor.l1.w", 0);
    add("actor.l2.w", 0);
    add("actor.l3.w", 0);
  } else {
    add("critic.proj.w", 1);
    for (int i = 0; i < 2; ++i)
      for (const char* l : {".l1.w", ".l2.w", ".l3.w"}) add(std::string(kHeads[i]) + l, 0);
  }
  s.elems = e;
  s.off = P.take(e * 2);
  return s;
}

BfLay plan_bf(const squint_dims& d, const Layout& L) {
  WsPlan P;
  BfLay w;
  const int B = d.batch, F = flat_dim(d), Lt = d.latent, Hc = d.critic_hidden, Ha = d.actor_hidden, N = head_out(d),
            A = d.action_dim, C = d.conv_ch, P1 = conv1_out(d) * conv1_out(d);
  const int nq = Lt + d.proprio_dim + A, npi = Lt + d.proprio_dim;
  const size_t f = sizeof(float);
  auto bm = [&](int rows, int cols) {
    BM m{0, rows, cols, ldp(cols)};
    m.off = P.take((size_t)rows * m.ld * 2);
    return m;
  };
  auto fl = [&](size_t n) { return P.take(n * f); };
  // column partials [mtiles * ks][3][N]: room for the largest split-K cluster gemm_launch plans
  auto fb = [&](size_t n) { return FB{P.take(kGemmMaxSplitK * n * f), (int64_t)(kGemmMaxSplitK * n)}; };
  w.Xh = bm(B, F);
  w.Xhn = bm(B, F);
  w.Xq = bm(B, nq);
  w.Xt = bm(B, nq);
  w.Xq1 = bm(B, nq);
  w.Xan = bm(B, npi);
  w.Xac = bm(B, npi);
  w.Xh_alt = bm(B, F);
  w.Xq1_alt = bm(B, nq);
  w.Xac_alt = bm(B, npi);
  w.H1an = bm(B, Ha);
  w.H2an = bm(B, Ha);
  w.H1ac = bm(B, Ha);
  w.H2ac = bm(B, Ha);
  w.XH1ac = bm(B, Ha);
  w.XH2ac = bm(B, Ha);
  w.XHpq = bm(B, Lt);
  w.XHpp = bm(B, Lt);
  w.XHpq1 = bm(B, Lt);
  for (int i = 0; i < 2; ++i) {
    w.tqH1[i] = bm(B, Hc);
    w.tqH2[i] = bm(B, Hc);
    w.qH1[i] = bm(B, Hc);
    w.qH2[i] = bm(B, Hc);
    w.qXH1[i] = bm(B, Hc);
    w.qXH2[i] = bm(B, Hc);
    w.q1H1[i] = bm(B, Hc);
    w.q1H2[i] = bm(B, Hc);
    w.q1XH1[i] = bm(B, Hc);
    w.q1XH2[i] = bm(B, Hc);
    w.dA2c[i] = bm(B, Hc);
    w.dA1c[i] = bm(B, Hc);
    w.dA2a[i] = bm(B, Hc);
    w.dA1a[i] = bm(B, Hc);
  }
  w.dlog = bm(2 * B, N);
  w.dlog1 = bm(2 * B, N);
  w.dAp = bm(B, Lt);
  w.dh = bm(B, F);
  w.dO = bm(B, 2 * A);
  w.adA2 = bm(B, Ha);
  w.adA1 = bm(B, Ha);
  w.adAp = bm(B, Lt);
  w.R1ac = fl(B);
  w.R2ac = fl(B);
  w.Rpq = fl(B);
  w.Rpp = fl(B);
  w.Rpq1 = fl(B);
  for (int i = 0; i < 2; ++i) {
    w.qR1[i] = fl(B);
    w.qR2[i] = fl(B);
    w.q1R1[i] = fl(B);
    w.q1R2[i] = fl(B);
  }
  w.tlogits = fl(2 * (size_t)B * N);
  w.logits = fl(2 * (size_t)B * N);
  w.logits1 = fl(2 * (size_t)B * N);
  w.m = fl((size_t)B * N);
  w.tgo_ac = fl((size_t)B * 2 * A);
  w.a_cur = fl((size_t)B * A);
  w.logp_cur = fl(B);
  w.logp_next = fl(B);
  w.row_loss = fl(B);
  w.row_q = fl(B);
  w.row_lpi = fl(B);
  const size_t mt = mtiles(B);
  for (int i = 0; i < 2; ++i) {
    w.part_q2[i] = fb(mt * 3 * Hc);
    w.part_q1[i] = fb(mt * 3 * Hc);
  }
  w.part_pq = fb(mt * 3 * Lt);
  w.part_a2 = fb(mt * 3 * Ha);
  w.part_a1 = fb(mt * 3 * Ha);
  w.part_pp = fb(mt * 3 * Lt);
  w.grad_critic = fl(L.gsize[SQUINT_GROUP_CRITIC] + kExtra);
  w.grad_actor = fl(L.gsize[SQUINT_GROUP_ACTOR] + kExtra);
  // [G * kAdamBlocks] with the peer-memory data-parallel Adam (f1)
  w.adam_part = fl(kDpMaxRanks * kAdamBlocks > kAdamBlocks + kEncAdamBlocks ? kDpMaxRanks * kAdamBlocks
                                                                            : kAdamBlocks + kEncAdamBlocks);
  w.dp_tail = fl(2 * kExtra);
  w.scal = fl(kScal);
  w.lpi_sums = fl(2);
  w.y1b = P.take((size_t)B * P1 * C * 2);
  w.img0 = P.take((size_t)B * d.img_c * d.img_h * d.img_w);
  w.img1 = P.take((size_t)B * d.img_c * d.img_h * d.img_w);
  w.dA1enc = 0;
  w.enc_part = fl(enc_bwd_tc_partial_floats(C, B));
  w.wtiles = P.take(conv_tiles_bytes(C));
  {
    // K-split weight gradients (dw_launch): up to kDwMaxSplit partial copies of the largest launch
    const size_t crit = 2 * ((size_t)N * Hc + (size_t)Hc * Hc + (size_t)Hc * nq + N + 2 * Hc) + (size_t)Lt * F + Lt;
    const size_t act = (size_t)2 * A * Ha + (size_t)Ha * Ha + (size_t)Ha * npi + (size_t)Lt * F + 2 * A + 2 * Ha + Lt;
    const size_t n = (size_t)kDwMaxSplit * (crit > act ? crit : act);
    w.dwsplit = FB{P.take(n * f), (int64_t)n};
  }
  // fused-chain exchange scratch: up to 4 problems x 2 hidden layers of B x 256 bf16
  w.xchg_bytes = (chain_supported(Hc) && chain_supported(Ha)) ? (size_t)4 * 2 * B * 256 * 2 : 0;
  w.xchg = P.take(w.xchg_bytes);
  w.sh[0] = shadow_plan(P, d, L, SQUINT_GROUP_CRITIC);
  w.sh[1] = shadow_plan(P, d, L, SQUINT_GROUP_TARGET);
  w.sh[2] = shadow_plan(P, d, L, SQUINT_GROUP_ACTOR);
  w.sh[3] = shadow_plan(P, d, L, SQUINT_GROUP_CRITIC);
  w.total = P.top + 256;
  return w;
}

// Per-thread auxiliary stream and events: the encoder backward and the encoder's Adam slice run
// on a branch forked from the caller's stream (graph capture turns this into parallel graph
// nodes) while the actor-loss chain proceeds; the branch joins before the metrics kernel.
struct Aux {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, scal = nullptr, join = nullptr, alpha = nullptr, qdone = nullptr;
  cudaEvent_t enc = nullptr, chn = nullptr;  // pipelined forward of the next update: encoder + projections, online heads
  bool ok() {
    if (s) return true;
    return cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) == cudaSuccess &&
           cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&scal, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&alpha, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&qdone, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&enc, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&chn, cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&join, cudaEventDisableTiming) == cudaSuccess;
  }
};
thread_local Aux t_aux;
// instrumentation (squint_set_option): 0 disables the auxiliary branch, so a launch timeline's
// consecutive events bracket consecutive launches of one stream
int g_branch_enabled = 1;
// option 2: pipeline the next update's critic-side forward onto the branch (early_fwd); off by
// default -- on B200 it measured even with the separate forward (the encoder backward that
// precedes it on the branch and the SMs it occupies set the pace), kept for other shapes
int g_pipe_enabled = 0;
// option 5: the encoder also stores the gathered, shifted next_obs images (workspace region 9)
int g_dump_next = 0;


struct Ctx {
  const squint_dims& d;
  const Layout& L;
  char* ws;
  cudaStream_t s;
  bool chain;      // fused forward MLP chains (hidden width 256) instead of one launch per layer
  Aux* aux;        // auxiliary branch (NULL: everything on the caller's stream)
  Mat mat(const BM& m) const { return Mat{ws + m.off, m.rows, m.cols, m.ld}; }
  bf16* bp(const BM& m) const { return reinterpret_cast<bf16*>(ws + m.off); }
  float* F(size_t off) const { return reinterpret_cast<float*>(ws + off); }
  float* F(const FB& b) const { return reinterpret_cast<float*>(ws + b.off); }
  // head i of a [2B][N] matrix
  Mat half(const BM& m, int i) const {
    return Mat{ws + m.off + (size_t)i * (m.rows / 2) * m.ld * 2, m.rows / 2, m.cols, m.ld};
  }
};

// One linear layer: bf16 shadow weight + fp32 bias / LN affine (from the master buffer).
struct Lin {
  Mat w;
  const float *b, *g, *beta;
};
Lin lin(const Ctx& c, const ShadowPlan& sp, const float* master, int grp, const std::string& p,
        const std::string& lnp) {
  Lin l;
  memset(&l, 0, sizeof(l));
  const int64_t woff = c.L.off(grp, p + ".w");
  for (int k = 0; k < sp.t.n; ++k)
    if (sp.t.e[k].src == woff) {
      const ShadowEnt& e = sp.t.e[k];
      l.w = Mat{c.ws + sp.off + (size_t)e.dst * 2, e.rows, e.cols, e.ld};
    }
  l.b = master + c.L.off(grp, p + ".b");
  if (!lnp.empty()) {
    l.g = master + c.L.off(grp, lnp + ".g");
    l.beta = master + c.L.off(grp, lnp + ".b");
  }
  return l;
}
struct Mlp {
  Lin l1, l2, l3;
};
Mlp mlp(const Ctx& c, const ShadowPlan& sp, const float* master, int grp, const std::string& p) {
  return Mlp{lin(c, sp, master, grp, p + ".l1", p + ".ln1"), lin(c, sp, master, grp, p + ".l2", p + ".ln2"),
             lin(c, sp, master, grp, p + ".l3", "")};
}
Lin proj(const Ctx& c, const ShadowPlan& sp, const float* master, int grp, const std::string& p) {
  return lin(c, sp, master, grp, p + ".proj", p + ".proj.ln");
}
// gradient views
struct LinG {
  float *w, *b, *g, *beta;
};
LinG ling(const Layout& L, float* base, int grp, const std::string& p, const std::string& lnp) {
  LinG v;
  v.w = base + L.off(grp, p + ".w");
  v.b = base + L.off(grp, p + ".b");
  v.g = lnp.empty() ? nullptr : base + L.off(grp, lnp + ".g");
  v.beta = lnp.empty() ? nullptr : base + L.off(grp, lnp + ".b");
  return v;
}

// ---- problem helpers ---------------------------------------------------------------------
// y = epi(X W^T + b): X [M][K] K-major, W [N][K] K-major.
GProb& fwd(GemmBuilder& gb, const Mat& X, const Lin& W, int epi, bf16* out, int ldo, float ln_eps) {
  GProb& p = gb.add(X.rows, W.w.rows, epi);
  gb.seg(p, X, 0, 0, W.w, 0, 0, W.w.cols);
  p.bias = W.b;
  p.g = W.g;
  p.beta = W.beta;
  p.out = out;
  p.ldo = ldo;
  p.ln_eps = ln_eps;
  return p;
}
// dX[m][j] = sum_n D[m][n] W[n][col0 + j], j < ncols: D K-major, W MN-major.
// The MN-major box start must be 16-byte aligned: an unaligned col0 is aligned down and the
// slack is skipped in the epilogue (acc_col0; only the tanh-Gaussian backward uses it).
GProb& dx(GemmBuilder& gb, const Mat& D, const Mat& W, int col0, int ncols, int epi) {
  const int al = col0 & ~7;
  GProb& p = gb.add(D.rows, ncols + (col0 - al), epi);
  gb.seg(p, D, 0, 0, W, 1, 0, W.rows);
  p.b_n = al;
  p.acc_col0 = col0 - al;
  return p;
}
// dW[n][k] = sum_m D[m][n] X[m][k]: both operands MN-major (the batch is the reduction).
GProb& dw(GemmBuilder& gb, const Mat& D, const Mat& X, const LinG& G, int nin) {
  GProb& p = gb.add(D.cols, nin, GE_DW);
  gb.seg(p, D, 1, 0, X, 1, 0, D.rows);
  p.outf = G.w;
  p.ldf = nin;
  p.db = G.b;
  p.dg = G.g;
  p.dbeta = G.beta;
  return p;
}
// Launches a weight-gradient batch (every problem from dw(): one MN-major segment over the K = B
// batch rows).  At large batches with few output tiles (c3's actor: ~40 tiles of K = 4096 on 148
// SMs, ~36 us of per-CTA latency-bound streaming) the problems are split over K into kspl copies
// that write fp32 partials (and the ones-column bias partials) into `scratch`; k_split_sum adds
// them in copy order (deterministic).  The LayerNorm-affine / bias partials of part_in are
// K-independent and stay with copy 0.
int dw_launch(GemmBuilder& gb, float* scratch, int64_t cap, cudaStream_t s) {
  const GBatch& b = gb.b;
  int tiles = 0, K = -1;
  bool ok = !gb.err;
  for (int i = 0; i < b.nprob && ok; ++i) {
    const GProb& p = b.p[i];
    const int n16 = (p.N + 15) & ~15, bn = n16 >= 256 ? 64 : (n16 > 128 ? 128 : n16);
    tiles += ((p.N + bn - 1) / bn) * ((p.M + 127) / 128);
    ok = p.nseg == 1 && p.epi == GE_DW && p.a_m == 0 && p.b_n == 0 && p.ldf == p.N && (K < 0 || K == p.seg[0].k);
    K = p.seg[0].k;
  }
  int kspl = 1;
  while (ok && K >= 2048 && kspl < kDwMaxSplit && tiles * kspl * 2 <= 148 && K % (kspl * 2 * 256) == 0 &&
         b.nprob * kspl * 2 <= kGemmMaxProb)
    kspl *= 2;
  int64_t need = 0;
  for (int i = 0; i < b.nprob; ++i) need += (int64_t)kspl * b.p[i].M * ((int64_t)b.p[i].N + (b.p[i].bias_ones ? 1 : 0));
  if (kspl == 1 || need > cap) return gemm_launch(gb, s);
  GemmBuilder g2(b.prefetch_b);
  SplitSumJobs jobs;
  memset(&jobs, 0, sizeof(jobs));
  jobs.nsplit = kspl;
  float* sp = scratch;
  const int kc = K / kspl;
  for (int i = 0; i < b.nprob; ++i) {
    const GProb o = b.p[i];
    const Mat A = gb.segA[i][0], Bm = gb.segB[i][0];
    float* wpart = sp;
    sp += (int64_t)kspl * o.M * o.N;
    float* dbpart = nullptr;
    if (o.bias_ones) {
      dbpart = sp;
      sp += (int64_t)kspl * o.M;
    }
    for (int r = 0; r < kspl; ++r) {
      GProb& p = g2.add(o.M, o.N, GE_DW);
      g2.seg(p, A, 1, o.seg[0].a_k + r * kc, Bm, 1, o.seg[0].b_k + r * kc, kc);
      p.outf = wpart + (int64_t)r * o.M * o.N;
      p.ldf = o.N;
      p.bias_ones = o.bias_ones;
      if (o.bias_ones) {
        p.db = dbpart + (int64_t)r * o.M;
      } else if (r == 0) {
        p.db = o.db;
        p.dg = o.dg;
        p.dbeta = o.dbeta;
        p.part_in = o.part_in;
        p.part_tiles = o.part_tiles;
      }
    }
    if (jobs.njobs + 2 > kMaxSplitJobs) return -1;
    jobs.dst[jobs.njobs] = o.outf;
    jobs.src[jobs.njobs] = wpart;
    jobs.n[jobs.njobs++] = o.M * o.N;
    if (o.bias_ones && o.db) {
      jobs.dst[jobs.njobs] = o.db;
      jobs.src[jobs.njobs] = dbpart;
      jobs.n[jobs.njobs++] = o.M;
    }
  }
  const int e = gemm_launch(g2, s);
  if (e) return e;
  return launch_split_sum(jobs, s);
}

void bwd_ln(GProb& p, const Lin& W, bf16* xh, int ldx, float* rstd, bf16* out, int ldo, float* part, int64_t part_cap) {
  p.g = W.g;
  p.beta = W.beta;
  p.xh = xh;
  p.ldx = ldx;
  p.rstd = rstd;
  p.out = out;
  p.ldo = ldo;
  p.part = part;
  p.part_cap = part_cap;
}

Mat none_mat() { return Mat{nullptr, 0, 0, 0}; }


// a LayerNorm layer (forward) of a fused chain
CLayer& ch_fwd(ChainBuilder& cb, CProb& p, int epi, const Lin& W, int N, int K, const Mat& O, const Mat& X, float* rstd,
               float ln_eps) {
  CLayer& L = cb.layer(p, epi, W.w, 0, N, K, O, X);
  L.bias = W.b;
  L.g = W.g;
  L.beta = W.beta;
  L.rstd = rstd;
  L.ln_eps = ln_eps;
  return L;
}
#define BF_CK(expr)                                                                                     \
  do {                                                                                                  \
    int _e = (int)(expr);                                                                               \
    if (_e != 0)                                                                                        \
      return set_error(SQUINT_ECUDA, std::string("bf16 path: ") + #expr + " failed (" +               \
                                         (_e > 0 ? cudaGetErrorString((cudaError_t)_e) : "plan/map error") + ")"); \
  } while (0)

ShadowTable table_at(const Ctx& c, const ShadowPlan& sp) {
  ShadowTable t = sp.t;
  t.base = reinterpret_cast<bf16*>(c.ws + sp.off);
  return t;
}

// one update's random inputs
struct UpdIn {
  const int64_t* idx;
  const uint8_t* sh;
  const float* eps;
  int rep;
};

// Update j's buffers: the matrices the pipelined forward of update j + 1 writes while update j's
// actor pass still reads them alternate by update parity.
BfLay with_parity(const BfLay& w, int par) {
  BfLay v = w;
  if (par & 1) {
    v.sh[0] = w.sh[3];
    v.sh[3] = w.sh[0];
    v.Xh = w.Xh_alt;
    v.Xq1 = w.Xq1_alt;
    v.Xac = w.Xac_alt;
  }
  return v;
}

// The part of an update's forward that depends only on the critic (theta), the target (theta_bar)
// and the replay rows, not on the actor: gather + shift + encoder (obs and next_obs), the critic
// and target projections and the online heads.  Pipelined (single GPU, chains): issued on the
// auxiliary branch of the previous update, beside its actor pass; enc_ev / chn_ev mark the
// encoder + projections and the online heads.
squint_status early_fwd(const Ctx& c, const BfLay& w_in, const squint_hparams& hp, const squint_replay& R,
                        const UpdIn& u, const squint_state& st, int par, cudaStream_t ss, int enc_ctas,
                        cudaEvent_t enc_ev, cudaEvent_t chn_ev) {
  const BfLay w = with_parity(w_in, par);
  const squint_dims& d = c.d;
  const Layout& L = c.L;
  const int B = d.batch, Lt = d.latent, Hc = d.critic_hidden, N = head_out(d), A = d.action_dim, P = d.proprio_dim,
            C = d.conv_ch;
  const int nq = Lt + P + A;
  const float le = hp.ln_eps;
  const int gC = SQUINT_GROUP_CRITIC, gT = SQUINT_GROUP_TARGET;
  const float* crit = st.critic;
  const float* tgt = st.critic_target;
  const Lin cproj = proj(c, w.sh[0], crit, gC, "critic"), tproj = proj(c, w.sh[1], tgt, gT, "critic");
  const Mlp cq[2] = {mlp(c, w.sh[0], crit, gC, kHeads[0]), mlp(c, w.sh[0], crit, gC, kHeads[1])};
  {
    PhaseScope ps(3, u.rep, ss);
    EncFwdArgs e;
    memset(&e, 0, sizeof(e));
    e.mode = 0;
    e.src[0] = R.obs;
    e.src[1] = R.next_obs;
    e.idx = u.idx;
    e.shifts = u.sh;
    e.B = B;
    e.nsrc = 2;
    e.w1 = crit + L.off(gC, "enc.conv1.w");
    e.b1 = crit + L.off(gC, "enc.conv1.b");
    e.w2 = crit + L.off(gC, "enc.conv2.w");
    e.b2 = crit + L.off(gC, "enc.conv2.b");
    e.hb[0] = c.bp(w.Xh);
    e.hb[1] = c.bp(w.Xhn);
    e.h_ld = w.Xh.ld;
    e.y1b = reinterpret_cast<bf16*>(c.ws + w.y1b);
    e.img0 = reinterpret_cast<uint8_t*>(c.ws + w.img0);
    if (g_dump_next) e.img1 = reinterpret_cast<uint8_t*>(c.ws + w.img1);
    e.C = C;
    e.c_in = d.img_c;
    e.H = d.img_h;
    e.pad = d.pad;
    e.gj[0][0] = GatherJob{R.proprio, P, c.bp(w.Xq), w.Xq.ld, Lt, 1};
    e.gj[0][1] = GatherJob{R.action, A, c.bp(w.Xq), w.Xq.ld, Lt + P, 1};
    e.gj[0][2] = GatherJob{R.proprio, P, c.bp(w.Xac), w.Xac.ld, Lt, 1};
    e.gj[0][3] = GatherJob{R.proprio, P, c.bp(w.Xq1), w.Xq1.ld, Lt, 1};
    e.ngj[0] = 4;
    e.gj[1][0] = GatherJob{R.next_proprio, P, c.bp(w.Xt), w.Xt.ld, Lt, 1};
    e.gj[1][1] = GatherJob{R.next_proprio, P, c.bp(w.Xan), w.Xan.ld, Lt, 1};
    e.ngj[1] = 2;
    e.wtiles = reinterpret_cast<uint8_t*>(c.ws + w.wtiles);
    e.max_ctas = enc_ctas;
    BF_CK(launch_enc_fwd_tc(e, ss));
  }
  {
    PhaseScope ps(4, u.rep, ss);
    GemmBuilder gb(1);
    GProb* p = &fwd(gb, c.mat(w.Xh), cproj, GE_LN_TANH, c.bp(w.Xq), w.Xq.ld, le);
    p->xh = c.bp(w.XHpq), p->ldx = w.XHpq.ld, p->rstd = c.F(w.Rpq);
    fwd(gb, c.mat(w.Xhn), tproj, GE_LN_TANH, c.bp(w.Xt), w.Xt.ld, le);
    BF_CK(gemm_launch(gb, ss));
  }
  if (enc_ev) BF_CK(cudaEventRecord(enc_ev, ss));
  {
    PhaseScope ps(6, u.rep, ss);
    ChainBuilder cb(1);
    for (int i = 0; i < 2; ++i) {
      CProb& p = cb.add(B, c.mat(w.Xq));
      ch_fwd(cb, p, GE_LN_RELU, cq[i].l1, Hc, nq, c.mat(w.qH1[i]), c.mat(w.qXH1[i]), c.F(w.qR1[i]), le);
      ch_fwd(cb, p, GE_LN_RELU, cq[i].l2, Hc, Hc, c.mat(w.qH2[i]), c.mat(w.qXH2[i]), c.F(w.qR2[i]), le);
      CLayer& l3 = cb.layer(p, GE_BIAS_F32, cq[i].l3.w, 0, N, Hc, none_mat(), none_mat());
      l3.bias = cq[i].l3.b;
      l3.outf = c.F(w.logits) + (size_t)i * B * N;
      l3.ldf = N;
    }
    BF_CK(chain_launch(cb, ss));
  }
  if (chn_ev) BF_CK(cudaEventRecord(chn_ev, ss));
  return SQUINT_OK;
}

// ---- f1: peer-memory all-reduce fused with a sharded Adam (comm mode 1) --------------------------
// Cross-rank barrier; with ntail > 0 also the sum over ranks of every rank's `tail` into `out`, and
// with ra != NULL first this rank's row sums (as k_row_sums / k_lpi_sums) into tail[0..1].
squint_status dp_barrier(Comm* cm, const float* tail, float* out, int ntail, cudaStream_t s,
                         const float* ra = nullptr, const float* rb = nullptr, int B = 0) {
  static_assert(kDpMaxRanks == kMaxRanks, "rank bound");
  DpSync a;
  memset(&a, 0, sizeof(a));
  a.G = comm_nranks(cm);
  a.rank = comm_rank(cm);
  void* f[kMaxRanks];
  if (comm_peer_ptrs(cm, comm_flags(cm), f) != 0) return set_error(SQUINT_ENCCL, comm_error());
  for (int q = 0; q < a.G; ++q) a.flag[q] = static_cast<unsigned*>(f[q]);
  a.own = comm_flags(cm);
  if (ntail > 0) {
    if (comm_peer_ptrs(cm, tail, f) != 0) return set_error(SQUINT_ENCCL, comm_error());
    for (int q = 0; q < a.G; ++q) a.tail[q] = static_cast<const float*>(f[q]);
    a.tail_out = out;
    a.ntail = ntail;
    if (ra) {
      a.ra = ra;
      a.rb = rb;
      a.B = B;
      a.tail_mine = const_cast<float*>(tail);
    }
  }
  BF_CK(launch_dp_sync(a, s));
  return SQUINT_OK;
}

// One group's optimizer step in peer mode: this rank's 1/G slice of sum_ranks(g) through Adam,
// stored (fp32 and its bf16 shadow entries) into every rank's copies; barrier.
squint_status dp_adam(Comm* cm, const float* g, float* p, float* m, float* v, int64_t n, float lr,
                      const squint_hparams& hp, const float* c1, const float* c2, float* part, const ShadowTable* t,
                      int grad_perm, cudaStream_t s) {
  DpAdam d;
  memset(&d, 0, sizeof(d));
  d.G = comm_nranks(cm);
  d.rank = comm_rank(cm);
  void* f[kMaxRanks];
  if (comm_peer_ptrs(cm, g, f) != 0) return set_error(SQUINT_ENCCL, comm_error());
  for (int q = 0; q < d.G; ++q) d.g[q] = static_cast<const float*>(f[q]);
  if (comm_peer_ptrs(cm, p, f) != 0) return set_error(SQUINT_ENCCL, comm_error());
  for (int q = 0; q < d.G; ++q) d.p[q] = static_cast<float*>(f[q]);
  if (part) {
    if (comm_peer_ptrs(cm, part, f) != 0) return set_error(SQUINT_ENCCL, comm_error());
    for (int q = 0; q < d.G; ++q) d.part[q] = static_cast<float*>(f[q]);
  }
  if (t && t->n) {
    if (comm_peer_ptrs(cm, t->base, f) != 0) return set_error(SQUINT_ENCCL, comm_error());
    for (int q = 0; q < d.G; ++q) d.sh[q] = static_cast<__nv_bfloat16*>(f[q]);
  }
  const int64_t n4 = n / 4;
  d.lo4 = n4 * d.rank / d.G;
  d.hi4 = n4 * (d.rank + 1) / d.G;
  BF_CK(launch_dp_adam(d, m, v, lr, hp.beta1, hp.beta2, hp.adam_eps, c1, c2, t, grad_perm, s));
  return dp_barrier(cm, nullptr, nullptr, 0, s);
}

// pipe: the early forward of this update already ran (early_fwd); next: the following update's
// inputs (its early forward is issued on this update's branch), NULL for the last update
squint_status update_one(const Ctx& c, const BfLay& w_in, const squint_hparams& hp, const squint_replay& R,
                         const int64_t* idx, const uint8_t* sh, const float* eps, const squint_state& st,
                         float* metrics, Comm* comm, float inv_btotal, int rep, int par, bool pipe,
                         const UpdIn* next) {
  const BfLay w = with_parity(w_in, par);
  const squint_dims& d = c.d;
  const Layout& L = c.L;
  cudaStream_t s = c.s;
  const int B = d.batch, F = flat_dim(d), Lt = d.latent, Hc = d.critic_hidden, Ha = d.actor_hidden, N = head_out(d),
            A = d.action_dim, P = d.proprio_dim, C = d.conv_ch;
  const int nq = Lt + P + A, npi = Lt + P;
  const int P2 = conv2_out(d) * conv2_out(d);
  const float* eps_next = eps;
  const float* eps_cur = eps + (size_t)B * A;
  const float le = hp.ln_eps;
  const int gC = SQUINT_GROUP_CRITIC, gA = SQUINT_GROUP_ACTOR, gT = SQUINT_GROUP_TARGET;
  const float* crit = st.critic;
  const float* tgt = st.critic_target;
  const float* act = st.actor;
  const Lin cproj = proj(c, w.sh[0], crit, gC, "critic"), tproj = proj(c, w.sh[1], tgt, gT, "critic"),
            aproj = proj(c, w.sh[2], act, gA, "actor");
  const Mlp cq[2] = {mlp(c, w.sh[0], crit, gC, kHeads[0]), mlp(c, w.sh[0], crit, gC, kHeads[1])};
  const Mlp tq[2] = {mlp(c, w.sh[1], tgt, gT, kHeads[0]), mlp(c, w.sh[1], tgt, gT, kHeads[1])};
  const Mlp am = mlp(c, w.sh[2], act, gA, "actor");
  const int mt = mtiles(B);

  // a3-a5: gather + shift + encoder (obs, next_obs); replay rows of s, a, s' into the layer
  // input matrices
  uint8_t* wtiles = reinterpret_cast<uint8_t*>(c.ws + w.wtiles);
  // conv weight tiles: with the auxiliary branch they were written at the end of the previous
  // update's branch (or by the call prologue)
  const bool branch = comm == nullptr && c.aux != nullptr;
  const bool dp_peer = comm && comm_mode(comm) == 1;
  if (!branch) BF_CK(launch_conv_tiles(crit + L.off(gC, "enc.conv1.w"), crit + L.off(gC, "enc.conv2.w"), C, wtiles, s));
  if (pipe) {
    // encoder, critic/target projections and online heads came from early_fwd (on the previous
    // update's branch, or the call prologue): the actor projections need the encoder output
    BF_CK(cudaStreamWaitEvent(s, c.aux->enc, 0));
    PhaseScope ps(4, rep, s);
    GemmBuilder gb(1);
    fwd(gb, c.mat(w.Xhn), aproj, GE_LN_TANH, c.bp(w.Xan), w.Xan.ld, le);
    GProb& p = fwd(gb, c.mat(w.Xh), aproj, GE_LN_TANH, c.bp(w.Xac), w.Xac.ld, le);
    p.xh = c.bp(w.XHpp), p.ldx = w.XHpp.ld, p.rstd = c.F(w.Rpp);
    BF_CK(gemm_launch(gb, s));
  }
  if (!pipe) {
    PhaseScope ps(3, rep, s);
    EncFwdArgs e;
    memset(&e, 0, sizeof(e));
    e.mode = 0;
    e.src[0] = R.obs;
    e.src[1] = R.next_obs;
    e.idx = idx;
    e.shifts = sh;
    e.B = B;
    e.nsrc = 2;
    e.w1 = crit + L.off(gC, "enc.conv1.w");
    e.b1 = crit + L.off(gC, "enc.conv1.b");
    e.w2 = crit + L.off(gC, "enc.conv2.w");
    e.b2 = crit + L.off(gC, "enc.conv2.b");
    e.hb[0] = c.bp(w.Xh);
    e.hb[1] = c.bp(w.Xhn);
    e.h_ld = w.Xh.ld;
    e.y1b = reinterpret_cast<bf16*>(c.ws + w.y1b);
    e.img0 = reinterpret_cast<uint8_t*>(c.ws + w.img0);
    if (g_dump_next) e.img1 = reinterpret_cast<uint8_t*>(c.ws + w.img1);
    e.C = C;
    e.c_in = d.img_c;
    e.H = d.img_h;
    e.pad = d.pad;
    e.gj[0][0] = GatherJob{R.proprio, P, c.bp(w.Xq), w.Xq.ld, Lt, 1};
    e.gj[0][1] = GatherJob{R.action, A, c.bp(w.Xq), w.Xq.ld, Lt + P, 1};
    e.gj[0][2] = GatherJob{R.proprio, P, c.bp(w.Xac), w.Xac.ld, Lt, 1};
    e.gj[0][3] = GatherJob{R.proprio, P, c.bp(w.Xq1), w.Xq1.ld, Lt, 1};
    e.ngj[0] = 4;
    e.gj[1][0] = GatherJob{R.next_proprio, P, c.bp(w.Xt), w.Xt.ld, Lt, 1};
    e.gj[1][1] = GatherJob{R.next_proprio, P, c.bp(w.Xan), w.Xan.ld, Lt, 1};
    e.ngj[1] = 2;
    e.wtiles = wtiles;
    BF_CK(launch_enc_fwd_tc(e, s));
  }
  // a6: projections Linear -> LN -> tanh (Q8): critic(h), target(h'), actor(h'), actor(h)
  if (!pipe) {
    PhaseScope ps(4, rep, s);
    GemmBuilder gb(1);
    GProb* p = &fwd(gb, c.mat(w.Xh), cproj, GE_LN_TANH, c.bp(w.Xq), w.Xq.ld, le);
    p->xh = c.bp(w.XHpq), p->ldx = w.XHpq.ld, p->rstd = c.F(w.Rpq);
    fwd(gb, c.mat(w.Xhn), tproj, GE_LN_TANH, c.bp(w.Xt), w.Xt.ld, le);
    fwd(gb, c.mat(w.Xhn), aproj, GE_LN_TANH, c.bp(w.Xan), w.Xan.ld, le);
    p = &fwd(gb, c.mat(w.Xh), aproj, GE_LN_TANH, c.bp(w.Xac), w.Xac.ld, le);
    p->xh = c.bp(w.XHpp), p->ldx = w.XHpp.ld, p->rstd = c.F(w.Rpp);
    BF_CK(gemm_launch(gb, s));
  }
  // a7: actor MLP on s' (target sample) and on s (alpha / actor losses)
  if (c.chain) {
    PhaseScope ps(5, rep, s);
    ChainBuilder cb(1);
    cb.xscr = c.ws + w.xchg;
    cb.xcap = w.xchg_bytes;
    CProb& pn = cb.add(B, c.mat(w.Xan));
    ch_fwd(cb, pn, GE_LN_RELU, am.l1, Ha, npi, none_mat(), none_mat(), nullptr, le);
    ch_fwd(cb, pn, GE_LN_RELU, am.l2, Ha, Ha, none_mat(), none_mat(), nullptr, le);
    CLayer& tn = cb.layer(pn, GE_TG_FWD, am.l3.w, 0, 2 * A, Ha, none_mat(), none_mat());
    tn.bias = am.l3.b;
    tn.eps = eps_next;
    tn.act_bf = c.bp(w.Xt) + Lt + P;
    tn.ld_act_bf = w.Xt.ld;
    tn.logp = c.F(w.logp_next);
    tn.lo = hp.log_std_min;
    tn.hi = hp.log_std_max;
    CProb& pc = cb.add(B, c.mat(w.Xac));
    ch_fwd(cb, pc, GE_LN_RELU, am.l1, Ha, npi, c.mat(w.H1ac), c.mat(w.XH1ac), c.F(w.R1ac), le);
    ch_fwd(cb, pc, GE_LN_RELU, am.l2, Ha, Ha, c.mat(w.H2ac), c.mat(w.XH2ac), c.F(w.R2ac), le);
    CLayer& tc_ = cb.layer(pc, GE_TG_FWD, am.l3.w, 0, 2 * A, Ha, none_mat(), none_mat());
    tc_.bias = am.l3.b;
    tc_.eps = eps_cur;
    tc_.act = c.F(w.a_cur);
    tc_.act_bf = c.bp(w.Xq1) + Lt + P;
    tc_.ld_act_bf = w.Xq1.ld;
    tc_.logp = c.F(w.logp_cur);
    tc_.tgo = c.F(w.tgo_ac);
    tc_.lo = hp.log_std_min;
    tc_.hi = hp.log_std_max;
    BF_CK(chain_launch(cb, s));
  } else {
    PhaseScope ps(5, rep, s);
    {
      GemmBuilder gb(1);
      fwd(gb, c.mat(w.Xan), am.l1, GE_LN_RELU, c.bp(w.H1an), w.H1an.ld, le);
      GProb& p = fwd(gb, c.mat(w.Xac), am.l1, GE_LN_RELU, c.bp(w.H1ac), w.H1ac.ld, le);
      p.xh = c.bp(w.XH1ac), p.ldx = w.XH1ac.ld, p.rstd = c.F(w.R1ac);
      BF_CK(gemm_launch(gb, s));
    }
    {
      GemmBuilder gb(1);
      fwd(gb, c.mat(w.H1an), am.l2, GE_LN_RELU, c.bp(w.H2an), w.H2an.ld, le);
      GProb& p = fwd(gb, c.mat(w.H1ac), am.l2, GE_LN_RELU, c.bp(w.H2ac), w.H2ac.ld, le);
      p.xh = c.bp(w.XH2ac), p.ldx = w.XH2ac.ld, p.rstd = c.F(w.R2ac);
      BF_CK(gemm_launch(gb, s));
    }
    {
      GemmBuilder gb(1);
      GProb& pn = fwd(gb, c.mat(w.H2an), am.l3, GE_TG_FWD, nullptr, 0, le);
      pn.eps = eps_next;
      pn.act_bf = c.bp(w.Xt) + Lt + P;
      pn.ld_act_bf = w.Xt.ld;
      pn.logp = c.F(w.logp_next);
      pn.lo = hp.log_std_min;
      pn.hi = hp.log_std_max;
      GProb& pc = fwd(gb, c.mat(w.H2ac), am.l3, GE_TG_FWD, nullptr, 0, le);
      pc.eps = eps_cur;
      pc.act = c.F(w.a_cur);
      pc.act_bf = c.bp(w.Xq1) + Lt + P;
      pc.ld_act_bf = w.Xq1.ld;
      pc.logp = c.F(w.logp_cur);
      pc.tgo = c.F(w.tgo_ac);
      pc.lo = hp.log_std_min;
      pc.hi = hp.log_std_max;
      BF_CK(gemm_launch(gb, s));
    }
  }
  // a8: target heads on (z', s', a~') and online heads on (z, s, a)
  if (c.chain) {
    PhaseScope ps(6, rep, s);
    ChainBuilder cb(1);
    cb.xscr = c.ws + w.xchg;
    cb.xcap = w.xchg_bytes;
    for (int i = 0; i < 2; ++i) {
      CProb& p = cb.add(B, c.mat(w.Xt));
      ch_fwd(cb, p, GE_LN_RELU, tq[i].l1, Hc, nq, none_mat(), none_mat(), nullptr, le);
      ch_fwd(cb, p, GE_LN_RELU, tq[i].l2, Hc, Hc, none_mat(), none_mat(), nullptr, le);
      CLayer& l3 = cb.layer(p, GE_BIAS_F32, tq[i].l3.w, 0, N, Hc, none_mat(), none_mat());
      l3.bias = tq[i].l3.b;
      l3.outf = c.F(w.tlogits) + (size_t)i * B * N;
      l3.ldf = N;
    }
    for (int i = 0; i < 2 && !pipe; ++i) {
      CProb& p = cb.add(B, c.mat(w.Xq));
      ch_fwd(cb, p, GE_LN_RELU, cq[i].l1, Hc, nq, c.mat(w.qH1[i]), c.mat(w.qXH1[i]), c.F(w.qR1[i]), le);
      ch_fwd(cb, p, GE_LN_RELU, cq[i].l2, Hc, Hc, c.mat(w.qH2[i]), c.mat(w.qXH2[i]), c.F(w.qR2[i]), le);
      CLayer& l3 = cb.layer(p, GE_BIAS_F32, cq[i].l3.w, 0, N, Hc, none_mat(), none_mat());
      l3.bias = cq[i].l3.b;
      l3.outf = c.F(w.logits) + (size_t)i * B * N;
      l3.ldf = N;
    }
    BF_CK(chain_launch(cb, s));
    if (pipe) BF_CK(cudaStreamWaitEvent(s, c.aux->chn, 0));  // online logits (early_fwd)
  } else {
    PhaseScope ps(6, rep, s);
    {
      GemmBuilder gb(1);
      for (int i = 0; i < 2; ++i) fwd(gb, c.mat(w.Xt), tq[i].l1, GE_LN_RELU, c.bp(w.tqH1[i]), w.tqH1[i].ld, le);
      for (int i = 0; i < 2; ++i) {
        GProb& p = fwd(gb, c.mat(w.Xq), cq[i].l1, GE_LN_RELU, c.bp(w.qH1[i]), w.qH1[i].ld, le);
        p.xh = c.bp(w.qXH1[i]), p.ldx = w.qXH1[i].ld, p.rstd = c.F(w.qR1[i]);
      }
      BF_CK(gemm_launch(gb, s));
    }
    {
      GemmBuilder gb(1);
      for (int i = 0; i < 2; ++i)
        fwd(gb, c.mat(w.tqH1[i]), tq[i].l2, GE_LN_RELU, c.bp(w.tqH2[i]), w.tqH2[i].ld, le);
      for (int i = 0; i < 2; ++i) {
        GProb& p = fwd(gb, c.mat(w.qH1[i]), cq[i].l2, GE_LN_RELU, c.bp(w.qH2[i]), w.qH2[i].ld, le);
        p.xh = c.bp(w.qXH2[i]), p.ldx = w.qXH2[i].ld, p.rstd = c.F(w.qR2[i]);
      }
      BF_CK(gemm_launch(gb, s));
    }
    {
      GemmBuilder gb(1);
      for (int i = 0; i < 2; ++i) {
        GProb& p = fwd(gb, c.mat(w.tqH2[i]), tq[i].l3, GE_BIAS_F32, nullptr, 0, le);
        p.outf = c.F(w.tlogits) + (size_t)i * B * N;
        p.ldf = N;
      }
      for (int i = 0; i < 2; ++i) {
        GProb& p = fwd(gb, c.mat(w.qH2[i]), cq[i].l3, GE_BIAS_F32, nullptr, 0, le);
        p.outf = c.F(w.logits) + (size_t)i * B * N;
        p.ldf = N;
      }
      BF_CK(gemm_launch(gb, s));
    }
  }
  // a9-a10: target distribution, categorical projection, CE, dL/dlogits
  {
    PhaseScope ps(7, rep, s);
    TargetCEArgs t;
    memset(&t, 0, sizeof(t));
    t.B = B;
    t.N = N;
    t.v_min = d.v_min;
    t.v_max = d.v_max;
    t.gamma = hp.gamma;
    t.cdq = hp.target_mode == SQUINT_TARGET_CDQ;
    t.mse = d.critic_kind == SQUINT_CRITIC_MSE;
    t.scale = inv_btotal;
    t.tlogits = c.F(w.tlogits);
    t.logits = c.F(w.logits);
    t.idx = idx;
    t.reward = R.reward;
    t.done = R.done;
    t.logp_next = c.F(w.logp_next);
    t.log_alpha = st.log_alpha;
    t.m = c.F(w.m);
    t.dlogits_bf = c.bp(w.dlog);
    t.ld_dl = w.dlog.ld;
    t.row_loss = c.F(w.row_loss);
    // the critic / actor Adam steps and bias corrections (the alpha step runs later)
    t.step = st.step;
    t.scal = c.F(w.scal);
    t.beta1 = hp.beta1;
    t.beta2 = hp.beta2;
    BF_CK(launch_target_ce(t, s));
  }
  // a10: critic backward: heads -> critic projection -> ReLU'(conv2)
  float* gc = c.F(w.grad_critic);
  int ks_pq = 1, ks_pp = 1;
  {
    PhaseScope ps(8, rep, s);
    {
      GemmBuilder gb(1);
      for (int i = 0; i < 2; ++i) {
        GProb& p = dx(gb, c.half(w.dlog, i), cq[i].l3.w, 0, Hc, GE_BWD_LN_RELU);
        bwd_ln(p, cq[i].l2, c.bp(w.qXH2[i]), w.qXH2[i].ld, c.F(w.qR2[i]), c.bp(w.dA2c[i]), w.dA2c[i].ld,
               c.F(w.part_q2[i]), w.part_q2[i].n);
      }
      BF_CK(gemm_launch(gb, s));
    }
    {
      GemmBuilder gb(1);
      for (int i = 0; i < 2; ++i) {
        GProb& p = dx(gb, c.mat(w.dA2c[i]), cq[i].l2.w, 0, Hc, GE_BWD_LN_RELU);
        bwd_ln(p, cq[i].l1, c.bp(w.qXH1[i]), w.qXH1[i].ld, c.F(w.qR1[i]), c.bp(w.dA1c[i]), w.dA1c[i].ld,
               c.F(w.part_q1[i]), w.part_q1[i].n);
      }
      BF_CK(gemm_launch(gb, s));
    }
    {
      // dz = sum_i dA1_i W1_i[:, :L] (K-concatenation of the two heads) -> tanh + LN of the projection
      GemmBuilder gb(1);
      GProb& p = dx(gb, c.mat(w.dA1c[0]), cq[0].l1.w, 0, Lt, GE_BWD_LN_TANH);
      gb.seg(p, c.mat(w.dA1c[1]), 0, 0, cq[1].l1.w, 1, 0, Hc);
      bwd_ln(p, cproj, c.bp(w.XHpq), w.XHpq.ld, c.F(w.Rpq), c.bp(w.dAp), w.dAp.ld, c.F(w.part_pq), w.part_pq.n);
      BF_CK(gemm_launch(gb, s));
      ks_pq = gb.b.ks;  // split-K launch: column partials per 128 / ks rows
    }
  }
  // encoder backward (dh GEMM + conv backward): on the auxiliary branch when single-GPU
  // (overlaps the critic dW GEMM and the actor-loss chain), inline when the gradients are
  // all-reduced
  cudaStream_t es = branch ? c.aux->s : s;
  // pipelined: the previous update's branch (its metrics and this update's early forward) must
  // be done before this update's weight gradients and Adam overwrite what it reads
  if (pipe && rep > 0) BF_CK(cudaStreamWaitEvent(s, c.aux->join, 0));
  float* extras = gc + L.gsize[gC];
  float* scal = c.F(w.scal);
  auto scalars = [&](cudaStream_t ss) -> squint_status {
    // a11 temperature step (Q17) from the row sums
    ScalarsArgs a;
    memset(&a, 0, sizeof(a));
    a.B = B;
    a.inv_btotal = inv_btotal;
    a.logp = c.F(w.logp_cur);
    a.row_loss = c.F(w.row_loss);
    a.extras = extras;
    a.compute_sums = comm ? 0 : 1;
    a.log_alpha = st.log_alpha;
    a.m_alpha = st.m_alpha;
    a.v_alpha = st.v_alpha;
    a.step = st.step;
    a.lr_alpha = hp.lr_alpha;
    a.beta1 = hp.beta1;
    a.beta2 = hp.beta2;
    a.adam_eps = hp.adam_eps;
    a.target_entropy = hp.target_entropy;
    a.loss_scale = inv_btotal;
    a.scal = scal;
    a.steps_done = 1;
    BF_CK(launch_scalars(a, ss));
    return SQUINT_OK;
  };
  if (branch) {
    BF_CK(cudaEventRecord(c.aux->fork, s));
    BF_CK(cudaStreamWaitEvent(es, c.aux->fork, 0));
    // the alpha step first on the branch: only the actor loss (k_actor_q) waits for it
    squint_status r = scalars(es);
    if (r != SQUINT_OK) return r;
    BF_CK(cudaEventRecord(c.aux->alpha, es));
  }
  {
    // dh = dAp Wp, masked by ReLU'(conv2) (h > 0), HWC
    PhaseScope ps(8, rep, es);
    GemmBuilder gb(1);
    GProb& p = dx(gb, c.mat(w.dAp), cproj.w, 0, F, GE_RELU_MASK);
    p.y = c.bp(w.Xh);
    p.ldy = w.Xh.ld;
    p.out = c.bp(w.dh);
    p.ldo = w.dh.ld;
    BF_CK(gemm_launch(gb, es));
  }
  {
    PhaseScope ps(10, rep, es);
    EncBwdArgs e;
    memset(&e, 0, sizeof(e));
    e.B = B;
    e.C = C;
    e.c_in = d.img_c;
    e.H = d.img_h;
    e.dA2_hwc = c.bp(w.dh);
    e.dA2_ld = w.dh.ld;
    e.y1_hwc = reinterpret_cast<const bf16*>(c.ws + w.y1b);
    e.img = reinterpret_cast<const uint8_t*>(c.ws + w.img0);
    e.w2 = crit + L.off(gC, "enc.conv2.w");
    e.part = c.F(w.enc_part);
    e.wtiles = wtiles;
    e.gw1 = gc + L.off(gC, "enc.conv1.w");
    e.gb1 = gc + L.off(gC, "enc.conv1.b");
    e.gw2 = gc + L.off(gC, "enc.conv2.w");
    e.gb2 = gc + L.off(gC, "enc.conv2.b");
    // on the branch, leave SMs to the critic dW GEMM and the actor-loss launches beside it at the
    // c2 batch (swept: 80 of 148 best at B = 512); at large batches (c3 on one GPU, B = 4096) the
    // branch is the longer path and takes every SM (148: +15 % updates/s over 80)
    const int bwd_ctas = B <= 1024 ? 80 : 148;
    e.max_ctas = branch ? bwd_ctas : 0;
    BF_CK(launch_enc_bwd_tc(e, es));
  }
  {
    PhaseScope ps(9, rep, s);
    GemmBuilder gb(1);
    for (int i = 0; i < 2; ++i) {
      const std::string hp_ = kHeads[i];
      GProb& p3 = dw(gb, c.half(w.dlog, i), c.mat(w.qH2[i]), ling(L, gc, gC, hp_ + ".l3", ""), Hc);
      p3.bias_ones = 1;
      GProb& p2 = dw(gb, c.mat(w.dA2c[i]), c.mat(w.qH1[i]), ling(L, gc, gC, hp_ + ".l2", hp_ + ".ln2"), Hc);
      p2.part_in = c.F(w.part_q2[i]);
      p2.part_tiles = mt;
      GProb& p1 = dw(gb, c.mat(w.dA1c[i]), c.mat(w.Xq), ling(L, gc, gC, hp_ + ".l1", hp_ + ".ln1"), nq);
      p1.part_in = c.F(w.part_q1[i]);
      p1.part_tiles = mt;
    }
    GProb& pp = dw(gb, c.mat(w.dAp), c.mat(w.Xh), ling(L, gc, gC, "critic.proj", "critic.proj.ln"), F);
    pp.part_in = c.F(w.part_pq);
    pp.part_tiles = mt * ks_pq;
    BF_CK(dw_launch(gb, c.F(w.dwsplit), w.dwsplit.n, s));
  }
  if (comm) {
    if (dp_peer) {
      // the gradients stay where they are: every rank's Adam slice reads them from the peers
      squint_status r = dp_barrier(comm, extras, c.F(w.dp_tail), kExtra, s, c.F(w.logp_cur), c.F(w.row_loss), B);
      if (r != SQUINT_OK) return r;
      extras = c.F(w.dp_tail);
    } else {
      BF_CK(launch_row_sums(c.F(w.logp_cur), c.F(w.row_loss), B, extras, s));
      if (comm_allreduce_sum(comm, gc, L.gsize[gC] + kExtra, s) != 0) return set_error(SQUINT_ENCCL, comm_error());
    }
  }
  // the critic Adam writes theta+ into the other critic shadow set (read by the actor pass below and by
  // the next update); theta's set stays intact for the branch
  const ShadowTable shC = table_at(c, w.sh[3]), shT = table_at(c, w.sh[1]), shA = table_at(c, w.sh[2]);
  // a11 temperature step + Adam bias corrections; a13 Adam on the critic group (+ shadow)
  {
    PhaseScope ps(11, rep, s);
    if (!branch) {
      squint_status r = scalars(s);
      if (r != SQUINT_OK) return r;
    }
    if (branch) {
      // heads + projection on the main stream (the actor loss needs theta+ of those only), the
      // encoder slice on the branch once its gradient is reduced
      const int64_t e0 = L.enc_end;
      BF_CK(launch_adam_shadow(st.critic + e0, gc + e0, st.m_critic + e0, st.v_critic + e0, L.gsize[gC] - e0,
                               hp.lr_critic, hp.beta1, hp.beta2, hp.adam_eps, scal + S_C1_CRITIC, scal + S_C2_CRITIC,
                               c.F(w.adam_part), &shC, s, e0, kAdamBlocks, 1));
      BF_CK(cudaEventRecord(c.aux->scal, s));
      BF_CK(cudaStreamWaitEvent(es, c.aux->scal, 0));
      BF_CK(launch_adam_shadow(st.critic, gc, st.m_critic, st.v_critic, e0, hp.lr_critic, hp.beta1, hp.beta2,
                               hp.adam_eps, scal + S_C1_CRITIC, scal + S_C2_CRITIC, c.F(w.adam_part) + kAdamBlocks,
                               nullptr, es, 0, kEncAdamBlocks));
      // a14 Polyak (needs only theta+ of the heads and projection) and the next update's conv
      // weight tiles (needs the stepped encoder) on the branch as well
      BF_CK(launch_polyak_shadow(st.critic_target, st.critic + L.enc_end, L.gsize[gT], hp.tau, &shT, es));
      BF_CK(launch_conv_tiles(crit + L.off(gC, "enc.conv1.w"), crit + L.off(gC, "enc.conv2.w"), C, wtiles, es));
      if (pipe && next) {
        // the next update's critic-side forward, beside this update's actor pass (encoder grid
        // capped so the main stream's launches keep SMs)
        squint_status r = early_fwd(c, w_in, hp, R, *next, st, par ^ 1, es, 74, c.aux->enc, c.aux->chn);
        if (r != SQUINT_OK) return r;
      }
    } else if (dp_peer) {
      squint_status r = dp_adam(comm, gc, st.critic, st.m_critic, st.v_critic, L.gsize[gC], hp.lr_critic, hp,
                                scal + S_C1_CRITIC, scal + S_C2_CRITIC, c.F(w.adam_part), &shC, 1, s);
      if (r != SQUINT_OK) return r;
    } else {
      BF_CK(launch_adam_shadow(st.critic, gc, st.m_critic, st.v_critic, L.gsize[gC], hp.lr_critic, hp.beta1,
                               hp.beta2, hp.adam_eps, scal + S_C1_CRITIC, scal + S_C2_CRITIC, c.F(w.adam_part), &shC,
                               s, 0, kAdamBlocks, 1));
    }
  }
  // a12: actor loss against theta+ on sg(h) (Q19)
  {
    PhaseScope ps(12, rep, s);
    const Lin cproj1 = proj(c, w.sh[3], crit, gC, "critic");  // theta+ (the other shadow set)
    const Mlp cq1[2] = {mlp(c, w.sh[3], crit, gC, kHeads[0]), mlp(c, w.sh[3], crit, gC, kHeads[1])};
    {
      GemmBuilder gb(0);  // theta+ shadow was written by the immediately preceding Adam kernel
      GProb& p = fwd(gb, c.mat(w.Xh), cproj1, GE_LN_TANH, c.bp(w.Xq1), w.Xq1.ld, le);
      p.xh = c.bp(w.XHpq1), p.ldx = w.XHpq1.ld, p.rstd = c.F(w.Rpq1);
      BF_CK(gemm_launch(gb, s));
    }
    if (c.chain) {
      ChainBuilder cb(1);
      cb.xscr = c.ws + w.xchg;
      cb.xcap = w.xchg_bytes;
      for (int i = 0; i < 2; ++i) {
        CProb& p = cb.add(B, c.mat(w.Xq1));
        ch_fwd(cb, p, GE_LN_RELU, cq1[i].l1, Hc, nq, none_mat(), c.mat(w.q1XH1[i]), c.F(w.q1R1[i]), le);
        ch_fwd(cb, p, GE_LN_RELU, cq1[i].l2, Hc, Hc, none_mat(), c.mat(w.q1XH2[i]), c.F(w.q1R2[i]), le);
        CLayer& l3 = cb.layer(p, GE_BIAS_F32, cq1[i].l3.w, 0, N, Hc, none_mat(), none_mat());
        l3.bias = cq1[i].l3.b;
        l3.outf = c.F(w.logits1) + (size_t)i * B * N;
        l3.ldf = N;
      }
      BF_CK(chain_launch(cb, s));
    } else {
    {
      GemmBuilder gb(1);
      for (int i = 0; i < 2; ++i) {
        GProb& p = fwd(gb, c.mat(w.Xq1), cq1[i].l1, GE_LN_RELU, c.bp(w.q1H1[i]), w.q1H1[i].ld, le);
        p.xh = c.bp(w.q1XH1[i]), p.ldx = w.q1XH1[i].ld, p.rstd = c.F(w.q1R1[i]);
      }
      BF_CK(gemm_launch(gb, s));
    }
    {
      GemmBuilder gb(1);
      for (int i = 0; i < 2; ++i) {
        GProb& p = fwd(gb, c.mat(w.q1H1[i]), cq1[i].l2, GE_LN_RELU, c.bp(w.q1H2[i]), w.q1H2[i].ld, le);
        p.xh = c.bp(w.q1XH2[i]), p.ldx = w.q1XH2[i].ld, p.rstd = c.F(w.q1R2[i]);
      }
      BF_CK(gemm_launch(gb, s));
    }
    {
      GemmBuilder gb(1);
      for (int i = 0; i < 2; ++i) {
        GProb& p = fwd(gb, c.mat(w.q1H2[i]), cq1[i].l3, GE_BIAS_F32, nullptr, 0, le);
        p.outf = c.F(w.logits1) + (size_t)i * B * N;
        p.ldf = N;
      }
      BF_CK(gemm_launch(gb, s));
    }
    }
    ActorQArgs q;
    memset(&q, 0, sizeof(q));
    q.mse = d.critic_kind == SQUINT_CRITIC_MSE;
    q.B = B;
    q.N = N;
    q.v_min = d.v_min;
    q.v_max = d.v_max;
    q.scale = inv_btotal;
    q.logits = c.F(w.logits1);
    q.logp = c.F(w.logp_cur);
    q.alpha1 = scal + S_ALPHA1;
    q.dlogits_bf = c.bp(w.dlog1);
    q.ld_dl = w.dlog1.ld;
    q.row_q = c.F(w.row_q);
    q.row_lpi = c.F(w.row_lpi);
    if (branch) BF_CK(cudaStreamWaitEvent(s, c.aux->alpha, 0));  // alpha+ from the branch
    BF_CK(launch_actor_q(q, s));
    if (branch) BF_CK(cudaEventRecord(c.aux->qdone, s));  // the metrics run on the branch
  }
  {
    PhaseScope ps(13, rep, s);
    const Lin cproj1 = proj(c, w.sh[3], crit, gC, "critic");
    const Mlp cq1[2] = {mlp(c, w.sh[3], crit, gC, kHeads[0]), mlp(c, w.sh[3], crit, gC, kHeads[1])};
    (void)cproj1;
    {
      GemmBuilder gb(1);
      for (int i = 0; i < 2; ++i) {
        GProb& p = dx(gb, c.half(w.dlog1, i), cq1[i].l3.w, 0, Hc, GE_BWD_LN_RELU);
        bwd_ln(p, cq1[i].l2, c.bp(w.q1XH2[i]), w.q1XH2[i].ld, c.F(w.q1R2[i]), c.bp(w.dA2a[i]), w.dA2a[i].ld,
               nullptr, 0);
      }
      BF_CK(gemm_launch(gb, s));
    }
    {
      GemmBuilder gb(1);
      for (int i = 0; i < 2; ++i) {
        GProb& p = dx(gb, c.mat(w.dA2a[i]), cq1[i].l2.w, 0, Hc, GE_BWD_LN_RELU);
        bwd_ln(p, cq1[i].l1, c.bp(w.q1XH1[i]), w.q1XH1[i].ld, c.F(w.q1R1[i]), c.bp(w.dA1a[i]), w.dA1a[i].ld,
               nullptr, 0);
      }
      BF_CK(gemm_launch(gb, s));
    }
    {
      // dL/da~ = sum_i dA1_i W1_i[:, L+P : L+P+A] -> tanh-Gaussian backward (+ the log pi path)
      GemmBuilder gb(1);
      GProb& p = dx(gb, c.mat(w.dA1a[0]), cq1[0].l1.w, Lt + P, A, GE_TG_BWD);
      gb.seg(p, c.mat(w.dA1a[1]), 0, 0, cq1[1].l1.w, 1, 0, Hc);
      p.tgo = c.F(w.tgo_ac);
      p.eps = eps_cur;
      p.dlogp_scale = scal + S_ALPHA1_SCALE;
      p.lo = hp.log_std_min;
      p.hi = hp.log_std_max;
      p.out = c.bp(w.dO);
      p.ldo = w.dO.ld;
      BF_CK(gemm_launch(gb, s));
    }
    {
      GemmBuilder gb(1);
      GProb& p = dx(gb, c.mat(w.dO), am.l3.w, 0, Ha, GE_BWD_LN_RELU);
      bwd_ln(p, am.l2, c.bp(w.XH2ac), w.XH2ac.ld, c.F(w.R2ac), c.bp(w.adA2), w.adA2.ld, c.F(w.part_a2), w.part_a2.n);
      BF_CK(gemm_launch(gb, s));
    }
    {
      GemmBuilder gb(1);
      GProb& p = dx(gb, c.mat(w.adA2), am.l2.w, 0, Ha, GE_BWD_LN_RELU);
      bwd_ln(p, am.l1, c.bp(w.XH1ac), w.XH1ac.ld, c.F(w.R1ac), c.bp(w.adA1), w.adA1.ld, c.F(w.part_a1), w.part_a1.n);
      BF_CK(gemm_launch(gb, s));
    }
    {
      GemmBuilder gb(1);
      GProb& p = dx(gb, c.mat(w.adA1), am.l1.w, 0, Lt, GE_BWD_LN_TANH);
      bwd_ln(p, aproj, c.bp(w.XHpp), w.XHpp.ld, c.F(w.Rpp), c.bp(w.adAp), w.adAp.ld, c.F(w.part_pp), w.part_pp.n);
      BF_CK(gemm_launch(gb, s));
      ks_pp = gb.b.ks;
    }
  }
  float* ga = c.F(w.grad_actor);
  {
    PhaseScope ps(14, rep, s);
    GemmBuilder gb(1);
    GProb& p3 = dw(gb, c.mat(w.dO), c.mat(w.H2ac), ling(L, ga, gA, "actor.l3", ""), Ha);
    p3.bias_ones = 1;
    GProb& p2 = dw(gb, c.mat(w.adA2), c.mat(w.H1ac), ling(L, ga, gA, "actor.l2", "actor.ln2"), Ha);
    p2.part_in = c.F(w.part_a2);
    p2.part_tiles = mt;
    GProb& p1 = dw(gb, c.mat(w.adA1), c.mat(w.Xac), ling(L, ga, gA, "actor.l1", "actor.ln1"), npi);
    p1.part_in = c.F(w.part_a1);
    p1.part_tiles = mt;
    GProb& pp = dw(gb, c.mat(w.adAp), c.mat(w.Xh), ling(L, ga, gA, "actor.proj", "actor.proj.ln"), F);
    pp.part_in = c.F(w.part_pp);
    pp.part_tiles = mt * ks_pp;
    BF_CK(dw_launch(gb, c.F(w.dwsplit), w.dwsplit.n, s));
  }
  float* lpis = c.F(w.lpi_sums);
  PhaseScope ps15(15, rep, s);
  if (comm) {
    float* ax = ga + L.gsize[gA];
    if (dp_peer) {
      squint_status r = dp_barrier(comm, ax, c.F(w.dp_tail) + kExtra, kExtra, s, c.F(w.row_lpi), c.F(w.row_q), B);
      if (r != SQUINT_OK) return r;
      lpis = c.F(w.dp_tail) + kExtra;
    } else {
      BF_CK(launch_lpi_sums(c.F(w.row_lpi), c.F(w.row_q), B, ax, s));
      if (comm_allreduce_sum(comm, ga, L.gsize[gA] + kExtra, s) != 0) return set_error(SQUINT_ENCCL, comm_error());
      lpis = ax;
    }
  }
  if (dp_peer) {
    squint_status r = dp_adam(comm, ga, st.actor, st.m_actor, st.v_actor, L.gsize[gA], hp.lr_actor, hp,
                              scal + S_C1_ACTOR, scal + S_C2_ACTOR, nullptr, &shA, 1, s);
    if (r != SQUINT_OK) return r;
  } else {
    BF_CK(launch_adam_shadow(st.actor, ga, st.m_actor, st.v_actor, L.gsize[gA], hp.lr_actor, hp.beta1, hp.beta2,
                             hp.adam_eps, scal + S_C1_ACTOR, scal + S_C2_ACTOR, nullptr, &shA, s, 0, kAdamBlocks, 1));
  }
  // a14: Polyak over every critic tensor except the encoder (+ target shadow)
  if (!branch) BF_CK(launch_polyak_shadow(st.critic_target, st.critic + L.enc_end, L.gsize[gT], hp.tau, &shT, s));
  {
    // metrics need the alpha step, all critic Adam partials and the actor-loss rows: on the
    // branch (after k_actor_q) they stay off the main stream's actor backward
    cudaStream_t ms = branch ? es : s;
    if (branch) BF_CK(cudaStreamWaitEvent(es, c.aux->qdone, 0));
    MetricsArgs m;
    memset(&m, 0, sizeof(m));
    m.npart = branch ? kAdamBlocks + kEncAdamBlocks : dp_peer ? comm_nranks(comm) * kAdamBlocks : kAdamBlocks;
    m.B = B;
    m.inv_btotal = inv_btotal;
    m.row_lpi = c.F(w.row_lpi);
    m.row_q = c.F(w.row_q);
    m.sumsq_part = c.F(w.adam_part);
    m.scal = scal;
    m.extras = extras;
    m.out = metrics;
    m.reduce_local = comm ? 0 : 1;
    m.extras2 = lpis;
    BF_CK(launch_metrics(m, ms));
    if (branch) {
      BF_CK(cudaEventRecord(c.aux->join, es));
      // join the branch now, or (pipelined, not the last update) in the next update before its fork
      if (!pipe || !next) BF_CK(cudaStreamWaitEvent(s, c.aux->join, 0));
    }
  }
  return SQUINT_OK;
}

}  // namespace

bool bf16_prepare() { return g_branch_enabled && t_aux.ok(); }
int bf16_options() { return g_branch_enabled | (g_pipe_enabled << 1) | (g_dump_next << 2); }

size_t bf16_workspace_bytes(const squint_dims& d) {
  Layout L = make_layout(d);
  return plan_bf(d, L).total;
}

bool bf16_region(const squint_dims& d, int region, size_t* offset, size_t* bytes) {
  Layout L = make_layout(d);
  BfLay w = plan_bf(d, L);
  const size_t B = d.batch, f = sizeof(float);
  switch (region) {
    case 0: *offset = w.grad_critic; *bytes = L.gsize[0] * f; break;
    case 1: *offset = w.grad_actor; *bytes = L.gsize[1] * f; break;
    case 2: *offset = w.m; *bytes = B * head_out(d) * f; break;
    case 3: *offset = w.Xh.off; *bytes = (size_t)w.Xh.rows * w.Xh.ld * 2; break;
    case 4: *offset = w.logp_cur; *bytes = B * f; break;
    case 5: *offset = w.logp_next; *bytes = B * f; break;
    case 6: *offset = w.a_cur; *bytes = B * d.action_dim * f; break;
    case 7: *offset = w.scal; *bytes = kScal * f; break;
    case 8: *offset = w.img0; *bytes = B * d.img_c * d.img_h * d.img_w; break;
    case 9: *offset = w.img1; *bytes = B * d.img_c * d.img_h * d.img_w; break;
    case 10: *offset = w.y1b; *bytes = B * conv1_out(d) * conv1_out(d) * d.conv_ch * 2; break;
    default: return false;
  }
  return true;
}

squint_status bf16_check(const squint_dims& d) {
  if (d.action_dim > 16) return set_error(SQUINT_EUNSUPPORTED, "bf16 path: action_dim > 16 not built");
  if (d.critic_hidden > 512 || d.actor_hidden > 512 || head_out(d) > 256 || d.latent > 256)
    return set_error(SQUINT_EUNSUPPORTED, "bf16 path: layer width not built");
  return SQUINT_OK;
}

squint_status bf16_update(const squint_dims& d, const squint_hparams& hp, const squint_replay& R,
                          const int64_t* idx, const uint8_t* shifts, const float* eps, int utd,
                          const squint_state& st, float* metrics, void* workspace, size_t workspace_bytes, Comm* comm,
                          cudaStream_t s) {
  squint_status chk = bf16_check(d);
  if (chk != SQUINT_OK) return chk;
  Layout L = make_layout(d);
  BfLay w = plan_bf(d, L);
  if (workspace_bytes < w.total) return set_error(SQUINT_EINVAL, "workspace too small (see squint_workspace_bytes)");
  const bool chain_ok = chain_supported(d.critic_hidden) && chain_supported(d.actor_hidden);
  Ctx c{d, L, reinterpret_cast<char*>(workspace), s, chain_ok, (g_branch_enabled && t_aux.ok()) ? &t_aux : nullptr};
  const int nranks = comm ? comm_nranks(comm) : 1;
  const float inv_btotal = 1.0f / ((float)d.batch * (float)nranks);
  // bf16 shadows of the current master weights (and the conv weight tiles, which with the
  // auxiliary branch are otherwise produced at the end of the previous update)
  {
    const ShadowTable t0 = table_at(c, w.sh[0]), t1 = table_at(c, w.sh[1]), t2 = table_at(c, w.sh[2]);
    const float* const masters[3] = {st.critic, st.critic_target, st.actor};
    const ShadowTable* const tabs[3] = {&t0, &t1, &t2};
    BF_CK(launch_shadow3(masters, tabs, s));
    if (comm == nullptr && c.aux != nullptr)
      BF_CK(launch_conv_tiles(st.critic + L.off(SQUINT_GROUP_CRITIC, "enc.conv1.w"),
                              st.critic + L.off(SQUINT_GROUP_CRITIC, "enc.conv2.w"), d.conv_ch,
                              reinterpret_cast<uint8_t*>(c.ws + w.wtiles), s));
  }
  const size_t B = d.batch, A = d.action_dim;
  const bool pipe = g_pipe_enabled && comm == nullptr && c.aux != nullptr && c.chain;
  auto in = [&](int j) { return UpdIn{idx + j * B, shifts + j * B * 4, eps + j * 2 * B * A, j}; };
  if (pipe) {
    const UpdIn u0 = in(0);
    squint_status r = early_fwd(c, w, hp, R, u0, st, 0, s, 0, c.aux->enc, c.aux->chn);
    if (r != SQUINT_OK) return r;
  }
  for (int j = 0; j < utd; ++j) {
    const UpdIn nx = in(j + 1);
    squint_status r = update_one(c, w, hp, R, idx + j * B, shifts + j * B * 4, eps + j * 2 * B * A, st, metrics + j * 8,
                                 comm, inv_btotal, j, j & 1, pipe, j + 1 < utd ? &nx : nullptr);
    if (r != SQUINT_OK) return r;
  }
  return SQUINT_OK;
}

size_t bf16_act_workspace_bytes(const squint_dims& d, int64_t n) {
  Layout L = make_layout(d);
  WsPlan P;
  const int F = flat_dim(d), npi = d.latent + d.proprio_dim, Ha = d.actor_hidden;
  P.take((size_t)n * ldp(F) * 2);
  P.take((size_t)n * ldp(npi) * 2);
  P.take((size_t)n * ldp(Ha) * 2);
  P.take((size_t)n * ldp(Ha) * 2);
  shadow_plan(P, d, L, SQUINT_GROUP_ACTOR);
  P.take(conv_tiles_bytes(d.conv_ch));
  P.take((size_t)n * 256 * 2 * 2);  // chain exchange scratch (2 hidden layers)
  return P.top + 256;
}

squint_status bf16_act(const squint_dims& d, const squint_hparams& hp, const float* actor_params,
                       const float* critic_params, const uint8_t* frames, int64_t n, int factor, const float* proprio,
                       const float* eps, float* action_out, float* logp_out, uint8_t* ring, const int64_t* slots,
                       void* workspace, cudaStream_t s) {
  squint_status chk = bf16_check(d);
  if (chk != SQUINT_OK) return chk;
  Layout L = make_layout(d);
  WsPlan P;
  const int F = flat_dim(d), Lt = d.latent, npi = Lt + d.proprio_dim, Ha = d.actor_hidden, M = (int)n;
  char* ws = reinterpret_cast<char*>(workspace);
  BM Xh{P.take((size_t)n * ldp(F) * 2), M, F, ldp(F)};
  BM Xa{P.take((size_t)n * ldp(npi) * 2), M, npi, ldp(npi)};
  BM H1{P.take((size_t)n * ldp(Ha) * 2), M, Ha, ldp(Ha)};
  BM H2{P.take((size_t)n * ldp(Ha) * 2), M, Ha, ldp(Ha)};
  ShadowPlan sp = shadow_plan(P, d, L, SQUINT_GROUP_ACTOR);
  uint8_t* wtiles = reinterpret_cast<uint8_t*>(ws + P.take(conv_tiles_bytes(d.conv_ch)));
  const size_t xchg_bytes = (size_t)n * 256 * 2 * 2;
  char* xchg = ws + P.take(xchg_bytes);
  Ctx c{d, L, ws, s, false, nullptr};
  const int gC = SQUINT_GROUP_CRITIC, gA = SQUINT_GROUP_ACTOR;
  std::optional<PhaseScope> ps;
  ps.emplace(1, 0, s);
  BF_CK(launch_shadow(actor_params, table_at(c, sp), s));
  BF_CK(launch_conv_tiles(critic_params + L.off(gC, "enc.conv1.w"), critic_params + L.off(gC, "enc.conv2.w"),
                          d.conv_ch, wtiles, s));
  {
    EncFwdArgs a;
    memset(&a, 0, sizeof(a));
    a.mode = 1;
    a.src[0] = frames;
    a.factor = factor;
    a.ring = ring;
    a.slots = slots;
    a.B = M;
    a.nsrc = 1;
    a.w1 = critic_params + L.off(gC, "enc.conv1.w");
    a.b1 = critic_params + L.off(gC, "enc.conv1.b");
    a.w2 = critic_params + L.off(gC, "enc.conv2.w");
    a.b2 = critic_params + L.off(gC, "enc.conv2.b");
    a.hb[0] = c.bp(Xh);
    a.h_ld = Xh.ld;
    a.C = d.conv_ch;
    a.c_in = d.img_c;
    a.H = d.img_h;
    a.pad = d.pad;
    a.gj[0][0] = GatherJob{proprio, d.proprio_dim, c.bp(Xa), Xa.ld, Lt, 0};
    a.ngj[0] = 1;
    a.wtiles = wtiles;
    BF_CK(launch_enc_fwd_tc(a, s));
  }
  ps.reset();
  ps.emplace(2, 0, s);
  const Lin ap = proj(c, sp, actor_params, gA, "actor");
  const Mlp am = mlp(c, sp, actor_params, gA, "actor");
  {
    GemmBuilder gb(1);
    fwd(gb, c.mat(Xh), ap, GE_LN_TANH, c.bp(Xa), Xa.ld, hp.ln_eps);
    BF_CK(gemm_launch(gb, s));
  }
  if (chain_supported(Ha)) {
    // the whole actor MLP + tanh-Gaussian head in one fused chain launch
    ChainBuilder cb(1);
    cb.xscr = xchg;
    cb.xcap = xchg_bytes;
    CProb& pa = cb.add(M, c.mat(Xa));
    ch_fwd(cb, pa, GE_LN_RELU, am.l1, Ha, npi, none_mat(), none_mat(), nullptr, hp.ln_eps);
    ch_fwd(cb, pa, GE_LN_RELU, am.l2, Ha, Ha, none_mat(), none_mat(), nullptr, hp.ln_eps);
    CLayer& tg = cb.layer(pa, GE_TG_FWD, am.l3.w, 0, 2 * d.action_dim, Ha, none_mat(), none_mat());
    tg.bias = am.l3.b;
    tg.eps = eps;
    tg.act = action_out;
    tg.logp = logp_out;
    tg.lo = hp.log_std_min;
    tg.hi = hp.log_std_max;
    BF_CK(chain_launch(cb, s));
    return SQUINT_OK;
  }
  {
    GemmBuilder gb(1);
    fwd(gb, c.mat(Xa), am.l1, GE_LN_RELU, c.bp(H1), H1.ld, hp.ln_eps);
    BF_CK(gemm_launch(gb, s));
  }
  {
    GemmBuilder gb(1);
    fwd(gb, c.mat(H1), am.l2, GE_LN_RELU, c.bp(H2), H2.ld, hp.ln_eps);
    BF_CK(gemm_launch(gb, s));
  }
  {
    GemmBuilder gb(1);
    GProb& p = fwd(gb, c.mat(H2), am.l3, GE_TG_FWD, nullptr, 0, hp.ln_eps);
    p.eps = eps;
    p.act = action_out;
    p.logp = logp_out;
    p.lo = hp.log_std_min;
    p.hi = hp.log_std_max;
    BF_CK(gemm_launch(gb, s));
  }
  return SQUINT_OK;
}

// option 3: validate the device-side preconditions (index ranges, distinct slots) before each
// call, synchronising the stream (a debugging aid, off by default; squint.h)
int g_check_enabled = 0;

}  // namespace sq

extern "C" squint_status squint_selftest_gemm(const void* A, int a_rows, int a_cols, int a_ld, int a_mn, const void* B,
                                              int b_rows, int b_cols, int b_ld, int b_mn, int M, int N, int K,
                                              float* out, squint_stream_t stream) {
  using namespace sq;
  if (!A || !B || !out || M < 1 || N < 1 || K < 1) return set_error(SQUINT_EINVAL, "selftest_gemm: bad argument");
  GemmBuilder gb(0);
  GProb& p = gb.add(M, N, GE_DW);
  gb.seg(p, Mat{A, a_rows, a_cols, a_ld}, a_mn, 0, Mat{B, b_rows, b_cols, b_ld}, b_mn, 0, K);
  p.outf = out;
  p.ldf = N;
  const int e = gemm_launch(gb, (cudaStream_t)stream);
  if (e)
    return set_error(SQUINT_ECUDA, std::string("selftest_gemm: ") +
                                       (e > 0 ? cudaGetErrorString((cudaError_t)e) : "plan/map error"));
  return SQUINT_OK;
}

extern "C" SQUINT_API int squint_debug_gemm_times(unsigned long long* host, int max_entries) {
  return sq::gemm_debug_times(host, max_entries);
}

// Instrumentation options (host): key 1 = auxiliary branch of the bf16 update (1 on, 0 off).
extern "C" SQUINT_API squint_status squint_set_option(int key, int value) {
  if (key == 1) {
    sq::g_branch_enabled = value != 0;
    return SQUINT_OK;
  }
  if (key == 2) {
    sq::g_pipe_enabled = value != 0;
    return SQUINT_OK;
  }
  if (key == 3) {
    sq::g_check_enabled = value != 0;
    return SQUINT_OK;
  }
  if (key == 5) {
    sq::g_dump_next = value != 0;
    return SQUINT_OK;
  }
  if (key == 4) {
    if (value < 0 || value > 15) return sq::set_error(SQUINT_EINVAL, "option 4: value must be 0..15");
    sq::g_emul = value;
    return SQUINT_OK;
  }
  return sq::set_error(SQUINT_EINVAL, "unknown option");
}
