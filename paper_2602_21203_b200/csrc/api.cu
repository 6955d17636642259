// api.cu -- the C ABI of libsquint (include/squint.h): argument checks, parameter and
// workspace layout, and the launch sequence of one SAC update (Algorithm 1 L9-24).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <optional>
#include <string>
#include <vector>

#include "../../include/squint.h"
#include "comm.hpp"
#include "common.cuh"
#include "dense.cuh"
#include "encoder.cuh"
#include "heads.cuh"
#include "layout.hpp"
#include "optim.cuh"
#include "update_bf16.hpp"

namespace sq {

static thread_local std::string g_err;

static squint_status fail(squint_status st, const std::string& m) {
  g_err = m;
  return st;
}
squint_status set_error(squint_status st, const std::string& m) { return fail(st, m); }

#define SQ_CK(expr)                                                                       \
  do {                                                                                    \
    int _e = (int)(expr);                                                                 \
    if (_e != 0)                                                                          \
      return fail(SQUINT_ECUDA, std::string("CUDA error in ") + #expr + ": " +            \
                                    cudaGetErrorString((cudaError_t)_e));                 \
  } while (0)

// ---- workspace plan ------------------------------------------------------------------
struct MlpC {
  size_t h1, xh1, rs1, h2, xh2, rs2;
};
struct ProjC {
  size_t z, xh, rs;
};
struct WsLay {
  size_t img0, y1, h, hn;
  ProjC pq, pqn, ppn, pp, pq1;
  MlpC an, ac, tq[2], q[2], q1[2];
  size_t out_an, out_ac, a_next, logp_next, a_cur, logp_cur;
  size_t tlogits, logits, logits1, m, dlogits, row_loss, row_q, row_lpi;
  size_t dA2[2], dN2[2], dA1[2], dN1[2], dAp, dNp, dAh, dA1enc, enc_part;
  size_t dO, adA2, adN2, adA1, adN1, adAp, adNp;
  size_t grad_critic, grad_actor, adam_part, scal, lpi_sums;
  size_t total;
};

static WsLay plan_ws(const squint_dims& d, const Layout& L) {
  WsPlan P;
  WsLay w;
  const size_t B = d.batch, F = flat_dim(d), Lt = d.latent, Hc = d.critic_hidden, Ha = d.actor_hidden,
               N = head_out(d), A = d.action_dim, C = d.conv_ch, P1 = conv1_out(d) * conv1_out(d);
  const size_t f = sizeof(float);
  auto proj = [&]() { return ProjC{P.take(B * Lt * f), P.take(B * Lt * f), P.take(B * f)}; };
  auto mlp = [&](size_t H) {
    return MlpC{P.take(B * H * f), P.take(B * H * f), P.take(B * f), P.take(B * H * f), P.take(B * H * f),
                P.take(B * f)};
  };
  w.img0 = P.take(B * d.img_c * d.img_h * d.img_w);
  w.y1 = P.take(B * C * P1 * f);
  w.h = P.take(B * F * f);
  w.hn = P.take(B * F * f);
  w.pq = proj();
  w.pqn = proj();
  w.ppn = proj();
  w.pp = proj();
  w.pq1 = proj();
  w.an = mlp(Ha);
  w.ac = mlp(Ha);
  for (int i = 0; i < 2; ++i) {
    w.tq[i] = mlp(Hc);
    w.q[i] = mlp(Hc);
    w.q1[i] = mlp(Hc);
  }
  w.out_an = P.take(B * 2 * A * f);
  w.out_ac = P.take(B * 2 * A * f);
  w.a_next = P.take(B * A * f);
  w.logp_next = P.take(B * f);
  w.a_cur = P.take(B * A * f);
  w.logp_cur = P.take(B * f);
  w.tlogits = P.take(2 * B * N * f);
  w.logits = P.take(2 * B * N * f);
  w.logits1 = P.take(2 * B * N * f);
  w.m = P.take(B * N * f);
  w.dlogits = P.take(2 * B * N * f);
  w.row_loss = P.take(B * f);
  w.row_q = P.take(B * f);
  w.row_lpi = P.take(B * f);
  for (int i = 0; i < 2; ++i) {
    w.dA2[i] = P.take(B * Hc * f);
    w.dN2[i] = P.take(B * Hc * f);
    w.dA1[i] = P.take(B * Hc * f);
    w.dN1[i] = P.take(B * Hc * f);
  }
  w.dAp = P.take(B * Lt * f);
  w.dNp = P.take(B * Lt * f);
  w.dAh = P.take(B * F * f);
  w.dA1enc = P.take(B * C * P1 * f);
  w.enc_part = P.take(enc_bwd_partial_floats(d.conv_ch, d.img_c, enc_bwd_nchunk(d.batch)) * f);
  w.dO = P.take(B * 2 * A * f);
  w.adA2 = P.take(B * Ha * f);
  w.adN2 = P.take(B * Ha * f);
  w.adA1 = P.take(B * Ha * f);
  w.adN1 = P.take(B * Ha * f);
  w.adAp = P.take(B * Lt * f);
  w.adNp = P.take(B * Lt * f);
  // gradient buffers carry kExtra floats of row sums behind them (one all-reduce each)
  w.grad_critic = P.take((L.gsize[SQUINT_GROUP_CRITIC] + kExtra) * f);
  w.grad_actor = P.take((L.gsize[SQUINT_GROUP_ACTOR] + kExtra) * f);
  w.adam_part = P.take(kAdamBlocks * f);
  w.scal = P.take(kScal * f);
  w.lpi_sums = P.take(2 * f);
  w.total = P.top + 256;
  return w;
}

// Views of one parameter set.
struct LinV {
  const float *w, *b, *g, *beta;
};
struct MlpV {
  LinV l1, l2, l3;
};
static LinV lin(const float* base, const Layout& L, int grp, const std::string& p, bool ln, const std::string& lnp) {
  LinV v;
  v.w = base + L.off(grp, p + ".w");
  v.b = base + L.off(grp, p + ".b");
  v.g = ln ? base + L.off(grp, lnp + ".g") : nullptr;
  v.beta = ln ? base + L.off(grp, lnp + ".b") : nullptr;
  return v;
}
static MlpV mlpv(const float* base, const Layout& L, int grp, const std::string& p) {
  return MlpV{lin(base, L, grp, p + ".l1", true, p + ".ln1"), lin(base, L, grp, p + ".l2", true, p + ".ln2"),
              lin(base, L, grp, p + ".l3", false, "")};
}
static LinV projv(const float* base, const Layout& L, int grp, const std::string& p) {
  return lin(base, L, grp, p + ".proj", true, p + ".proj.ln");
}

// gradient views (writable)
struct LinG {
  float *w, *b, *g, *beta;
};
static LinG ling(float* base, const Layout& L, int grp, const std::string& p, bool ln, const std::string& lnp) {
  LinG v;
  v.w = base + L.off(grp, p + ".w");
  v.b = base + L.off(grp, p + ".b");
  v.g = ln ? base + L.off(grp, lnp + ".g") : nullptr;
  v.beta = ln ? base + L.off(grp, lnp + ".b") : nullptr;
  return v;
}

static ASeg seg(const float* p, int ld, int width, const int64_t* rows = nullptr) { return ASeg{p, rows, ld, width}; }

static DenseProb fwd_prob(int M, const LinV& W, int nout, int nin, std::initializer_list<ASeg> A, int epi, float* out,
                          float* xh, float* rs, float ln_eps) {
  DenseProb p;
  memset(&p, 0, sizeof(p));
  p.M = M;
  p.N = nout;
  p.K = nin;
  p.nA = 0;
  for (const auto& s : A) p.A[p.nA++] = s;
  p.nB = 1;
  p.B[0] = BSeg{W.w, nin, nin, 1};
  p.epi = epi;
  p.bias = W.b;
  p.g = W.g;
  p.beta = W.beta;
  p.out = out;
  p.ldo = nout;
  p.xh = xh;
  p.rstd = rs;
  p.ln_eps = ln_eps;
  return p;
}

// dX = D @ W (W [nout][nin] row-major): B(n, k) = W[k][col0 + n]
static DenseProb bwd_prob(int M, int ncols, std::initializer_list<ASeg> D, std::initializer_list<BSeg> W, int epi,
                          float* out, int ldo) {
  DenseProb p;
  memset(&p, 0, sizeof(p));
  p.M = M;
  p.N = ncols;
  p.K = 0;
  p.nA = 0;
  for (const auto& s : D) {
    p.A[p.nA++] = s;
    p.K += s.width;
  }
  p.nB = 0;
  for (const auto& s : W) p.B[p.nB++] = s;
  p.epi = epi;
  p.out = out;
  p.ldo = ldo;
  return p;
}

struct Ctx {
  const squint_dims& d;
  const squint_hparams& hp;
  const Layout& L;
  const WsLay& w;
  char* ws;
  cudaStream_t s;
  float* F(size_t off) const { return reinterpret_cast<float*>(ws + off); }
};


// Dense layers: fp32 SIMT (parity mode) or bf16 tcgen05 tensor cores.
// squint_set_option key 4 (numerics measurement, fp32 path only): round to bf16 what the tensor-core
// path holds in bf16 -- bit 0: dense-layer GEMM activations / dY, bit 1: dense weights, bit 2: the
// LayerNorm x_hat cache, bit 3: the encoder's conv weights, conv1 activations and conv gradients --
// to measure the error bf16 storage alone introduces (DESIGN.md R-tol-bf16)
int g_emul = 0;
static int emul_flags() { return g_emul; }
static int run_dense(DenseBatch& b, cudaStream_t s) {
  b.emul = emul_flags();
  const int tn = plan_dense(b);
  return launch_dense_f32(b, tn, s);
}
static int run_dw(DwBatch& b, cudaStream_t s) {
  b.emul = emul_flags();
  plan_dw(b);
  return launch_dw_f32(b, s);
}

// ---- one update ---------------------------------------------------------------------------
static squint_status update_one(const Ctx& c, const squint_replay& R, const int64_t* idx, const uint8_t* sh,
                                    const float* eps, const squint_state& st, float* metrics, Comm* comm,
                                    float inv_btotal, int rep) {
  const squint_dims& d = c.d;
  const squint_hparams& hp = c.hp;
  const Layout& L = c.L;
  const WsLay& w = c.w;
  cudaStream_t s = c.s;
  const int B = d.batch, F = flat_dim(d), Lt = d.latent, Hc = d.critic_hidden, Ha = d.actor_hidden, N = head_out(d),
            A = d.action_dim, P = d.proprio_dim, C = d.conv_ch;
  const int nq = Lt + P + A, npi = Lt + P;
  const float* eps_next = eps;
  const float* eps_cur = eps + (size_t)B * A;
  const float le = hp.ln_eps;

  const int gC = SQUINT_GROUP_CRITIC, gA = SQUINT_GROUP_ACTOR, gT = SQUINT_GROUP_TARGET;
  const float* crit = st.critic;
  const float* tgt = st.critic_target;
  const float* act = st.actor;
  const LinV cproj = projv(crit, L, gC, "critic"), tproj = projv(tgt, L, gT, "critic"),
             aproj = projv(act, L, gA, "actor");
  const MlpV cq[2] = {mlpv(crit, L, gC, "critic.q1"), mlpv(crit, L, gC, "critic.q2")};
  const MlpV tq[2] = {mlpv(tgt, L, gT, "critic.q1"), mlpv(tgt, L, gT, "critic.q2")};
  const MlpV am = mlpv(act, L, gA, "actor");

  // a3-a5: gather + shift + encoder for obs and next_obs
  {
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
    e.h[0] = c.F(w.h);
    e.h[1] = c.F(w.hn);
    e.y1 = c.F(w.y1);
    e.img0 = reinterpret_cast<uint8_t*>(c.ws + w.img0);
    e.C = C;
    e.c_in = d.img_c;
    e.H = d.img_h;
    e.pad = d.pad;
    e.emul = g_emul;
    SQ_CK(launch_enc_fwd(e, s));
  }
  // a6: four projections
  {
    PhaseScope ps(4, rep, s);
    DenseBatch b;
    b.nprob = 4;
    b.p[0] = fwd_prob(B, cproj, Lt, F, {seg(c.F(w.h), F, F)}, EPI_LN_TANH, c.F(w.pq.z), c.F(w.pq.xh), c.F(w.pq.rs), le);
    b.p[1] = fwd_prob(B, tproj, Lt, F, {seg(c.F(w.hn), F, F)}, EPI_LN_TANH, c.F(w.pqn.z), nullptr, nullptr, le);
    b.p[2] = fwd_prob(B, aproj, Lt, F, {seg(c.F(w.hn), F, F)}, EPI_LN_TANH, c.F(w.ppn.z), nullptr, nullptr, le);
    b.p[3] = fwd_prob(B, aproj, Lt, F, {seg(c.F(w.h), F, F)}, EPI_LN_TANH, c.F(w.pp.z), c.F(w.pp.xh), c.F(w.pp.rs), le);
    SQ_CK(run_dense(b, s));
  }
  // a7: actor MLP on next obs (target sample) and on current obs (alpha / actor losses)
  {
    PhaseScope ps(5, rep, s);
    DenseBatch b;
    b.nprob = 2;
    b.p[0] = fwd_prob(B, am.l1, Ha, npi, {seg(c.F(w.ppn.z), Lt, Lt), seg(R.next_proprio, P, P, idx)}, EPI_LN_RELU,
                      c.F(w.an.h1), nullptr, nullptr, le);
    b.p[1] = fwd_prob(B, am.l1, Ha, npi, {seg(c.F(w.pp.z), Lt, Lt), seg(R.proprio, P, P, idx)}, EPI_LN_RELU,
                      c.F(w.ac.h1), c.F(w.ac.xh1), c.F(w.ac.rs1), le);
    SQ_CK(run_dense(b, s));
    b.p[0] = fwd_prob(B, am.l2, Ha, Ha, {seg(c.F(w.an.h1), Ha, Ha)}, EPI_LN_RELU, c.F(w.an.h2), nullptr, nullptr, le);
    b.p[1] = fwd_prob(B, am.l2, Ha, Ha, {seg(c.F(w.ac.h1), Ha, Ha)}, EPI_LN_RELU, c.F(w.ac.h2), c.F(w.ac.xh2),
                      c.F(w.ac.rs2), le);
    SQ_CK(run_dense(b, s));
    b.p[0] = fwd_prob(B, am.l3, 2 * A, Ha, {seg(c.F(w.an.h2), Ha, Ha)}, EPI_TG_FWD, c.F(w.out_an), nullptr, nullptr, le);
    b.p[1] = fwd_prob(B, am.l3, 2 * A, Ha, {seg(c.F(w.ac.h2), Ha, Ha)}, EPI_TG_FWD, c.F(w.out_ac), nullptr, nullptr, le);
    b.p[0].eps = eps_next;
    b.p[0].act = c.F(w.a_next);
    b.p[0].logp = c.F(w.logp_next);
    b.p[1].eps = eps_cur;
    b.p[1].act = c.F(w.a_cur);
    b.p[1].logp = c.F(w.logp_cur);
    for (int i = 0; i < 2; ++i) {
      b.p[i].lo = hp.log_std_min;
      b.p[i].hi = hp.log_std_max;
    }
    SQ_CK(run_dense(b, s));
  }
  // a8: target heads on (z', s', a') and online heads on (z, s, a)
  {
    PhaseScope ps(6, rep, s);
    DenseBatch b;
    b.nprob = 4;
    for (int i = 0; i < 2; ++i) {
      b.p[i] = fwd_prob(B, tq[i].l1, Hc, nq,
                        {seg(c.F(w.pqn.z), Lt, Lt), seg(R.next_proprio, P, P, idx), seg(c.F(w.a_next), A, A)},
                        EPI_LN_RELU, c.F(w.tq[i].h1), nullptr, nullptr, le);
      b.p[2 + i] = fwd_prob(B, cq[i].l1, Hc, nq,
                            {seg(c.F(w.pq.z), Lt, Lt), seg(R.proprio, P, P, idx), seg(R.action, A, A, idx)},
                            EPI_LN_RELU, c.F(w.q[i].h1), c.F(w.q[i].xh1), c.F(w.q[i].rs1), le);
    }
    SQ_CK(run_dense(b, s));
    for (int i = 0; i < 2; ++i) {
      b.p[i] = fwd_prob(B, tq[i].l2, Hc, Hc, {seg(c.F(w.tq[i].h1), Hc, Hc)}, EPI_LN_RELU, c.F(w.tq[i].h2), nullptr,
                        nullptr, le);
      b.p[2 + i] = fwd_prob(B, cq[i].l2, Hc, Hc, {seg(c.F(w.q[i].h1), Hc, Hc)}, EPI_LN_RELU, c.F(w.q[i].h2),
                            c.F(w.q[i].xh2), c.F(w.q[i].rs2), le);
    }
    SQ_CK(run_dense(b, s));
    for (int i = 0; i < 2; ++i) {
      b.p[i] = fwd_prob(B, tq[i].l3, N, Hc, {seg(c.F(w.tq[i].h2), Hc, Hc)}, EPI_BIAS, c.F(w.tlogits) + (size_t)i * B * N,
                        nullptr, nullptr, le);
      b.p[2 + i] = fwd_prob(B, cq[i].l3, N, Hc, {seg(c.F(w.q[i].h2), Hc, Hc)}, EPI_BIAS,
                            c.F(w.logits) + (size_t)i * B * N, nullptr, nullptr, le);
    }
    SQ_CK(run_dense(b, s));
  }
  // a9-a10: target distribution, projection, CE and dL/dlogits
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
    t.dlogits = c.F(w.dlogits);
    t.row_loss = c.F(w.row_loss);
    SQ_CK(launch_target_ce(t, s));
  }
  // a10: critic backward (heads -> projection -> encoder)
  float* gc = c.F(w.grad_critic);
  {
    PhaseScope ps(8, rep, s);
    DenseBatch b;
    b.nprob = 2;
    for (int i = 0; i < 2; ++i) {
      b.p[i] = bwd_prob(B, Hc, {seg(c.F(w.dlogits) + (size_t)i * B * N, N, N)}, {BSeg{cq[i].l3.w, Hc, N, 0}},
                        EPI_BWD_LN_RELU, c.F(w.dA2[i]), Hc);
      b.p[i].y = c.F(w.q[i].h2);
      b.p[i].xh = c.F(w.q[i].xh2);
      b.p[i].rstd = c.F(w.q[i].rs2);
      b.p[i].g = cq[i].l2.g;
      b.p[i].out2 = c.F(w.dN2[i]);
    }
    SQ_CK(run_dense(b, s));
    for (int i = 0; i < 2; ++i) {
      b.p[i] = bwd_prob(B, Hc, {seg(c.F(w.dA2[i]), Hc, Hc)}, {BSeg{cq[i].l2.w, Hc, Hc, 0}}, EPI_BWD_LN_RELU,
                        c.F(w.dA1[i]), Hc);
      b.p[i].y = c.F(w.q[i].h1);
      b.p[i].xh = c.F(w.q[i].xh1);
      b.p[i].rstd = c.F(w.q[i].rs1);
      b.p[i].g = cq[i].l1.g;
      b.p[i].out2 = c.F(w.dN1[i]);
    }
    SQ_CK(run_dense(b, s));
    // dz = sum_i dA1_i W1_i[:, :L]  -> through tanh + LN of the critic projection
    b.nprob = 1;
    b.p[0] = bwd_prob(B, Lt, {seg(c.F(w.dA1[0]), Hc, Hc), seg(c.F(w.dA1[1]), Hc, Hc)},
                      {BSeg{cq[0].l1.w, nq, Hc, 0}, BSeg{cq[1].l1.w, nq, Hc, 0}}, EPI_BWD_LN_TANH, c.F(w.dAp), Lt);
    b.p[0].y = c.F(w.pq.z);
    b.p[0].xh = c.F(w.pq.xh);
    b.p[0].rstd = c.F(w.pq.rs);
    b.p[0].g = cproj.g;
    b.p[0].out2 = c.F(w.dNp);
    SQ_CK(run_dense(b, s));
    // dh = dAp Wp, masked by ReLU'(conv2)
    b.p[0] = bwd_prob(B, F, {seg(c.F(w.dAp), Lt, Lt)}, {BSeg{cproj.w, F, Lt, 0}}, EPI_RELU_MASK, c.F(w.dAh), F);
    b.p[0].y = c.F(w.h);
    SQ_CK(run_dense(b, s));
  }
  {
    PhaseScope ps(9, rep, s);
    DwBatch b;
    b.nprob = 7;
    int k = 0;
    for (int i = 0; i < 2; ++i) {
      const std::string p = i == 0 ? "critic.q1" : "critic.q2";
      LinG g3 = ling(gc, L, gC, p + ".l3", false, ""), g2 = ling(gc, L, gC, p + ".l2", true, p + ".ln2"),
           g1 = ling(gc, L, gC, p + ".l1", true, p + ".ln1");
      DwProb& a3 = b.p[k++];
      a3 = DwProb{B, N, Hc, c.F(w.dlogits) + (size_t)i * B * N, 1, {seg(c.F(w.q[i].h2), Hc, Hc)}, g3.w, g3.b,
                  nullptr, nullptr, nullptr, nullptr, 0, 0};
      DwProb& a2 = b.p[k++];
      a2 = DwProb{B, Hc, Hc, c.F(w.dA2[i]), 1, {seg(c.F(w.q[i].h1), Hc, Hc)}, g2.w, g2.b, c.F(w.dN2[i]),
                  c.F(w.q[i].xh2), g2.g, g2.beta, 0, 0};
      DwProb& a1 = b.p[k++];
      a1 = DwProb{B, Hc, nq, c.F(w.dA1[i]), 3,
                  {seg(c.F(w.pq.z), Lt, Lt), seg(R.proprio, P, P, idx), seg(R.action, A, A, idx)}, g1.w, g1.b,
                  c.F(w.dN1[i]), c.F(w.q[i].xh1), g1.g, g1.beta, 0, 0};
    }
    LinG gp = ling(gc, L, gC, "critic.proj", true, "critic.proj.ln");
    b.p[k++] = DwProb{B, Lt, F, c.F(w.dAp), 1, {seg(c.F(w.h), F, F)}, gp.w, gp.b, c.F(w.dNp), c.F(w.pq.xh), gp.g,
                      gp.beta, 0, 0};
    SQ_CK(run_dw(b, s));
  }
  {
    PhaseScope ps(10, rep, s);
    EncBwdArgs e;
    memset(&e, 0, sizeof(e));
    e.B = B;
    e.C = C;
    e.c_in = d.img_c;
    e.H = d.img_h;
    e.dA2 = c.F(w.dAh);
    e.y1 = c.F(w.y1);
    e.img = reinterpret_cast<const uint8_t*>(c.ws + w.img0);
    e.w2 = crit + L.off(gC, "enc.conv2.w");
    e.dA1 = c.F(w.dA1enc);
    e.part = c.F(w.enc_part);
    e.nchunk = enc_bwd_nchunk(B);
    e.gw1 = gc + L.off(gC, "enc.conv1.w");
    e.gb1 = gc + L.off(gC, "enc.conv1.b");
    e.gw2 = gc + L.off(gC, "enc.conv2.w");
    e.gb2 = gc + L.off(gC, "enc.conv2.b");
    e.emul = g_emul;
    SQ_CK(launch_enc_bwd(e, s));
  }
  float* extras = gc + L.gsize[gC];
  float* scal = c.F(w.scal);
  // data parallel: sum critic gradients and the row sums (log pi, L_Q) over ranks
  if (comm) {
    SQ_CK(launch_row_sums(c.F(w.logp_cur), c.F(w.row_loss), B, extras, s));
    if (comm_allreduce_sum(comm, gc, L.gsize[gC] + kExtra, s) != 0) return fail(SQUINT_ENCCL, comm_error());
  }
  // a11: temperature step; Adam step counters and bias corrections; a13 Adam (critic)
  {
    PhaseScope ps(11, rep, s);
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
    SQ_CK(launch_scalars(a, s));
    // a13: Adam on the critic group (psi, projection, heads)
    SQ_CK(launch_adam(st.critic, gc, st.m_critic, st.v_critic, L.gsize[gC], hp.lr_critic, hp.beta1, hp.beta2,
                      hp.adam_eps, scal + S_C1_CRITIC, scal + S_C2_CRITIC, c.F(w.adam_part), s));
  }
  // a12: actor loss against theta+ on sg(h)
  {
    std::optional<PhaseScope> ps;
    ps.emplace(12, rep, s);
    const MlpV cq1[2] = {mlpv(crit, L, gC, "critic.q1"), mlpv(crit, L, gC, "critic.q2")};  // same buffer, now theta+
    DenseBatch b;
    b.nprob = 1;
    b.p[0] = fwd_prob(B, cproj, Lt, F, {seg(c.F(w.h), F, F)}, EPI_LN_TANH, c.F(w.pq1.z), nullptr, nullptr, le);
    SQ_CK(run_dense(b, s));
    b.nprob = 2;
    for (int i = 0; i < 2; ++i)
      b.p[i] = fwd_prob(B, cq1[i].l1, Hc, nq,
                        {seg(c.F(w.pq1.z), Lt, Lt), seg(R.proprio, P, P, idx), seg(c.F(w.a_cur), A, A)}, EPI_LN_RELU,
                        c.F(w.q1[i].h1), c.F(w.q1[i].xh1), c.F(w.q1[i].rs1), le);
    SQ_CK(run_dense(b, s));
    for (int i = 0; i < 2; ++i)
      b.p[i] = fwd_prob(B, cq1[i].l2, Hc, Hc, {seg(c.F(w.q1[i].h1), Hc, Hc)}, EPI_LN_RELU, c.F(w.q1[i].h2),
                        c.F(w.q1[i].xh2), c.F(w.q1[i].rs2), le);
    SQ_CK(run_dense(b, s));
    for (int i = 0; i < 2; ++i)
      b.p[i] = fwd_prob(B, cq1[i].l3, N, Hc, {seg(c.F(w.q1[i].h2), Hc, Hc)}, EPI_BIAS,
                        c.F(w.logits1) + (size_t)i * B * N, nullptr, nullptr, le);
    SQ_CK(run_dense(b, s));
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
    q.dlogits = c.F(w.dlogits);
    q.row_q = c.F(w.row_q);
    q.row_lpi = c.F(w.row_lpi);
    SQ_CK(launch_actor_q(q, s));
    // dL/da~ through theta+ heads
    ps.reset();
    ps.emplace(13, rep, s);
    for (int i = 0; i < 2; ++i) {
      b.p[i] = bwd_prob(B, Hc, {seg(c.F(w.dlogits) + (size_t)i * B * N, N, N)}, {BSeg{cq1[i].l3.w, Hc, N, 0}},
                        EPI_BWD_LN_RELU, c.F(w.dA2[i]), Hc);
      b.p[i].y = c.F(w.q1[i].h2);
      b.p[i].xh = c.F(w.q1[i].xh2);
      b.p[i].rstd = c.F(w.q1[i].rs2);
      b.p[i].g = cq1[i].l2.g;
      b.p[i].out2 = c.F(w.dN2[i]);
    }
    SQ_CK(run_dense(b, s));
    for (int i = 0; i < 2; ++i) {
      b.p[i] = bwd_prob(B, Hc, {seg(c.F(w.dA2[i]), Hc, Hc)}, {BSeg{cq1[i].l2.w, Hc, Hc, 0}}, EPI_BWD_LN_RELU,
                        c.F(w.dA1[i]), Hc);
      b.p[i].y = c.F(w.q1[i].h1);
      b.p[i].xh = c.F(w.q1[i].xh1);
      b.p[i].rstd = c.F(w.q1[i].rs1);
      b.p[i].g = cq1[i].l1.g;
      b.p[i].out2 = c.F(w.dN1[i]);
    }
    SQ_CK(run_dense(b, s));
    b.nprob = 1;
    b.p[0] = bwd_prob(B, A, {seg(c.F(w.dA1[0]), Hc, Hc), seg(c.F(w.dA1[1]), Hc, Hc)},
                      {BSeg{cq1[0].l1.w + Lt + P, nq, Hc, 0}, BSeg{cq1[1].l1.w + Lt + P, nq, Hc, 0}}, EPI_TG_BWD,
                      c.F(w.dO), 2 * A);
    b.p[0].tg_o = c.F(w.out_ac);
    b.p[0].eps = eps_cur;
    b.p[0].dlogp_scale = scal + S_ALPHA1_SCALE;
    b.p[0].dlogp_mult = 1.f;
    b.p[0].lo = hp.log_std_min;
    b.p[0].hi = hp.log_std_max;
    SQ_CK(run_dense(b, s));
    // actor MLP backward
    b.p[0] = bwd_prob(B, Ha, {seg(c.F(w.dO), 2 * A, 2 * A)}, {BSeg{am.l3.w, Ha, 2 * A, 0}}, EPI_BWD_LN_RELU,
                      c.F(w.adA2), Ha);
    b.p[0].y = c.F(w.ac.h2);
    b.p[0].xh = c.F(w.ac.xh2);
    b.p[0].rstd = c.F(w.ac.rs2);
    b.p[0].g = am.l2.g;
    b.p[0].out2 = c.F(w.adN2);
    SQ_CK(run_dense(b, s));
    b.p[0] = bwd_prob(B, Ha, {seg(c.F(w.adA2), Ha, Ha)}, {BSeg{am.l2.w, Ha, Ha, 0}}, EPI_BWD_LN_RELU, c.F(w.adA1), Ha);
    b.p[0].y = c.F(w.ac.h1);
    b.p[0].xh = c.F(w.ac.xh1);
    b.p[0].rstd = c.F(w.ac.rs1);
    b.p[0].g = am.l1.g;
    b.p[0].out2 = c.F(w.adN1);
    SQ_CK(run_dense(b, s));
    b.p[0] = bwd_prob(B, Lt, {seg(c.F(w.adA1), Ha, Ha)}, {BSeg{am.l1.w, npi, Ha, 0}}, EPI_BWD_LN_TANH, c.F(w.adAp), Lt);
    b.p[0].y = c.F(w.pp.z);
    b.p[0].xh = c.F(w.pp.xh);
    b.p[0].rstd = c.F(w.pp.rs);
    b.p[0].g = aproj.g;
    b.p[0].out2 = c.F(w.adNp);
    SQ_CK(run_dense(b, s));
  }
  float* ga = c.F(w.grad_actor);
  {
    PhaseScope ps(14, rep, s);
    DwBatch b;
    b.nprob = 4;
    LinG g3 = ling(ga, L, gA, "actor.l3", false, ""), g2 = ling(ga, L, gA, "actor.l2", true, "actor.ln2"),
         g1 = ling(ga, L, gA, "actor.l1", true, "actor.ln1"), gp = ling(ga, L, gA, "actor.proj", true, "actor.proj.ln");
    b.p[0] = DwProb{B, 2 * A, Ha, c.F(w.dO), 1, {seg(c.F(w.ac.h2), Ha, Ha)}, g3.w, g3.b, nullptr, nullptr, nullptr,
                    nullptr, 0, 0};
    b.p[1] = DwProb{B, Ha, Ha, c.F(w.adA2), 1, {seg(c.F(w.ac.h1), Ha, Ha)}, g2.w, g2.b, c.F(w.adN2), c.F(w.ac.xh2),
                    g2.g, g2.beta, 0, 0};
    b.p[2] = DwProb{B, Ha, npi, c.F(w.adA1), 2, {seg(c.F(w.pp.z), Lt, Lt), seg(R.proprio, P, P, idx)}, g1.w, g1.b,
                    c.F(w.adN1), c.F(w.ac.xh1), g1.g, g1.beta, 0, 0};
    b.p[3] = DwProb{B, Lt, F, c.F(w.adAp), 1, {seg(c.F(w.h), F, F)}, gp.w, gp.b, c.F(w.adNp), c.F(w.pp.xh), gp.g,
                    gp.beta, 0, 0};
    SQ_CK(run_dw(b, s));
  }
  float* lpis = c.F(w.lpi_sums);
  PhaseScope ps15(15, rep, s);
  if (comm) {
    float* ax = ga + L.gsize[gA];
    SQ_CK(launch_lpi_sums(c.F(w.row_lpi), c.F(w.row_q), B, ax, s));
    if (comm_allreduce_sum(comm, ga, L.gsize[gA] + kExtra, s) != 0) return fail(SQUINT_ENCCL, comm_error());
    lpis = ax;
  }
  SQ_CK(launch_adam(st.actor, ga, st.m_actor, st.v_actor, L.gsize[gA], hp.lr_actor, hp.beta1, hp.beta2, hp.adam_eps,
                    scal + S_C1_ACTOR, scal + S_C2_ACTOR, nullptr, s));
  // a14: Polyak over every critic tensor except the encoder
  SQ_CK(launch_polyak(st.critic_target, st.critic + L.enc_end, L.gsize[SQUINT_GROUP_TARGET], hp.tau, s));
  {
    MetricsArgs m;
    memset(&m, 0, sizeof(m));
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
    SQ_CK(launch_metrics(m, s));
  }
  return SQUINT_OK;
}

static bool check_hp(const squint_hparams& h, std::string* e) {
  if (!(h.gamma >= 0.f && h.gamma <= 1.f)) return *e = "gamma must be in [0, 1]", false;
  if (!(h.tau >= 0.f && h.tau <= 1.f)) return *e = "tau must be in [0, 1]", false;
  if (!(h.beta1 >= 0.f && h.beta1 < 1.f && h.beta2 >= 0.f && h.beta2 < 1.f)) return *e = "Adam betas in [0, 1)", false;
  if (!(h.adam_eps >= 0.f) || !(h.ln_eps > 0.f)) return *e = "eps must be positive", false;
  if (!(h.log_std_min < h.log_std_max)) return *e = "log_std_min must be < log_std_max", false;
  if (h.target_mode != SQUINT_TARGET_AVG && h.target_mode != SQUINT_TARGET_CDQ) return *e = "unknown target_mode", false;
  return true;
}

// ---- option 3: device-side precondition checks (squint.h) ---------------------------------
__device__ unsigned int g_check_bad;
__global__ void k_check_range(const int64_t* __restrict__ v, int64_t n, int64_t hi) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (v[i] < 0 || v[i] >= hi) atomicOr(&g_check_bad, 1u);
}
__global__ void k_check_distinct(const int64_t* __restrict__ v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t j = i + 1; j < n; ++j)
      if (v[j] == v[i]) atomicOr(&g_check_bad, 2u);
}
// Range check of v[0..n) against [0, hi) and (distinct) pairwise distinctness; synchronises s.
static squint_status check_indices(const int64_t* v, int64_t n, int64_t hi, bool distinct, const char* what,
                                   cudaStream_t s) {
  if (!g_check_enabled || n <= 0 || !v) return SQUINT_OK;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return SQUINT_OK;  // no synchronising check inside a capture
  }
  const unsigned int zero = 0;
  SQ_CK(cudaMemcpyToSymbolAsync(g_check_bad, &zero, sizeof(zero), 0, cudaMemcpyHostToDevice, s));
  const unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 1024);
  k_check_range<<<blocks, 256, 0, s>>>(v, n, hi);
  if (distinct) k_check_distinct<<<blocks, 256, 0, s>>>(v, n);
  unsigned int bad = 0;
  SQ_CK(cudaMemcpyFromSymbolAsync(&bad, g_check_bad, sizeof(bad), 0, cudaMemcpyDeviceToHost, s));
  SQ_CK(cudaStreamSynchronize(s));
  if (bad & 1u) return set_error(SQUINT_EINVAL, std::string(what) + ": index out of range (precondition check)");
  if (bad & 2u) return set_error(SQUINT_EINVAL, std::string(what) + ": slots not distinct (precondition check)");
  return SQUINT_OK;
}

}  // namespace sq

using namespace sq;

extern "C" {

const char* squint_last_error(void) { return g_err.c_str(); }
const char* squint_version(void) { return "libsquint 0.1 (sm_100a)"; }

squint_status squint_param_layout(const squint_dims* dims, squint_tensor_desc* out, int max_out, int* n_tensors,
                                  int64_t group_sizes[4]) {
  if (!dims) return fail(SQUINT_EINVAL, "dims is NULL");
  std::string e;
  if (!check_dims(*dims, &e)) return fail(SQUINT_EINVAL, e);
  Layout L = make_layout(*dims);
  if (n_tensors) *n_tensors = (int)L.t.size();
  if (group_sizes)
    for (int g = 0; g < 4; ++g) group_sizes[g] = L.gsize[g];
  if (out) {
    const int n = (int)L.t.size() < max_out ? (int)L.t.size() : max_out;
    for (int i = 0; i < n; ++i) {
      squint_tensor_desc& o = out[i];
      memset(&o, 0, sizeof(o));
      strncpy(o.name, L.t[i].name.c_str(), sizeof(o.name) - 1);
      o.group = L.t[i].group;
      o.offset = L.t[i].off;
      o.numel = L.t[i].numel;
      o.ndim = L.t[i].ndim;
      for (int k = 0; k < 4; ++k) o.shape[k] = L.t[i].shape[k];
    }
  }
  return SQUINT_OK;
}

squint_status squint_workspace_bytes(const squint_dims* dims, int utd, size_t* bytes) {
  if (!dims || !bytes) return fail(SQUINT_EINVAL, "NULL argument");
  std::string e;
  if (!check_dims(*dims, &e)) return fail(SQUINT_EINVAL, e);
  if (utd < 1) return fail(SQUINT_EINVAL, "utd must be >= 1");
  Layout L = make_layout(*dims);
  *bytes = dims->precision == SQUINT_BF16 ? bf16_workspace_bytes(*dims) : plan_ws(*dims, L).total;
  return SQUINT_OK;
}

squint_status squint_workspace_region(const squint_dims* dims, int region, size_t* offset, size_t* bytes) {
  if (!dims || !offset || !bytes) return fail(SQUINT_EINVAL, "NULL argument");
  std::string e;
  if (!check_dims(*dims, &e)) return fail(SQUINT_EINVAL, e);
  if (dims->precision == SQUINT_BF16) {
    if (!bf16_region(*dims, region, offset, bytes)) return fail(SQUINT_EINVAL, "unknown region");
    return SQUINT_OK;
  }
  Layout L = make_layout(*dims);
  WsLay w = plan_ws(*dims, L);
  const size_t B = dims->batch, f = sizeof(float);
  switch (region) {
    case 0: *offset = w.grad_critic; *bytes = L.gsize[0] * f; break;
    case 1: *offset = w.grad_actor; *bytes = L.gsize[1] * f; break;
    case 2: *offset = w.m; *bytes = B * head_out(*dims) * f; break;
    case 3: *offset = w.h; *bytes = B * flat_dim(*dims) * f; break;
    case 4: *offset = w.logp_cur; *bytes = B * f; break;
    case 5: *offset = w.logp_next; *bytes = B * f; break;
    case 6: *offset = w.a_cur; *bytes = B * dims->action_dim * f; break;
    case 7: *offset = w.scal; *bytes = kScal * f; break;
    case 8: *offset = w.img0; *bytes = B * dims->img_c * dims->img_h * dims->img_w; break;
    default: return fail(SQUINT_EINVAL, "unknown region");
  }
  return SQUINT_OK;
}

// squint_act_ex's weight snapshot (the ACTOR group and the CRITIC encoder head), placed past the
// act's own workspace
static size_t act_snapshot_floats(const squint_dims& d) {
  const Layout L = make_layout(d);
  return (size_t)((L.gsize[SQUINT_GROUP_ACTOR] + 3) & ~int64_t(3)) + (size_t)((L.enc_end + 3) & ~int64_t(3));
}
static size_t act_core_bytes(const squint_dims& d, int64_t n);

squint_status squint_act_workspace_bytes(const squint_dims* dims, int64_t n, size_t* bytes) {
  if (!dims || !bytes) return fail(SQUINT_EINVAL, "NULL argument");
  std::string e;
  if (!check_dims(*dims, &e)) return fail(SQUINT_EINVAL, e);
  if (n < 0) return fail(SQUINT_EINVAL, "n must be >= 0");
  *bytes = ((act_core_bytes(*dims, n) + 255) & ~size_t(255)) + act_snapshot_floats(*dims) * sizeof(float);
  return SQUINT_OK;
}

static size_t act_core_bytes(const squint_dims& dd, int64_t n) {
  const squint_dims* dims = &dd;
  if (dims->precision == SQUINT_BF16) return bf16_act_workspace_bytes(*dims, n);
  const size_t f = sizeof(float), F = flat_dim(*dims);
  WsPlan P;
  P.take(n * F * f);                           // h
  P.take(n * dims->latent * f);                // z
  P.take(n * dims->actor_hidden * f);          // h1
  P.take(n * dims->actor_hidden * f);          // h2
  P.take(n * 2 * dims->action_dim * f);        // out
  return P.top + 256;
}

squint_status squint_insert2(const uint8_t* frames, int64_t n, int c, int h, int w, int factor, const int64_t* slots,
                             uint8_t* ring, const int64_t* slots2, uint8_t* ring2, int64_t capacity,
                             squint_stream_t stream) {
  if (!ring2 != !slots2) return fail(SQUINT_EINVAL, "ring2 and slots2 must both be given or both be NULL");
  if (n < 0) return fail(SQUINT_EINVAL, "n must be >= 0");
  if (factor < 1) return fail(SQUINT_EINVAL, "factor must be >= 1");
  if (capacity < 1) return fail(SQUINT_EINVAL, "capacity must be >= 1");
  if (c < 1 || h < 1 || w < 1) return fail(SQUINT_ESHAPE, "frame dims must be positive");
  if (h % factor || w % factor) return fail(SQUINT_ESHAPE, "frame size not divisible by factor (S:41)");
  if (n == 0) return SQUINT_OK;
  if (!frames || !slots || !ring) return fail(SQUINT_EINVAL, "NULL pointer");
  if (factor == 8 && (w % 16) == 0 && (reinterpret_cast<uintptr_t>(frames) & 15))
    return fail(SQUINT_EINVAL, "frames must be 16-byte aligned");
  if (factor == 8 && (w % 16) == 0 && ((h / 8) * (w / 8) % 2))
    return fail(SQUINT_EINVAL, "odd output row length not supported by the vector path");
  {
    squint_status r = check_indices(slots, n, capacity, true, "squint_insert slots", (cudaStream_t)stream);
    if (r == SQUINT_OK) r = check_indices(slots2, n, capacity, true, "squint_insert2 slots2", (cudaStream_t)stream);
    if (r != SQUINT_OK) return r;
  }
  PhaseScope ps(0, 0, (cudaStream_t)stream);
  SQ_CK(launch_insert(frames, n, c, h, w, factor, slots, ring, (cudaStream_t)stream, slots2, ring2));
  return SQUINT_OK;
}

squint_status squint_insert_ex(const uint8_t* frames, int64_t n, int c, int h, int w, int factor, int layout,
                               const float* jitter, const int64_t* slots, uint8_t* ring, const int64_t* slots2,
                               uint8_t* ring2, int64_t capacity, squint_stream_t stream) {
  if (layout != SQUINT_LAYOUT_CHW && layout != SQUINT_LAYOUT_HWC) return fail(SQUINT_EINVAL, "unknown frame layout");
  if (!ring2 != !slots2) return fail(SQUINT_EINVAL, "ring2 and slots2 must both be given or both be NULL");
  if (n < 0) return fail(SQUINT_EINVAL, "n must be >= 0");
  if (factor < 1) return fail(SQUINT_EINVAL, "factor must be >= 1");
  if (capacity < 1) return fail(SQUINT_EINVAL, "capacity must be >= 1");
  if (c < 1 || h < 1 || w < 1) return fail(SQUINT_ESHAPE, "frame dims must be positive");
  if (h % factor || w % factor) return fail(SQUINT_ESHAPE, "frame size not divisible by factor (S:41)");
  if (jitter && c != 3) return fail(SQUINT_EINVAL, "colour jitter needs RGB frames (c == 3)");
  if (layout == SQUINT_LAYOUT_CHW && !jitter)
    return squint_insert2(frames, n, c, h, w, factor, slots, ring, slots2, ring2, capacity, stream);
  if (c > 4 || (int64_t)c * h * w > 200 * 1024)
    return fail(SQUINT_EUNSUPPORTED, "HWC / jitter insert: c <= 4 and c*h*w <= 200 KB per frame");
  if (n > 0x7fffffff) return fail(SQUINT_EUNSUPPORTED, "n > 2^31 - 1");
  if (n == 0) return SQUINT_OK;
  if (!frames || !slots || !ring) return fail(SQUINT_EINVAL, "NULL pointer");
  {
    squint_status r = check_indices(slots, n, capacity, true, "squint_insert_ex slots", (cudaStream_t)stream);
    if (r == SQUINT_OK) r = check_indices(slots2, n, capacity, true, "squint_insert_ex slots2", (cudaStream_t)stream);
    if (r != SQUINT_OK) return r;
  }
  PhaseScope ps(0, 0, (cudaStream_t)stream);
  SQ_CK(launch_insert_ex(frames, n, c, h, w, factor, layout, jitter, slots, ring, (cudaStream_t)stream, slots2, ring2));
  return SQUINT_OK;
}

squint_status squint_insert(const uint8_t* frames, int64_t n, int c, int h, int w, int factor, const int64_t* slots,
                            uint8_t* ring, int64_t capacity, squint_stream_t stream) {
  return squint_insert2(frames, n, c, h, w, factor, slots, ring, nullptr, nullptr, capacity, stream);
}

squint_status squint_stage_pinned(void* dst, const void* src, size_t bytes, squint_stream_t stream) {
  if (bytes == 0) return SQUINT_OK;
  if (!dst || !src) return fail(SQUINT_EINVAL, "NULL pointer");
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, src) != cudaSuccess || at.type != cudaMemoryTypeHost || !at.devicePointer) {
    cudaGetLastError();
    return fail(SQUINT_EINVAL, "src is not page-locked host memory");
  }
  SQ_CK(launch_stage_pinned(dst, at.devicePointer, bytes, (cudaStream_t)stream));
  return SQUINT_OK;
}

squint_status squint_soft_update(float* target, const float* online, int64_t n, float tau, squint_stream_t stream) {
  if (n < 0) return fail(SQUINT_EINVAL, "n must be >= 0");
  if (!(tau >= 0.f && tau <= 1.f)) return fail(SQUINT_EINVAL, "tau must be in [0, 1]");
  if (n == 0) return SQUINT_OK;
  if (!target || !online) return fail(SQUINT_EINVAL, "NULL pointer");
  SQ_CK(launch_polyak(target, online, n, tau, (cudaStream_t)stream));
  return SQUINT_OK;
}

squint_status squint_act(const squint_dims* dims, const squint_hparams* hp, const float* actor_params,
                         const float* critic_params, const uint8_t* frames, int64_t n, int frame_h, int frame_w,
                         const float* proprio, const float* eps, float* action_out, float* logp_out, uint8_t* ring,
                         const int64_t* slots, int64_t ring_capacity, void* workspace, squint_stream_t stream) {
  return squint_act_ex(dims, hp, actor_params, critic_params, frames, n, frame_h, frame_w, proprio, eps, action_out,
                       logp_out, ring, slots, ring_capacity, workspace, stream, nullptr);
}

squint_status squint_act_ex(const squint_dims* dims, const squint_hparams* hp, const float* actor_params,
                            const float* critic_params, const uint8_t* frames, int64_t n, int frame_h, int frame_w,
                            const float* proprio, const float* eps, float* action_out, float* logp_out, uint8_t* ring,
                            const int64_t* slots, int64_t ring_capacity, void* workspace, squint_stream_t stream,
                            squint_event_t weights_read) {
  if (!dims || !hp) return fail(SQUINT_EINVAL, "NULL dims/hparams");
  std::string e;
  if (!check_dims(*dims, &e)) return fail(SQUINT_EINVAL, e);
  if (!check_hp(*hp, &e)) return fail(SQUINT_EINVAL, e);
  if (n < 0) return fail(SQUINT_EINVAL, "n must be >= 0");
  if (frame_h % dims->img_h || frame_w % dims->img_w || frame_h / dims->img_h != frame_w / dims->img_w)
    return fail(SQUINT_ESHAPE, "frame size must be an integer multiple of the stored resolution (S:41)");
  if ((ring == nullptr) != (slots == nullptr)) return fail(SQUINT_EINVAL, "ring and slots go together");
  if (ring && ring_capacity < 1) return fail(SQUINT_EINVAL, "ring_capacity must be >= 1");
  if (dims->conv_ch > 128 || 256 % dims->conv_ch) return fail(SQUINT_EUNSUPPORTED, "conv_ch must divide 256");
  if (n == 0) return SQUINT_OK;
  if (!actor_params || !critic_params || !frames || !proprio || !action_out || !workspace)
    return fail(SQUINT_EINVAL, "NULL pointer");
  {
    squint_status r = check_indices(slots, n, ring_capacity, true, "squint_act slots", (cudaStream_t)stream);
    if (r != SQUINT_OK) return r;
  }
  const int f = frame_h / dims->img_h;
  if (f == 8 && (frame_w % 16) == 0 && (reinterpret_cast<uintptr_t>(frames) & 15))
    return fail(SQUINT_EINVAL, "frames must be 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  const squint_dims& d = *dims;
  if (weights_read) {
    // snapshot the weights the act reads (ACTOR, CRITIC encoder head) into the workspace tail, then
    // signal: from here on the act reads only the copies, so the caller may start optimizer steps
    const Layout Ls = make_layout(d);
    float* snap = reinterpret_cast<float*>(reinterpret_cast<char*>(workspace) +
                                           ((act_core_bytes(d, n) + 255) & ~size_t(255)));
    float* snap_c = snap + ((Ls.gsize[SQUINT_GROUP_ACTOR] + 3) & ~int64_t(3));
    if (cudaMemcpyAsync(snap, actor_params, Ls.gsize[SQUINT_GROUP_ACTOR] * sizeof(float), cudaMemcpyDeviceToDevice, s) !=
            cudaSuccess ||
        cudaMemcpyAsync(snap_c, critic_params, Ls.enc_end * sizeof(float), cudaMemcpyDeviceToDevice, s) != cudaSuccess ||
        cudaEventRecord((cudaEvent_t)weights_read, s) != cudaSuccess)
      return fail(SQUINT_ECUDA, "squint_act_ex: weight snapshot");
    actor_params = snap;
    critic_params = snap_c;
  }
  if (d.precision == SQUINT_BF16)
    return bf16_act(d, *hp, actor_params, critic_params, frames, n, f, proprio, eps, action_out, logp_out, ring, slots,
                    workspace, s);
  Layout L = make_layout(d);
  const int F = flat_dim(d), Lt = d.latent, Ha = d.actor_hidden, A = d.action_dim, P = d.proprio_dim;
  const size_t fl = sizeof(float);
  WsPlan WP;
  char* ws = reinterpret_cast<char*>(workspace);
  float* h = reinterpret_cast<float*>(ws + WP.take(n * F * fl));
  float* z = reinterpret_cast<float*>(ws + WP.take(n * Lt * fl));
  float* h1 = reinterpret_cast<float*>(ws + WP.take(n * Ha * fl));
  float* h2 = reinterpret_cast<float*>(ws + WP.take(n * Ha * fl));
  float* out = reinterpret_cast<float*>(ws + WP.take(n * 2 * A * fl));
  const int gC = SQUINT_GROUP_CRITIC, gA = SQUINT_GROUP_ACTOR;
  std::optional<PhaseScope> ps;
  ps.emplace(1, 0, s);
  {
    EncFwdArgs a;
    memset(&a, 0, sizeof(a));
    a.mode = 1;
    a.src[0] = frames;
    a.factor = f;
    a.ring = ring;
    a.slots = slots;
    a.B = (int)n;
    a.nsrc = 1;
    a.w1 = critic_params + L.off(gC, "enc.conv1.w");
    a.b1 = critic_params + L.off(gC, "enc.conv1.b");
    a.w2 = critic_params + L.off(gC, "enc.conv2.w");
    a.b2 = critic_params + L.off(gC, "enc.conv2.b");
    a.h[0] = h;
    a.C = d.conv_ch;
    a.c_in = d.img_c;
    a.H = d.img_h;
    a.pad = d.pad;
    SQ_CK(launch_enc_fwd(a, s));
  }
  const LinV ap = projv(actor_params, L, gA, "actor");
  const MlpV am = mlpv(actor_params, L, gA, "actor");
  const int M = (int)n;
  ps.reset();
  ps.emplace(2, 0, s);
  DenseBatch b;
  b.nprob = 1;
  b.p[0] = fwd_prob(M, ap, Lt, F, {seg(h, F, F)}, EPI_LN_TANH, z, nullptr, nullptr, hp->ln_eps);
  SQ_CK(run_dense(b, s));
  b.p[0] = fwd_prob(M, am.l1, Ha, Lt + P, {seg(z, Lt, Lt), seg(proprio, P, P)}, EPI_LN_RELU, h1, nullptr, nullptr,
                    hp->ln_eps);
  SQ_CK(run_dense(b, s));
  b.p[0] = fwd_prob(M, am.l2, Ha, Ha, {seg(h1, Ha, Ha)}, EPI_LN_RELU, h2, nullptr, nullptr, hp->ln_eps);
  SQ_CK(run_dense(b, s));
  b.p[0] = fwd_prob(M, am.l3, 2 * A, Ha, {seg(h2, Ha, Ha)}, EPI_TG_FWD, out, nullptr, nullptr, hp->ln_eps);
  b.p[0].eps = eps;
  b.p[0].act = action_out;
  b.p[0].logp = logp_out;
  b.p[0].lo = hp->log_std_min;
  b.p[0].hi = hp->log_std_max;
  SQ_CK(run_dense(b, s));
  return SQUINT_OK;
}

squint_status squint_update(const squint_dims* dims, const squint_hparams* hp, const squint_replay* replay,
                            const int64_t* idx, const uint8_t* shifts, const float* eps, int utd,
                            const squint_state* state, float* metrics, void* workspace, size_t workspace_bytes,
                            void* comm, squint_stream_t stream) {
  if (!dims || !hp || !replay || !state) return fail(SQUINT_EINVAL, "NULL struct argument");
  std::string e;
  if (!check_dims(*dims, &e)) return fail(SQUINT_EINVAL, e);
  if (!check_hp(*hp, &e)) return fail(SQUINT_EINVAL, e);
  if (utd < 1) return fail(SQUINT_EINVAL, "utd must be >= 1 (Q30)");
  if (replay->size < 1) return fail(SQUINT_EINVAL, "replay is empty (S:129)");
  if (replay->size > replay->capacity) return fail(SQUINT_EINVAL, "replay size > capacity");
  if (dims->conv_ch > 128 || 256 % dims->conv_ch) return fail(SQUINT_EUNSUPPORTED, "conv_ch must divide 256");
  if (!idx || !shifts || !eps || !metrics || !workspace) return fail(SQUINT_EINVAL, "NULL pointer");
  if (!replay->obs || !replay->next_obs || !replay->proprio || !replay->next_proprio || !replay->action ||
      !replay->reward || !replay->done)
    return fail(SQUINT_EINVAL, "NULL replay field");
  if (!state->critic || !state->critic_target || !state->actor || !state->log_alpha || !state->m_critic ||
      !state->v_critic || !state->m_actor || !state->v_actor || !state->m_alpha || !state->v_alpha || !state->step)
    return fail(SQUINT_EINVAL, "NULL state field");
  {
    squint_status r = check_indices(idx, (int64_t)utd * dims->batch, replay->size, false, "squint_update idx",
                                    (cudaStream_t)stream);
    if (r != SQUINT_OK) return r;
  }
  Comm* cm = reinterpret_cast<Comm*>(comm);
  if (dims->precision == SQUINT_BF16) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) {
      cudaGetLastError();
      cs = cudaStreamCaptureStatusActive;  // unknown: launch directly
    }
    // (the debug switches allocate or synchronise inside their launches: no capture with them)
    static const bool no_graph = getenv("SQUINT_NO_GRAPH") || getenv("SQUINT_DEBUG_SYNC") || getenv("SQUINT_GEMM_DBG") ||
                                 getenv("SQUINT_CHAIN_DBG") || getenv("SQUINT_ENC_DBG") || getenv("SQUINT_TCE_DBG");
    const bool branch = bf16_prepare();
    if (no_graph || cm || cs != cudaStreamCaptureStatusNone || instrumentation_active())
      return bf16_update(*dims, *hp, *replay, idx, shifts, eps, utd, *state, metrics, workspace, workspace_bytes, cm, s);
    // the ~30 launches per update are captured once per distinct argument set and replayed as a
    // CUDA graph (host cost of a call: one graph launch)
    std::string key;
    auto put = [&](const void* p, size_t n) { key.append(reinterpret_cast<const char*>(p), n); };
    put(dims, sizeof(*dims));
    put(hp, sizeof(*hp));
    {
      // replay.size grows while the ring fills; it only bounds the host-side index check, so it is
      // not part of the key (the captured launches do not read it)
      squint_replay rk = *replay;
      rk.size = 0;
      put(&rk, sizeof(rk));
    }
    put(state, sizeof(*state));
    const void* ptrs[6] = {idx, shifts, eps, metrics, workspace, nullptr};
    put(ptrs, sizeof(ptrs));
    put(&utd, sizeof(utd));
    put(&workspace_bytes, sizeof(workspace_bytes));
    put(&branch, sizeof(branch));
    const int opts = bf16_options();
    put(&opts, sizeof(opts));
    struct Entry {
      std::string key;
      cudaGraphExec_t exec;
    };
    static thread_local std::vector<Entry> cache;
    cudaGraphExec_t exec = nullptr;
    for (auto& e : cache)
      if (e.key == key) exec = e.exec;
    if (!exec) {
      // captured on a private stream (the caller's may be the legacy default stream, which cannot
      // capture); the graph is then launched on the caller's stream
      static thread_local cudaStream_t cap = nullptr;
      if (!cap && cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess)
        return fail(SQUINT_ECUDA, "update graph: capture stream");
      if (cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
        return fail(SQUINT_ECUDA, "update graph: begin capture failed");
      squint_status r = bf16_update(*dims, *hp, *replay, idx, shifts, eps, utd, *state, metrics, workspace,
                                    workspace_bytes, cm, cap);
      cudaGraph_t g = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(cap, &g);
      if (r != SQUINT_OK || ce != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        return r != SQUINT_OK ? r : fail(SQUINT_ECUDA, std::string("update graph capture: ") + cudaGetErrorString(ce));
      }
      const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
      cudaGraphDestroy(g);
      if (ie != cudaSuccess) return fail(SQUINT_ECUDA, std::string("update graph instantiate: ") + cudaGetErrorString(ie));
      if (cache.size() >= 8) {
        cudaGraphExecDestroy(cache.front().exec);
        cache.erase(cache.begin());
      }
      cache.push_back(Entry{key, exec});
    }
    const cudaError_t le = cudaGraphLaunch(exec, s);
    if (le != cudaSuccess) return fail(SQUINT_ECUDA, std::string("update graph launch: ") + cudaGetErrorString(le));
    return SQUINT_OK;
  }
  Layout L = make_layout(*dims);
  WsLay w = plan_ws(*dims, L);
  if (workspace_bytes < w.total) return fail(SQUINT_EINVAL, "workspace too small (see squint_workspace_bytes)");
  const int nranks = cm ? comm_nranks(cm) : 1;
  const float inv_btotal = 1.0f / ((float)dims->batch * (float)nranks);
  Ctx c{*dims, *hp, L, w, reinterpret_cast<char*>(workspace), (cudaStream_t)stream};
  const size_t B = dims->batch, A = dims->action_dim;
  for (int j = 0; j < utd; ++j) {
    const int64_t* ij = idx + j * B;
    const uint8_t* sj = shifts + j * B * 4;
    const float* ej = eps + j * 2 * B * A;
    float* mj = metrics + j * 8;
    squint_status st = update_one(c, *replay, ij, sj, ej, *state, mj, cm, inv_btotal, j);
    if (st != SQUINT_OK) return st;
  }
  return SQUINT_OK;
}

squint_status squint_comm_unique_id(void* id_out) {
  if (!id_out) return fail(SQUINT_EINVAL, "NULL id");
  if (comm_unique_id(id_out) != 0) return fail(SQUINT_ENCCL, comm_error());
  return SQUINT_OK;
}
squint_status squint_comm_init(void** comm, const void* id, int rank, int nranks) {
  if (!comm || !id) return fail(SQUINT_EINVAL, "NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SQUINT_EINVAL, "bad rank/nranks");
  Comm* c = nullptr;
  if (comm_init(&c, id, rank, nranks) != 0) return fail(SQUINT_ENCCL, comm_error());
  *comm = c;
  return SQUINT_OK;
}
squint_status squint_comm_set_mode(void* comm, int mode) {
  if (!comm) return fail(SQUINT_EINVAL, "NULL comm");
  if (mode != 0 && mode != 1) return fail(SQUINT_EINVAL, "mode must be 0 or 1");
  if (comm_set_mode(reinterpret_cast<Comm*>(comm), mode) != 0) return fail(SQUINT_EUNSUPPORTED, comm_error());
  return SQUINT_OK;
}
squint_status squint_comm_destroy(void* comm) {
  if (comm) comm_destroy(reinterpret_cast<Comm*>(comm));
  return SQUINT_OK;
}

}  // extern "C"
