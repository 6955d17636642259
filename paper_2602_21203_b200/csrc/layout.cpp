// layout.cpp -- parameter layout table (names follow the paper's roles; shapes per Q7-Q12).
#include "layout.hpp"

#include <cstdio>
#include <cstring>

namespace sq {

int64_t Layout::off(int group, const std::string& name) const {
  for (const auto& x : t)
    if (x.group == group && x.name == name) return x.off;
  return -1;
}

bool check_dims(const squint_dims& d, std::string* err) {
  char buf[256];
  auto fail = [&](const char* m) {
    if (err) *err = m;
    return false;
  };
  if (d.img_c < 1 || d.img_h < 7 || d.img_w < 7) return fail("img dims too small (need >= 7)");
  if (d.img_h != d.img_w) return fail("square images only");
  if (d.pad < 0 || d.pad > 8) return fail("pad must be in [0, 8]");
  if (d.conv_ch < 1 || d.latent < 2 || d.proprio_dim < 0 || d.action_dim < 1) return fail("invalid layer width");
  if (d.critic_hidden < 2 || d.actor_hidden < 2) return fail("hidden width must be >= 2");
  if (d.critic_kind != SQUINT_CRITIC_C51 && d.critic_kind != SQUINT_CRITIC_MSE) return fail("unknown critic_kind");
  const bool c51 = d.critic_kind == SQUINT_CRITIC_C51;
  if (c51 && d.n_atoms < 2) return fail("n_atoms must be >= 2 (S:272)");
  if (c51 && !(d.v_min < d.v_max)) return fail("v_min must be < v_max (S:272)");
  if (d.batch < 1) return fail("batch must be >= 1");
  if (d.precision != SQUINT_FP32 && d.precision != SQUINT_BF16) return fail("unknown precision");
  if (d.critic_hidden > 512 || d.actor_hidden > 512) return fail("hidden width > 512 not built");
  if ((c51 && d.n_atoms > 512) || d.latent > 512) return fail("n_atoms/latent > 512 not built");
  if (2 * d.action_dim > 64) return fail("action_dim > 32 not built");
  if (d.img_c * d.img_h * d.img_w > 4096) return fail("stored image larger than 4096 bytes not built");
  (void)buf;
  return true;
}

namespace {
struct Builder {
  Layout L;
  void add(int g, const std::string& n, std::initializer_list<int> shape) {
    TInfo x;
    x.name = n;
    x.group = g;
    x.ndim = (int)shape.size();
    int64_t ne = 1;
    int i = 0;
    for (int s : shape) {
      x.shape[i++] = s;
      ne *= s;
    }
    for (; i < 4; ++i) x.shape[i] = 0;
    x.numel = ne;
    int64_t o = (L.gsize[g] + 31) & ~int64_t(31);
    x.off = o;
    L.gsize[g] = o + ne;
    L.t.push_back(x);
  }
  void mlp(int g, const std::string& p, int nin, int hid, int nout) {
    add(g, p + ".l1.w", {hid, nin});
    add(g, p + ".l1.b", {hid});
    add(g, p + ".ln1.g", {hid});
    add(g, p + ".ln1.b", {hid});
    add(g, p + ".l2.w", {hid, hid});
    add(g, p + ".l2.b", {hid});
    add(g, p + ".ln2.g", {hid});
    add(g, p + ".ln2.b", {hid});
    add(g, p + ".l3.w", {nout, hid});
    add(g, p + ".l3.b", {nout});
  }
  void proj(int g, const std::string& p, int flat, int lat) {
    add(g, p + ".proj.w", {lat, flat});
    add(g, p + ".proj.b", {lat});
    add(g, p + ".proj.ln.g", {lat});
    add(g, p + ".proj.ln.b", {lat});
  }
};
}  // namespace

Layout make_layout(const squint_dims& d) {
  Builder b;
  const int C = d.conv_ch, F = flat_dim(d);
  const int nq = d.latent + d.proprio_dim + d.action_dim, npi = d.latent + d.proprio_dim;
  auto critic_tail = [&](int g) {
    b.proj(g, "critic", F, d.latent);
    b.mlp(g, "critic.q1", nq, d.critic_hidden, head_out(d));
    b.mlp(g, "critic.q2", nq, d.critic_hidden, head_out(d));
  };
  b.add(SQUINT_GROUP_CRITIC, "enc.conv1.w", {C, d.img_c, 3, 3});
  b.add(SQUINT_GROUP_CRITIC, "enc.conv1.b", {C});
  b.add(SQUINT_GROUP_CRITIC, "enc.conv2.w", {C, C, 3, 3});
  b.add(SQUINT_GROUP_CRITIC, "enc.conv2.b", {C});
  b.L.gsize[SQUINT_GROUP_CRITIC] = (b.L.gsize[SQUINT_GROUP_CRITIC] + 31) & ~int64_t(31);
  b.L.enc_end = b.L.gsize[SQUINT_GROUP_CRITIC];
  critic_tail(SQUINT_GROUP_CRITIC);
  critic_tail(SQUINT_GROUP_TARGET);
  b.proj(SQUINT_GROUP_ACTOR, "actor", F, d.latent);
  b.mlp(SQUINT_GROUP_ACTOR, "actor", npi, d.actor_hidden, 2 * d.action_dim);
  b.add(SQUINT_GROUP_ALPHA, "log_alpha", {1});
  for (int g = 0; g < 4; ++g) b.L.gsize[g] = (b.L.gsize[g] + 31) & ~int64_t(31);
  return b.L;
}

}  // namespace sq
