"""Closed-form pins of the oracle's composition (round-2 additions).

Each test builds a degenerate but valid network whose outputs the paper's definitions fix by
hand, so a plausible mistake in the oracle's orchestration (not only in its layers) fails:

* the C51 target's terminal mask (Q22): with d = 1 every atom collapses onto
  r, so m is the two-atom split of the point mass at clip(r) -- whatever the networks say;
* ``act`` (Algorithm 1 line 5: a ~ pi_phi(f_psi(o), s)): with the actor's last layer
  zeroed the action and log pi are closed forms of its bias; the result depends on psi and
  phi and on nothing in theta (the critic's projection);
* the order of one update (Q19) and the metrics row: with the heads' second
  LayerNorm affine zeroed (h2 = 0, so every head outputs its bias) and the actor's last layer
  zeroed, the critic step moves only the heads' output biases by one Adam step, the alpha step
  is one Adam step on -alpha_0 (mean log pi + H_t) (Q17), and the actor loss must use alpha+
  and the stepped biases theta+;
* the random-shift columns (Q5): (dx, dy) of obs and (dx', dy') of next_obs, checked with a
  single bright pixel whose shifted position is known.
"""
import math

import numpy as np

import oracle as O
import squint_inputs as SI

TINY = dict(img_c=3, img_h=16, img_w=16, pad=2, conv_ch=4, latent=8, proprio_dim=3, action_dim=2,
            critic_hidden=16, actor_hidden=16, n_atoms=7, v_min=-2.0, v_max=2.0, batch=5)
LOG_2PI = math.log(2.0 * math.pi)


def _setup(seed=0, **over):
    dims = dict(TINY, **over)
    d = O.Dims(**dims)
    specs = O.param_specs(d)
    vals = SI.make_params(specs, seed=seed + 1, perturb=True)
    R = SI.make_replay(40, dims, seed=seed)
    return d, specs, vals, R


def _point_mass_split(r, v_min, v_max, n):
    """The projection of a point mass at clip(r) onto z_j = v_min + j dz (Q23), by hand."""
    dz = (v_max - v_min) / (n - 1)
    m = np.zeros((len(r), n))
    for k, rk in enumerate(r):
        g = min(max(float(rk), v_min), v_max)
        b = (g - v_min) / dz
        lo, hi = math.floor(b), math.ceil(b)
        if lo == hi:
            m[k, lo] = 1.0
        else:
            m[k, lo] = hi - b
            m[k, hi] = b - lo
    return m


# ---- C51 terminal mask (Q22) ------------------------------------------------------------------
def test_c51_all_terminal_is_point_mass_of_reward():
    d, specs, vals, R = _setup(seed=3)
    st = O.init_state(specs, vals)
    hp = O.HParams(target_entropy=-2.0)
    B = d.batch
    rng = np.random.default_rng(0)
    hn = rng.uniform(0.0, 1.0, (B, d.flat))
    sn = rng.standard_normal((B, d.proprio_dim))
    r = np.array([0.3, -1.7, 2.9, -3.5, 1.0])     # two clip onto the edge atoms
    eps = rng.standard_normal((B, d.action_dim))
    m, _ = O.target_distribution(d, hp, st["target"], st["actor"], hn, sn, r, np.ones(B, np.uint8), eps, 0.8)
    assert np.abs(m - _point_mass_split(r, d.v_min, d.v_max, d.n_atoms)).max() < 1e-12


def test_c51_terminal_rows_independent_of_the_rest():
    """Mixed batch: the terminal rows are the closed form; the others are not point masses."""
    d, specs, vals, R = _setup(seed=4)
    st = O.init_state(specs, vals)
    hp = O.HParams(target_entropy=-2.0)
    B = d.batch
    rng = np.random.default_rng(1)
    hn = rng.uniform(0.0, 1.0, (B, d.flat))
    sn = rng.standard_normal((B, d.proprio_dim))
    r = rng.uniform(0.0, 1.0, B)
    done = np.array([1, 0, 1, 0, 0], np.uint8)
    eps = rng.standard_normal((B, d.action_dim))
    m, _ = O.target_distribution(d, hp, st["target"], st["actor"], hn, sn, r, done, eps, 0.5)
    ref = _point_mass_split(r, d.v_min, d.v_max, d.n_atoms)
    assert np.abs(m[done == 1] - ref[done == 1]).max() < 1e-12
    assert (np.count_nonzero(m[done == 0] > 1e-9, axis=1) > 2).all()
    assert np.abs(m.sum(axis=1) - 1.0).max() < 1e-12


# ---- act (Algorithm 1 line 5) ---------------------------------------------------------------
def _zero_actor_head(vals, d):
    vals = dict(vals)
    vals[("actor", "actor.l3.w")] = np.zeros_like(vals[("actor", "actor.l3.w")])
    return vals


def _tg_closed_form(bias, eps, lo, hi):
    """a = tanh(mu + sigma eps), log pi = sum_d [-eps^2/2 - log sigma - ln(2 pi)/2 - ln(1 - a^2 + 1e-6)],
    log sigma = lo + (hi - lo)/2 (tanh l + 1) (Q13, Q14), for out = bias = [mu | l]."""
    A = bias.shape[0] // 2
    mu, l = bias[:A], bias[A:]
    log_sigma = lo + 0.5 * (hi - lo) * (np.tanh(l) + 1.0)
    u = mu[None, :] + np.exp(log_sigma)[None, :] * eps
    a = np.tanh(u)
    logp = (-0.5 * eps * eps - log_sigma[None, :] - 0.5 * LOG_2PI - np.log(1.0 - a * a + 1e-6)).sum(axis=1)
    return a, logp


def test_act_zero_head_closed_form():
    d, specs, vals, R = _setup(seed=5)
    vals = _zero_actor_head(vals, d)
    st = O.init_state(specs, vals)
    hp = O.HParams()
    frames = SI.make_frames(4, 128, seed=2)
    proprio = np.random.default_rng(2).standard_normal((4, d.proprio_dim)).astype(np.float32)
    b3 = np.asarray(vals[("actor", "actor.l3.b")], np.float64)
    # mean action (eps = None): a = tanh(mu), log pi at eps = 0 (R-act)
    a, logp, _ = O.act(d, hp, st["critic"], st["actor"], frames, proprio)
    a_ref, lp_ref = _tg_closed_form(b3, np.zeros((4, d.action_dim)), hp.log_std_min, hp.log_std_max)
    assert np.abs(a - np.tanh(b3[:d.action_dim])[None, :]).max() < 1e-15
    assert np.abs(logp - lp_ref).max() < 1e-12
    eps = np.random.default_rng(3).standard_normal((4, d.action_dim)).astype(np.float32)
    a, logp, _ = O.act(d, hp, st["critic"], st["actor"], frames, proprio, eps)
    a_ref, lp_ref = _tg_closed_form(b3, eps.astype(np.float64), hp.log_std_min, hp.log_std_max)
    assert np.abs(a - a_ref).max() < 1e-14 and np.abs(logp - lp_ref).max() < 1e-12


def test_act_reads_psi_and_phi_not_theta():
    """a = pi_phi(f_psi(o), s) (Q8: the actor's own projection): perturbing the critic's
    projection or heads leaves act bitwise unchanged; perturbing the actor projection or the
    encoder changes it."""
    d, specs, vals, R = _setup(seed=6)
    hp = O.HParams()
    frames = SI.make_frames(3, 128, seed=4)
    proprio = np.random.default_rng(4).standard_normal((3, d.proprio_dim)).astype(np.float32)
    eps = np.random.default_rng(5).standard_normal((3, d.action_dim)).astype(np.float32)

    def run(v):
        st = O.init_state(specs, v)
        a, lp, _ = O.act(d, hp, st["critic"], st["actor"], frames, proprio, eps)
        return a, lp

    a0, lp0 = run(vals)
    for name in ("critic.proj.w", "critic.proj.b", "critic.proj.ln.g", "critic.proj.ln.b", "critic.q1.l1.w"):
        v = dict(vals)
        v[("critic", name)] = vals[("critic", name)] + 0.3
        a1, lp1 = run(v)
        assert np.array_equal(a0, a1) and np.array_equal(lp0, lp1), name
    rng = np.random.default_rng(6)
    for grp, name in (("actor", "actor.proj.w"), ("actor", "actor.proj.ln.b"), ("critic", "enc.conv1.b")):
        v = dict(vals)
        # (a random perturbation: a constant added to a projection weight is removed by the LayerNorm)
        v[(grp, name)] = vals[(grp, name)] + rng.uniform(-0.3, 0.3, vals[(grp, name)].shape)
        a1, lp1 = run(v)
        assert np.abs(a1 - a0).max() > 1e-4, name


# ---- one update with hand-computable networks (Q17-Q19, Q24, Q25, metrics) ---------------------
def _degenerate_vals(vals):
    """Heads (online and target) with ln2 affine = 0 -> h2 = 0 -> logits = l3.b; actor l3.w = 0."""
    v = dict(vals)
    for grp in ("critic", "target"):
        for i in (1, 2):
            for t in ("ln2.g", "ln2.b"):
                v[(grp, f"critic.q{i}.{t}")] = np.zeros_like(vals[(grp, f"critic.q{i}.{t}")])
    v[("actor", "actor.l3.w")] = np.zeros_like(vals[("actor", "actor.l3.w")])
    return v


def _softmax(x):
    e = np.exp(x - x.max())
    return e / e.sum()


def _adam1(g, lr, eps=1e-8):
    """First Adam step from zero moments (Q26): m_hat = g, v_hat = g^2."""
    return -lr * g / (np.abs(g) + eps)


def test_update_closed_form_order_and_metrics():
    d, specs, vals, R = _setup(seed=7)
    vals = _degenerate_vals(vals)
    vals[("alpha", "log_alpha")] = np.array([-0.4], np.float32)
    hp = O.HParams(target_entropy=-2.0, lr_critic=0.05, lr_actor=0.01, lr_alpha=0.05, gamma=0.9)
    st = O.init_state(specs, vals)
    B, A, N = d.batch, d.action_dim, d.n_atoms
    idx = SI.make_indices(1, B, 40, seed=8)
    sh = SI.make_shifts(1, B, d.pad, seed=8)
    eps = SI.make_eps(1, B, A, seed=9).astype(np.float64)
    trace = []
    st1, met = O.update(d, hp, R, idx, sh, eps, st, trace=trace)
    tr = trace[0]
    lo, hi = hp.log_std_min, hp.log_std_max
    b3a = np.asarray(vals[("actor", "actor.l3.b")], np.float64)
    _, logp_next = _tg_closed_form(b3a, eps[0, 0], lo, hi)
    a_cur, logp = _tg_closed_form(b3a, eps[0, 1], lo, hi)
    assert np.abs(tr["logp_next"] - logp_next).max() < 1e-12
    assert np.abs(tr["logp"] - logp).max() < 1e-12
    assert np.abs(tr["a_cur"] - a_cur).max() < 1e-14
    # target (lines 11-13): pbar is the same for every row; the projection is pinned on its own
    z, dz = O.make_support(d.v_min, d.v_max, N)
    tb = [np.asarray(vals[("target", f"critic.q{i}.l3.b")], np.float64) for i in (1, 2)]
    pbar = 0.5 * (_softmax(tb[0]) + _softmax(tb[1]))
    la0 = float(np.float32(-0.4))      # the state holds log alpha as stored (float32)
    alpha0 = math.exp(la0)
    r = R["reward"][idx[0]].astype(np.float64)
    nd = 1.0 - R["done"][idx[0]].astype(np.float64)
    m = O.categorical_project(np.tile(pbar, (B, 1)), r, nd, hp.gamma, alpha0 * logp_next, d.v_min, d.v_max)
    assert np.abs(tr["m"] - m).max() < 1e-12
    # critic loss and gradient (lines 14-15, Q24): only the output biases get a gradient
    cb = [np.asarray(vals[("critic", f"critic.q{i}.l3.b")], np.float64) for i in (1, 2)]
    LQ = sum(float(-(m * np.log(_softmax(cb[i]))[None, :]).sum(axis=1).mean()) for i in (0, 1))
    assert abs(met[0, 0] - LQ) < 1e-12
    g3 = [(_softmax(cb[i])[None, :] - m).mean(axis=0) for i in (0, 1)]
    for name, g in tr["grad_critic"].items():
        if name in ("critic.q1.l3.b", "critic.q2.l3.b"):
            assert np.abs(g - g3[int(name[8]) - 1]).max() < 1e-14, name
        else:
            assert not np.any(g), name
    assert abs(met[0, 6] - math.sqrt(sum(float((g * g).sum()) for g in g3))) < 1e-13
    cb1 = [cb[i] + _adam1(g3[i], hp.lr_critic) for i in (0, 1)]
    for i in (0, 1):
        assert np.abs(st1["critic"][f"critic.q{i + 1}.l3.b"] - cb1[i]).max() < 1e-15
    # alpha step (lines 16-17, Q17, Q18): pre-step phi's sample at the current states
    La = -alpha0 * (logp.mean() + hp.target_entropy)
    assert abs(met[0, 2] - La) < 1e-13
    log_alpha1 = la0 + _adam1(np.array([La]), hp.lr_alpha)[0]
    alpha1 = math.exp(log_alpha1)
    assert abs(st1["log_alpha"] - log_alpha1) < 1e-15
    assert abs(met[0, 3] - alpha1) < 1e-14
    # actor loss (lines 18-22, Q19, Q25): alpha+ and the stepped critic theta+
    Q1 = [float(_softmax(cb1[i]) @ z) for i in (0, 1)]
    Lpi = float(alpha1 * logp.mean()) - 0.5 * (Q1[0] + Q1[1])
    assert abs(met[0, 1] - Lpi) < 1e-12
    assert abs(met[0, 4] - 0.5 * (Q1[0] + Q1[1])) < 1e-12
    assert abs(met[0, 5] - (-logp.mean())) < 1e-13     # entropy metric = -mean log pi
    # the actor gradient: Q does not depend on a~ (h2 = 0 in theta+ too), so only alpha+ log pi / B
    eps1 = eps[0, 1]
    mu, l = b3a[:A], b3a[A:]
    sig = np.exp(lo + 0.5 * (hi - lo) * (np.tanh(l) + 1.0))
    a = np.tanh(mu[None, :] + sig[None, :] * eps1)
    dsq = 2.0 * a * (1.0 - a * a) / (1.0 - a * a + 1e-6)       # d/du of -ln(1 - tanh(u)^2 + 1e-6)
    dmu = dsq
    dl = (-1.0 + dsq * sig[None, :] * eps1) * 0.5 * (hi - lo) * (1.0 - np.tanh(l) ** 2)[None, :]
    gb3 = alpha1 / B * np.concatenate([dmu, dl], axis=1).sum(axis=0)
    assert np.abs(tr["grad_actor"]["actor.l3.b"] - gb3).max() < 1e-12 * max(1.0, np.abs(gb3).max())
    # Polyak (line 24, Q28): target biases move toward theta+
    for i in (0, 1):
        ref = (1 - hp.tau) * tb[i] + hp.tau * cb1[i]
        assert np.abs(st1["target"][f"critic.q{i + 1}.l3.b"] - ref).max() < 1e-15


# ---- random-shift columns (Q5) ----------------------------------------------------------------
def test_update_shift_columns_single_pixel():
    d, specs, vals, R = _setup(seed=10)
    st = O.init_state(specs, vals)
    hp = O.HParams(target_entropy=-2.0)
    B, p = d.batch, d.pad
    idx = np.arange(B, dtype=np.int64)[None, :] + 3
    sh = np.array([[[0, 4, 3, 1], [4, 0, 1, 3], [2, 2, 0, 0], [1, 3, 4, 4], [3, 0, 2, 4]]], np.uint8)
    R = dict(R)
    R["obs"] = np.zeros_like(R["obs"])
    R["next_obs"] = np.zeros_like(R["next_obs"])
    exp_o = np.zeros((B, 3, 16, 16), np.uint8)
    exp_n = np.zeros((B, 3, 16, 16), np.uint8)
    for k in range(B):
        y0, x0, y1, x1 = 5 + k, 9 - k, 10 - k, 6 + k
        R["obs"][idx[0, k], k % 3, y0, x0] = 255
        R["next_obs"][idx[0, k], (k + 1) % 3, y1, x1] = 200
        dx, dy, dxn, dyn = (int(v) for v in sh[0, k])
        # out[y][x] = in[y + dy - p][x + dx - p]: the pixel moves to (y0 - dy + p, x0 - dx + p)
        exp_o[k, k % 3, y0 - dy + p, x0 - dx + p] = 255
        exp_n[k, (k + 1) % 3, y1 - dyn + p, x1 - dxn + p] = 200
    eps = SI.make_eps(1, B, d.action_dim, seed=1).astype(np.float64)
    trace = []
    O.update(d, hp, R, idx, sh, eps, st, trace=trace)
    h_ref, _ = O.encoder_fwd(st["critic"], exp_o.astype(np.float64) / 255.0)
    hn_ref, _ = O.encoder_fwd(st["critic"], exp_n.astype(np.float64) / 255.0)
    assert np.abs(trace[0]["h"] - h_ref).max() < 1e-14
    assert np.abs(trace[0]["hn"] - hn_ref).max() < 1e-14
